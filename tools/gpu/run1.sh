set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r1s3_pytest_gpu.log
timeout 300 python tools/step_once.py --config 5 --steps 3 > gpurun_out/r1s3_step5.log 2>&1
BBF_DEBUG=1 timeout 300 python tools/step_once.py --config 3 --steps 2 > gpurun_out/r1s3_step3.log 2>&1
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/r1s3_bench5.json 2> gpurun_out/r1s3_bench5.err
timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r1s3_bench3.json 2> gpurun_out/r1s3_bench3.err
tail -3 gpurun_out/*.log
