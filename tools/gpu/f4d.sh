timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/b5_bench4.json 2>gpurun_out/b5_bench4.err
python tools/step_once.py --config 4 --steps 1 --path dense > gpurun_out/pr_step4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_dense_f4 -c 1 -o gpurun_out/pr_k_dense_f4q_c4 \
  python tools/step_once.py --config 4 --steps 1 --path dense > gpurun_out/pr_ncu4.log 2>&1
tail -1 gpurun_out/pr_ncu4.log
