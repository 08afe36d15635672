timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/trace_step.py --config 5 --steps 2 > gpurun_out/tr6_c5.txt 2>&1; grep -A14 "busy by op" gpurun_out/tr6_c5.txt; head -3 gpurun_out/tr6_c5.txt
