timeout 600 python tools/trace_step.py --config 5 --steps 3 > gpurun_out/tr2_c5.txt 2>&1; head -3 gpurun_out/tr2_c5.txt; sed -n '/longest runtime/,$p' gpurun_out/tr2_c5.txt
