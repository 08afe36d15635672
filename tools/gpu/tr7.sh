timeout 600 python tools/trace_step.py --config 4 --steps 2 > gpurun_out/tr7_c4.txt 2>&1; timeout 600 python tools/trace_step.py --config 3 --steps 2 > gpurun_out/tr7_c3.txt 2>&1
