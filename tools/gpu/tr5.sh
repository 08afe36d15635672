timeout 600 python tools/trace_step.py --config 5 --steps 2 > gpurun_out/tr5_c5.txt 2>&1; timeout 600 python tools/trace_step.py --config 3 --steps 2 > gpurun_out/tr5_c3.txt 2>&1
