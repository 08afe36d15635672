timeout 600 python tools/trace_step.py --config 5 > gpurun_out/tr1_c5.txt 2>&1; cat gpurun_out/tr1_c5.txt | head -80
