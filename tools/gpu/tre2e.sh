timeout 600 python tools/trace_step.py --config 5 --steps 4 --e2e > gpurun_out/tr_e2e.txt 2>&1; grep -A30 "^copies" gpurun_out/tr_e2e.txt | grep -v "all ops" | head -32
