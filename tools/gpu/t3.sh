timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not dense" 2>&1 | tail -3 > gpurun_out/t3_pytest.log
for c in 3 5; do BBF_DEBUG=1 timeout 300 python tools/step_once.py --config $c --steps 2 > gpurun_out/t3_step$c.log 2>&1; done
cat gpurun_out/t3_pytest.log; tail -n 2 gpurun_out/t3_step3.log gpurun_out/t3_step5.log
