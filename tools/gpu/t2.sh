timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/t2_pytest.log
for c in 3 5; do BBF_DEBUG=1 timeout 300 python tools/step_once.py --config $c --steps 3 > gpurun_out/t2_step$c.log 2>&1; done
cat gpurun_out/t2_pytest.log; tail -n 3 gpurun_out/t2_step3.log gpurun_out/t2_step5.log
