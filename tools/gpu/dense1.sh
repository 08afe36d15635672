BBF_DEBUG=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "dense" 2>&1 | tail -30 > gpurun_out/d1_pytest.log
cat gpurun_out/d1_pytest.log
