timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "dense" 2>&1 | tail -2
BBF_DEBUG=1 timeout 120 python tools/step_once.py --config 4 --steps 3 --path dense 2>&1 | grep "dense:" | tail -1
