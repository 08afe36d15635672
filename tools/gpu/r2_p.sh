timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -k "per_edge" > gpurun_out/r2p_pytest.log 2>&1; echo "edge rc=$?"; tail -25 gpurun_out/r2p_pytest.log
