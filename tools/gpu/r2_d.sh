bash tools/gpu/ab.sh "base0 default"
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -k "full_per_vertex and (config3 or config5 or zoned)" > gpurun_out/r2d_pytest.log 2>&1; echo "fullsize rc=$?"; tail -3 gpurun_out/r2d_pytest.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep or zoned or kmn or schedule" > gpurun_out/r2d_pytest2.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/r2d_pytest2.log
