timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep or zoned or kmn or schedule or encodings or packing or config2 or corpus" > gpurun_out/r2k_pytest2.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/r2k_pytest2.log
bash tools/gpu/ab.sh "base0 default"
bash tools/gpu/r2_j.sh
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -k "full_per_vertex and (config3 or config5 or zoned)" > gpurun_out/r2k_pytest.log 2>&1; echo "fullsize rc=$?"; tail -3 gpurun_out/r2k_pytest.log
