bash tools/gpu/ab.sh "base0 default"
for v in prof; do for c in 5 3; do echo "== $v c$c"; BBF_LIB=paper_2308_07932_b200/_build_$v/libbbf.so BBF_DEBUG=1 timeout 300 python tools/step_once.py --config $c --steps 1 2>&1 | grep -E "phases" | tail -1; done; done
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -k "full_per_vertex and (config3 or config5 or zoned)" > gpurun_out/r2g_pytest.log 2>&1; echo "fullsize rc=$?"; tail -3 gpurun_out/r2g_pytest.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep or zoned or kmn or schedule or encodings or packing" > gpurun_out/r2g_pytest2.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/r2g_pytest2.log
