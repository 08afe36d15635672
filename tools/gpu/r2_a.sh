# Round 2, first box call: full-size parity tests, default bench (parity gate + full oracle
# baseline), and the hub-kernel phase split / chunk statistics of the profiling variant.
nproc > gpurun_out/r2a_host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/r2a_host.txt; free -g >> gpurun_out/r2a_host.txt
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/r2a_pytest_full.log 2>&1; echo "fullsize rc=$?"
tail -3 gpurun_out/r2a_pytest_full.log
( time timeout 900 python bench.py ) > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/r2a_bench.err
for c in 5 3; do BBF_LIB=paper_2308_07932_b200/_build_prof/libbbf.so BBF_DEBUG=1 timeout 300 python tools/step_once.py --config $c --steps 2 2>&1 | grep -E "engine|phases|CTA ends" | tail -3; done
