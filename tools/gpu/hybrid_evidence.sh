# Evidence run for the hybrid path and the default bench: smoke(), GPU suite, the driver's bench
# command (both arms), bench config 6 (hybrid) and its sparse-only twin, the launch list of one
# config-6 step, ncu --set full of the fused cross-term kernel k_dense_f4q<true>.
# Usage: bash tools/gpu/hybrid_evidence.sh PREFIX
P=${1:-hy}
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${P}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${P}_smoke.log
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/${P}_pytest.log 2>&1; echo "gpu suite rc=$?"; tail -1 gpurun_out/${P}_pytest.log
( time timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/${P}_bench5.json 2> gpurun_out/${P}_bench5.err; echo "bench rc=$?"; tail -3 gpurun_out/${P}_bench5.err
( time timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/${P}_ref5.json 2> gpurun_out/${P}_ref5.err; echo "ref rc=$?"
timeout 600 python bench.py --config 3 --no-cpu-baseline > gpurun_out/${P}_bench3.json 2>&1; echo "bench3 rc=$?"
timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/${P}_bench4.json 2>&1; echo "bench4 rc=$?"
timeout 900 python bench.py --config 6 > gpurun_out/${P}_bench6.json 2> gpurun_out/${P}_bench6.err; echo "bench6 rc=$?"
BBF_NO_HYBRID=1 timeout 900 python bench.py --config 6 --no-cpu-baseline > gpurun_out/${P}_bench6_sparse.json 2> gpurun_out/${P}_bench6_sparse.err; echo "bench6 sparse rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P}_launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1; echo "launch list c5 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P}_launches_c6.csv python tools/step_once.py --config 6 --steps 2 > gpurun_out/${P}_ncu_launch6.log 2>&1; echo "launch list rc=$?"
python tools/step_once.py --config 6 --steps 1 > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dense_f4q --launch-skip 2 -c 1 -o gpurun_out/${P}_f4q_cross_c6 python tools/step_once.py --config 6 --steps 1 > gpurun_out/${P}_ncu_cross.log 2>&1; echo "ncu cross rc=$?"
