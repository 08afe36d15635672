# Evidence run: GPU suite, the driver's bench command (both arms), configs 3 and 4, the launch list of
# the default bench command, ncu --set full of k_t3 (configs 5, 3).  Usage: bash tools/gpu/evidence.sh PREFIX
P=${1:-ev}
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/${P}_pytest.log 2>&1; echo "gpu suite rc=$?"; tail -1 gpurun_out/${P}_pytest.log
( time timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/${P}_bench5.json 2> gpurun_out/${P}_bench5.err; echo "bench rc=$?"; tail -3 gpurun_out/${P}_bench5.err
( time timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/${P}_ref5.json 2> gpurun_out/${P}_ref5.err; echo "ref rc=$?"; tail -3 gpurun_out/${P}_ref5.err
timeout 600 python bench.py --config 3 --no-cpu-baseline > gpurun_out/${P}_bench3.json 2>&1; echo "bench3 rc=$?"
timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/${P}_bench4.json 2>&1; echo "bench4 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P}_launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${P}_ncu_launch.log 2>&1; echo "launch list rc=$?"
python tools/step_once.py --config 5 --steps 1 > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_t3 -c 1 -o gpurun_out/${P}_k_t3_c5 python tools/step_once.py --config 5 --steps 1 > gpurun_out/${P}_ncu5.log 2>&1; echo "ncu5 rc=$?"
python tools/step_once.py --config 3 --steps 1 > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_t3 -c 1 -o gpurun_out/${P}_k_t3_c3 python tools/step_once.py --config 3 --steps 1 > gpurun_out/${P}_ncu3.log 2>&1; echo "ncu3 rc=$?"
