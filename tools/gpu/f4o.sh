# FP4-only dense operands: dense GPU tests, then the config 4 bench and its launch list
timeout 900 python -m pytest tests -m gpu -x -q  2>&1 | tail -3
timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/f4o_bench4.json 2>gpurun_out/f4o_bench4.err; tail -c 1500 gpurun_out/f4o_bench4.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/f4o_launches4.csv \
  python tools/step_once.py --config 4 --steps 1 --path dense > gpurun_out/f4o_ncu.log 2>&1; python tools/launch_summary.py gpurun_out/f4o_launches4.csv
