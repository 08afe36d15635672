timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b1_bench5.json 2> gpurun_out/b1_bench5.err
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b1_bench3.json 2> gpurun_out/b1_bench3.err
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b1_bench4.json 2> gpurun_out/b1_bench4.err
python - <<'PY'
import json
for c in (5,3,4):
    try:
        d=json.load(open(f"gpurun_out/b1_bench{c}.json")); print(c, d["value"]/1e9, d["ms_per_step"], d["e2e"]["ms_per_step"], d["roofline"]["ms_per_launch"], d["roofline"]["frac"])
    except Exception as e: print(c, "ERR", e, open(f"gpurun_out/b1_bench{c}.err").read()[-500:])
PY
