timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b2_a.json 2>&1
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-clocks > gpurun_out/b2_b.json 2>&1
timeout 600 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b2_c.json 2>&1
python - <<'PY'
import json
for c in "abc":
    d=json.load(open(f"gpurun_out/b2_{c}.json")); print(c, d["value"]/1e9, d["ms_per_step"], d["roofline"]["ms_per_launch"], d["clocks"])
PY
