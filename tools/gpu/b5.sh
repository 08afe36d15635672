timeout 900 python bench.py > gpurun_out/b5_bench5.json 2> gpurun_out/b5_bench5.err
for c in 3 4; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/b5_bench$c.json 2> gpurun_out/b5_bench$c.err; done
python - <<'PY'
import json
for c in (5,3,4):
    try:
        d=json.load(open(f"gpurun_out/b5_bench{c}.json")); r=d["roofline"]
        print(c, round(d["value"]/1e9,1), round(d["ms_per_step"],2), "e2e", round(d["e2e"]["value"]/1e9,1), r["bound"], round(r["achieved"],1), r["unit"], round(r["frac"],3), round(r["ms_per_launch"],2), d["clocks"], d.get("cpu_baseline",{}).get("value"))
    except Exception as e: print(c, "ERR", e, open(f"gpurun_out/b5_bench{c}.err").read()[-800:])
PY
