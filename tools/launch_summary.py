"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel name the
launch count, total ms and share of all launches, the library's (bbf::) kernels separated from
the bench's own set-up kernels (torch / synthetic-input generation).
python tools/launch_summary.py profiles/r1_launches_c5_v9.csv [--json out.json] [--source "..."]"""
import argparse
import csv
import io
import json
from collections import defaultdict


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--json")
    ap.add_argument("--source", default="")
    a = ap.parse_args()
    lines = [ln for ln in open(a.csv) if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"].replace(",", ""))
        name = r["Kernel Name"]
        agg[name][0] += 1
        agg[name][1] += ns * 1e-6
    lib = {k: v for k, v in agg.items() if "bbf::" in k or "CUB_" in k}
    tot_lib = sum(v[1] for v in lib.values())
    out = {"source": a.source, "launches": sum(v[0] for v in agg.values()),
           "library_launches": sum(v[0] for v in lib.values()), "library_ms": round(tot_lib, 3),
           "kernels": [{"name": k[:140], "launches": v[0], "ms": round(v[1], 3),
                        "share_of_library": round(v[1] / tot_lib, 4) if tot_lib else None}
                       for k, v in sorted(lib.items(), key=lambda kv: -kv[1][1])]}
    for k in out["kernels"][:12]:
        print(f'{k["ms"]:9.3f} ms {k["launches"]:4d}x {k["share_of_library"]:.4f}  {k["name"][:90]}')
    if a.json:
        with open(a.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
