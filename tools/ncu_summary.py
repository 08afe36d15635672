"""Summarise an ncu --set full report: key throughput metrics, stall reasons, hottest source lines.
python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json]"""
import csv
import io
import json
import subprocess
import sys


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    raw = ncu_csv(rep, "--page", "raw")
    h, v = raw[0], raw[2] if len(raw) > 2 else raw[1]
    d = dict(zip(h, v))
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "smsp__sass_inst_executed_op_global_ld.sum", "smsp__inst_executed_op_shared_atom.sum",
            "lts__t_bytes.sum", "l1tex__t_bytes.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]
    units = dict(zip(h, raw[1])) if len(raw) > 2 else {}
    summary = {k: (d.get(k), units.get(k)) for k in keys if k in d}
    stalls = {k.split("stalled_")[1].split("_per")[0]: float(x) for k, x in d.items()
              if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")
              and x not in ("", "n/a")}
    src = ncu_csv(rep, "--page", "source", "--print-source=cuda,sass")
    cur, hdr, lines = None, None, []
    for r in src:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0].isdigit():
            dd = dict(zip(hdr, r))
            try:
                s = int(dd["Warp Stall Sampling (All Samples)"])
            except Exception:
                continue
            lines.append((s, f"{cur}:{r[0]}", r[1].strip()[:80]))
    tot = sum(x[0] for x in lines) or 1
    hot = [(round(100 * s / tot, 1), loc, code) for s, loc, code in sorted(lines, reverse=True)[:15]]
    res = {"metrics": summary, "stalls_per_issue": dict(sorted(stalls.items(), key=lambda t: -t[1])[:10]),
           "hot_lines_pct_of_samples": hot}
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(res, f, indent=1)
    for k, (val, u) in summary.items():
        print(f"{k:70s} {val} {u or ''}")
    print("stalls:", res["stalls_per_issue"])
    for x in hot:
        print(x)


if __name__ == "__main__":
    main()
