"""Tensor-pipe evidence of the dense-path kernels from their ncu --set full captures: tensor-pipe
utilisation counters, the FP4 / int8 tensor op counts against the per-SM peak ncu reports, DRAM
traffic, and an executed-SASS opcode histogram (UTC*MMA = tcgen05.mma, UTMALDG = TMA tensor
load, LDTM = tcgen05.ld, UTCCP = tcgen05.cp).

    python tools/ncu_dense_summary.py out.json rep1.ncu-rep [rep2.ncu-rep ...]
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys

KEYS = ("gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_op_utcomma_src_fp4_dst_fp32_sparsity_off.sum",
        "sm__ops_path_tensor_op_utcomma_src_fp4_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
        "sm__ops_path_tensor_op_utcomma_src_fp4_dst_fp32_sparsity_off.avg.peak_sustained",
        "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.sum",
        "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.sum.pct_of_peak_sustained_elapsed",
        "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.avg.peak_sustained",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "smsp__sass_inst_executed_op_utcmma.sum", "smsp__sass_inst_executed_op_tmem_ldt.sum",
        "smsp__sass_inst_executed_op_utccp.sum", "sm__cycles_elapsed.avg.per_second")


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def summary(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, u, v = rows[0], rows[1], rows[2]
    out = {"kernel": v[h.index("Kernel Name")], "metrics": {}}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            out["metrics"][k] = [v[i], u[i]]
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    hdr, data = src[1], src[2:]
    ie = hdr.index("Instructions Executed")
    hist = collections.Counter()
    for r in data:
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[1])
        if m and r[ie].isdigit():
            hist[m.group(2)] += int(r[ie])
    keep = ("UTCOMMA", "UTCIMMA", "UTCQMMA", "UTCHMMA", "UTMALDG", "UTMACCTL", "LDTM", "STTM", "UTCCP", "UTCBAR")
    out["sass_executed"] = {k: hist[k] for k in sorted(hist) if k.startswith(keep)}
    out["sass_executed_total"] = sum(hist.values())
    return out


if __name__ == "__main__":
    res = [summary(r) for r in sys.argv[2:]]
    json.dump(res, open(sys.argv[1], "w"), indent=1)
    for r in res:
        print(r["kernel"][:60], r["sass_executed"])
