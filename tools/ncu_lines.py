"""Per-CUDA-source-line executed instructions and stall samples from an ncu report.
python tools/ncu_lines.py rep.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, cur = None, None
inst, samp, srcs = collections.defaultdict(float), collections.defaultdict(float), {}
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] == "Function Name":
        continue
    if r[0].strip().isdigit() and hdr:
        cur = (fname, int(r[0]))
        srcs[cur] = r[1]
        try:
            inst[cur] += float(r[hdr.index("Instructions Executed")] or 0)
            samp[cur] += float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except (ValueError, IndexError):
            pass
ti, ts = sum(inst.values()), sum(samp.values())
print(f"total warp inst {ti/1e9:.2f} G, samples {ts:.0f}")
for k, v in sorted(inst.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{v/1e9:6.2f}G {100*v/ti:5.1f}%  smp {100*samp[k]/max(ts,1):5.1f}%  {k[0]}:{k[1]}  {srcs[k][:80]}")
