"""The paper's BB-Base vs BB-Bucket regime on the GPU: Senate-shaped
synthetic graphs (few dense left vertices, many right ones, density 0.5, signs 50/50 — the
shape of the paper's Senate/House roll-call graphs; seeded, synthetic), counted by Alg. 1
(bbf_count_global_base) and Alg. 2 (bbf_count_global, sparse path) through the C ABI; device
time per call (median of --reps), counts checked equal.  The smallest shape is also timed on
the oracle (both algorithms, one host thread) for the CPU regime.
python tests/scripts/base_vs_bucket.py [--json profiles/r1_base_vs_bucket.json]"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    from paper_2308_07932_b200 import bbf
    from synth import graphs as G
    import oracle as O
    rows = []
    for (nl, nr) in ((10, 1000), (50, 20000), (100, 100000)):
        g = G.random_bipartite(nl, nr, 0.5, 0.5, seed=nl)
        with bbf.Graph.from_synth(g, flags=bbf.BBF_FORCE_SPARSE) as h:
            h.count_global(); h.count_global_base()  # warm-up (plan, scratch)
            tb, tk, rb, rk = [], [], None, None
            for _ in range(a.reps):
                rb = h.count_global_base(); tb.append(rb["ms_count"])
                rk = h.count_global(); tk.append(rk["ms_count"])
        assert (rb["balanced"], rb["unbalanced"]) == (rk["balanced"], rk["unbalanced"])
        r = dict(shape=f"{nl} x {nr}, density 0.5, p+ 0.5", edges=int(g.col.size),
                 wedges_G=rk["wedges_G"], butterflies=rk["total"],
                 gpu_base_ms=float(np.median(tb)), gpu_bucket_ms=float(np.median(tk)))
        r["gpu_speedup"] = r["gpu_base_ms"] / r["gpu_bucket_ms"]
        if nl == 10:
            ob, og = O.bb_base(g, threads=1), O.route_g(g, threads=1)
            assert (ob["B"], ob["N"]) == (rb["balanced"], rb["unbalanced"])
            r["oracle_base_ms_1thread"] = ob["count_s"] * 1e3
            r["oracle_bucket_ms_1thread"] = og["count_s"] * 1e3
        rows.append(r)
        print(json.dumps(r), flush=True)
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"what": __doc__.split("\n")[0], "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
