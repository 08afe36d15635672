"""Measurement of the rows beyond the bench step:
top-k pairs (route S), the SBESPAR estimate, per-edge counts, BB-Base (Alg. 1) and top-k vertices,
each timed with CUDA events on the library's stream after a warm-up call, on the synthetic
configs (synth/), with the hub kernel's algorithmic bytes per second from bbf_graph_stats against
the measured HBM copy peak.  Parity of every one of these calls is in tests/ (-m gpu); this script
only times them.  Prints one JSON line per measurement.

python tools/next_rows_bench.py [--configs 2 3] [--reps 3]"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[2, 3])
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch
    from paper_2308_07932_b200 import bbf
    from synth import graphs as G

    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    hbm = float(peaks.get("hbm_gbs") or peaks.get("hbm_copy_gbs") or 0.0)
    dev = torch.device("cuda", 0)
    s = torch.cuda.Stream(dev)
    torch.cuda.set_stream(s)

    def timed(fn):
        try:
            fn()  # warm-up (plans, buffers)
        except bbf.BBFError as e:
            return e, None
        torch.cuda.synchronize()
        ms = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            r = fn()
            e1.record(s)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        return r, float(np.median(ms))

    for c in a.configs:
        g = G.make_config(c)
        rp = torch.from_numpy(g.row_ptr.view(np.int64)).to(dev)
        col = torch.from_numpy(g.col.view(np.int32)).to(dev)
        sg = torch.from_numpy(g.sign).to(dev)
        h = bbf.Graph(g.n_u, g.n_v, rp, col, sg, stream=s)
        base = {"config": c, "n_u": g.n_u, "n_v": g.n_v, "nnz": int(g.row_ptr[-1])}

        def hub(st):
            gbs = st["algo_bytes"] / (st["ms_main_kernel"] * 1e6) if st["ms_main_kernel"] > 0 else None
            return {"hub_kernel_ms": round(st["ms_main_kernel"], 4),
                    "hub_kernel_algo_GBps": round(gbs, 1) if gbs else None,
                    "hub_kernel_frac_of_hbm": round(gbs / hbm, 4) if gbs and hbm else None}

        for side in (bbf.BBF_SIDE_U, bbf.BBF_SIDE_V):
            r, ms = timed(lambda: h.count_pairs_topk(100, side=side))
            if ms is None:
                print(json.dumps({**base, "row": "S11 top-k pairs", "error": str(r)}), flush=True)
                continue
            print(json.dumps({**base, "row": "S11 top-k pairs (route S)", "side": "UV"[side], "k": 100,
                              "ms": round(ms, 3), "pairs_returned": len(r), **hub(h.stats())}), flush=True)
        out = (torch.zeros(base["nnz"], dtype=torch.int64, device=dev),
               torch.zeros(base["nnz"], dtype=torch.int64, device=dev))
        r, ms = timed(lambda: h.count_per_edge(rp, col, out=out))
        if ms is not None:
          print(json.dumps({**base, "row": "NEXT-4 per-edge counts (eBBFC semantics)", "ms": round(ms, 3),
                          "edges_per_s": round(base["nnz"] / (ms * 1e-3), 1), **hub(h.stats())}), flush=True)
        r, ms = timed(lambda: h.count_global_base())
        print(json.dumps({**base, "row": "NEXT-4 Alg. 1 BB-Base (global)",
                          **({"ms": round(ms, 3), "balanced": r["balanced"]} if ms is not None else {"error": str(r)})}),
              flush=True)
        r, ms = timed(lambda: h.topk_vertices(100, side=bbf.BBF_SIDE_U))
        if ms is not None:
          print(json.dumps({**base, "row": "NEXT-2 top-k vertices (per-vertex balanced)", "ms": round(ms, 3)}),
              flush=True)
        h.free()
        trials = 4
        r, ms = timed(lambda: bbf.estimate_global(g.n_u, g.n_v, rp, col, sg, 0.5, trials, seed=7, stream=s))
        if ms is not None:
          print(json.dumps({**base, "row": "NEXT-1 SBESPAR estimate (rho 0.5)", "trials": trials,
                          "ms": round(ms, 3), "ms_per_trial": round(ms / trials, 3)}), flush=True)


if __name__ == "__main__":
    main()
