"""Projected N-GPU strong scaling of the count from single-GPU shard runs (BBF_FAKE_WORLD=r/N: rank
r's shard of the work items counted alone on one GPU, exactly the kernels an N-GPU run launches on
rank r, without the NCCL all-reduce).  For N in {1,2,4,8}: per-rank device time of the count call
(plan + kernels; bbf_counts.ms_count) and of the hub kernel; the projected count time is the max
over ranks plus an all-reduce estimate (16 bytes per row of degree >= 2 — the rows the library
reduces — at the given NVLink all-reduce bandwidth).

    python tools/fakeworld_scaling.py --config 5 [--steps 3] [--allreduce-gbs 400]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--allreduce-gbs", type=float, default=400.0,
                    help="assumed NCCL u64 all-reduce bus bandwidth over NVLink 5 (GB/s)")
    a = ap.parse_args()
    import torch
    from paper_2308_07932_b200 import bbf
    from synth import graphs as G
    g = G.make_config(a.config)
    dev = torch.device("cuda", 0)
    rp = torch.from_numpy(g.row_ptr.view(np.int64)).to(dev)
    col = torch.from_numpy(g.col.view(np.int32)).to(dev)
    sg = torch.from_numpy(g.sign).to(dev)
    outs = tuple(torch.zeros(k, dtype=torch.int64, device=dev) for k in (g.n_u, g.n_u, g.n_v, g.n_v))
    st = torch.cuda.Stream(dev)
    torch.cuda.set_stream(st)
    # the per-vertex all-reduce covers the rows of degree >= 2 only (api.cu finish_collective)
    du = np.diff(g.row_ptr.astype(np.int64))
    dv = np.bincount(g.col, minlength=g.n_v)
    res = {"config": a.config, "n": g.n_u + g.n_v, "rows_reduced": int((du >= 2).sum() + (dv >= 2).sum()),
           "ranks": {}}
    with bbf.Graph(g.n_u, g.n_v, rp, col, sg, stream=st) as h:  # built once; the count is what is sharded
        for N in (1, 2, 4, 8):
            per = []
            for r in range(N):
                if N > 1:
                    os.environ["BBF_FAKE_WORLD"] = f"{r}/{N}"
                else:
                    os.environ.pop("BBF_FAKE_WORLD", None)
                cms, kms = [], []
                for _ in range(a.steps + 1):
                    tot = h.count_per_vertex(out=outs)[0]
                    cms.append(tot["ms_count"])
                    kms.append(h.stats()["ms_main_kernel"])
                per.append({"rank": r, "ms_count": float(np.median(cms[1:])), "ms_t3": float(np.median(kms[1:])),
                            "balanced": int(tot["balanced"])})
            os.environ.pop("BBF_FAKE_WORLD", None)
            ar_ms = 0.0 if N == 1 else 16.0 * res["rows_reduced"] * 2 * (N - 1) / N / (a.allreduce_gbs * 1e9) * 1e3
            res["ranks"][N] = {"per_rank": per, "max_ms_count": max(p["ms_count"] for p in per),
                               "allreduce_ms_est": ar_ms}
    t1 = res["ranks"][1]["max_ms_count"]
    for N, v in res["ranks"].items():
        tN = v["max_ms_count"] + v["allreduce_ms_est"]
        v["projected_ms"] = tN
        v["projected_efficiency"] = t1 / (N * tN)
        print(f"N={N}: max rank count {v['max_ms_count']:.2f} ms (+ all-reduce ~{v['allreduce_ms_est']:.2f}) "
              f"-> efficiency {v['projected_efficiency']:.3f}; per rank "
              + " ".join(f"{p['ms_count']:.1f}" for p in v["per_rank"]), flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
