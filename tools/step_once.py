"""One hot-path step (device CSR -> build/plan -> per-vertex count -> free) for profiling.
python tools/step_once.py --config 3 [--steps 1] [--global-only]"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--global-only", action="store_true")
    ap.add_argument("--path", choices=["auto", "dense", "sparse"], default="auto")
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
    s = torch.cuda.Stream(dev)
    torch.cuda.set_stream(s)
    torch.cuda.synchronize()
    for _ in range(a.steps):
        t0 = time.perf_counter()
        fl = {"auto": 0, "dense": bbf.BBF_FORCE_DENSE, "sparse": bbf.BBF_FORCE_SPARSE}[a.path]
        h = bbf.Graph(g.n_u, g.n_v, rp, col, sg, stream=s, flags=fl)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        r = h.count_global() if a.global_only else h.count_per_vertex(out=outs)[0]
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        st = h.stats()
        h.free()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        print(f"load {1e3*(t1-t0):.1f} ms  count {1e3*(t2-t1):.1f} ms (device {r['ms_count']:.1f}, main {st['ms_main_kernel']:.1f})  free {1e3*(t3-t2):.1f} ms", r, flush=True)


if __name__ == "__main__":
    main()
