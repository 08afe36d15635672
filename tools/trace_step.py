"""Timeline of one bench step (torch.profiler / CUPTI): kernels, memcpy/memset and the idle gaps
between them on the library's stream.  python tools/trace_step.py --config 5"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--out", default="gpurun_out/trace.json")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--e2e", action="store_true", help="trace the pipelined host-buffer loop (bench e2e)")
    a = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile
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

    def step():
        h = bbf.Graph(g.n_u, g.n_v, rp, col, sg, stream=s)
        h.count_per_vertex(out=outs)
        h.free()

    if a.e2e:  # bench.py's e2e loop: uploads one step ahead, asynchronous outputs
        pin = [torch.from_numpy(x).pin_memory() for x in (g.row_ptr.view(np.int64), g.col.view(np.int32), g.sign)]
        hout = tuple(torch.zeros(k, dtype=torch.int64).pin_memory() for k in (g.n_u, g.n_u, g.n_v, g.n_v))
        state = {"up": None}

        def step():
            up = state["up"] or bbf.Upload(g.n_u, g.n_v, *pin)
            h = bbf.Graph.from_upload(up, stream=s)
            state["up"] = bbf.Upload(g.n_u, g.n_v, *pin)
            h.count_per_vertex(out=hout, flags=bbf.BBF_OUTPUT_ASYNC)
            h.free()

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(a.steps):
            step()
        if a.e2e:
            bbf.device_sync(0)
        torch.cuda.synchronize()
    prof.export_chrome_trace(a.out)
    ev = json.load(open(a.out))["traceEvents"]
    gpu = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")],
                 key=lambda e: e["ts"])
    t0 = gpu[0]["ts"]
    tend = max(e["ts"] + e.get("dur", 0) for e in gpu)
    busy = sum(e.get("dur", 0) for e in gpu)
    print(f"span {1e-3*(tend-t0):.2f} ms, busy {1e-3*busy:.2f} ms, {len(gpu)} gpu ops")
    prev = t0
    gaps = []
    for e in gpu:
        gap = e["ts"] - prev
        gaps.append((gap, e["name"][:70]))
        prev = max(prev, e["ts"] + e.get("dur", 0))
    gaps.sort(reverse=True)
    print("largest idle gaps before op (ms):")
    for gp, nm in gaps[:25]:
        print(f"  {1e-3*gp:8.3f}  {nm}")
    agg = {}
    for e in gpu:
        agg.setdefault(e["name"][:70], [0, 0.0])
        agg[e["name"][:70]][0] += 1
        agg[e["name"][:70]][1] += e.get("dur", 0)
    print("busy by op (ms):")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
        print(f"  {1e-3*v[1]:8.3f} x{v[0]:3d}  {k}")
    if a.e2e:
        print("copies (start ms, dur ms, stream, name):")
        for e in gpu:
            if e.get("cat") == "gpu_memcpy" and e.get("dur", 0) > 200:
                print(f"  {1e-3*(e['ts']-t0):8.2f} {1e-3*e['dur']:7.2f}  s{e.get('args', {}).get('stream')}  {e['name']}")
        w0, w1 = float(os.environ.get("TR_W0", "84")), float(os.environ.get("TR_W1", "101"))
        print(f"all ops in [{w0}, {w1}] ms:")
        for e in gpu:
            t = 1e-3 * (e["ts"] - t0)
            if w0 <= t <= w1:
                print(f"  {t:8.3f} {1e-3*e.get('dur',0):7.3f}  s{e.get('args', {}).get('stream')}  {e['name'][:60]}")
        for e in gpu:
            if e.get("cat") == "kernel" and ("k_t3" in e["name"] or "k_hist_v" in e["name"]):
                print(f"  {1e-3*(e['ts']-t0):8.2f} {1e-3*e['dur']:7.2f}  s{e.get('args', {}).get('stream')}  {e['name'][:40]}")
    cpu = sorted([e for e in ev if e.get("cat") == "cuda_runtime" or e.get("cat") == "cuda_driver"],
                 key=lambda e: -e.get("dur", 0))
    print("longest runtime API calls (ms):")
    for e in cpu[:15]:
        print(f"  {1e-3*e.get('dur',0):8.3f}  {e['name']}  at +{1e-3*(e['ts']-t0):.1f} ms")


if __name__ == "__main__":
    main()
