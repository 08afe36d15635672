"""Time the hybrid dense-core path against the plain sparse engine on the hybrid workload
(synth.graphs.config_hybrid) or a BASELINE config: count_global / count_per_vertex, automatic
dispatch vs BBF_NO_HYBRID vs forced cores.  Synchronous library calls timed on the host after
warm-up (each call ends with a stream synchronize); one JSON line per case."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_07932_b200 import bbf as B  # noqa: E402
from synth import graphs as G  # noqa: E402


def timed(h, pv, reps):
    f = h.count_per_vertex if pv else h.count_global
    f()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        r = f()
        ts.append(time.perf_counter() - t)
    c = r[0] if pv else r
    return min(ts) * 1e3, c["balanced"], c["unbalanced"], c["wedges_G"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="hybrid")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cores", default="", help="forced cores 'a,b;c,d'")
    a = ap.parse_args()
    g = G.config_hybrid() if a.config == "hybrid" else G.make_config(int(a.config))
    cases = [("auto", {}), ("sparse", {"BBF_NO_HYBRID": "1"})]
    for c in filter(None, a.cores.split(";")):
        cases.append((f"core{c}", {"BBF_HYBRID_CORE": c}))
    with B.Graph.from_synth(g) as h:
        for name, env in cases:
            for pv in (False, True):
                for k, v in env.items():
                    os.environ[k] = v
                ms, b, n, w = timed(h, pv, a.reps)
                core = h.hybrid_core()
                for k in env:
                    del os.environ[k]
                print(json.dumps(dict(config=a.config, case=name, per_vertex=pv, ms=round(ms, 3), B=b, N=n,
                                      W_G=w, core=core, gwedges_per_s=round(w / ms / 1e6, 1))), flush=True)


if __name__ == "__main__":
    main()
