"""Write tests/golden/expected_counts.json: the oracle's counts for the five BASELINE configs and
the NEXT-3 hybrid workload (synth.graphs.config_hybrid, "config 6").

Calls only oracle/ (Alg. 2 + 4-role scatter, oracle_route_g_pv) and synth/ (the seeded input
generators).  Nothing here reads the CUDA path.  bench.py asserts its counts against this file
before it prints a throughput number, and tests/test_gpu_parity.py compares against the oracle
directly.  Per config: the graph's SHA-256 (synth.graphs.SignedBipartite.sha256), B, N, W_G and
the SHA-256 of the per-vertex arrays (bal_u, unb_u, bal_v, unb_v as little-endian uint64,
concatenated in that order).

    python tests/scripts/write_expected.py [configs...]      (default: 1 2 3 4 5 6)
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from synth import graphs  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "expected_counts.json")


def pv_sha256(bal_u, unb_u, bal_v, unb_v) -> str:
    h = hashlib.sha256()
    for a in (bal_u, unb_u, bal_v, unb_v):
        h.update(np.ascontiguousarray(a, dtype="<u8").tobytes())
    return h.hexdigest()


def main(cfgs):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for c in cfgs:
        t0 = time.time()
        g = graphs.make_config(c)
        r = oracle.route_g_pv(g)
        data[f"config{c}"] = dict(
            graph_sha256=g.sha256(), n_u=g.n_u, n_v=g.n_v, nnz=g.nnz,
            B=r["B"], N=r["N"], W_G=r["W_G"],
            pv_sha256=pv_sha256(r["bal_u"], r["unb_u"], r["bal_v"], r["unb_v"]),
            oracle="oracle_route_g_pv (Alg. 2 + 4-role scatter)",
            oracle_threads=os.cpu_count(), oracle_count_s=round(r["count_s"], 3))
        print(c, data[f"config{c}"], f"{time.time() - t0:.1f} s", flush=True)
        json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5, 6])
