"""ctypes wrapper of oracle/bbf_oracle.c (plain C, pthreads) — TEST INFRASTRUCTURE ONLY.

Each function takes a `synth.graphs.SignedBipartite` (U-side CSR, 1 = positive edge) and
returns plain numpy / int results.  See bbf_oracle.c's header for which paper passage each
routine follows.  Parity unpinned: none (every routine is pinned in tests/test_oracle_pins.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bbf_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_ERR = {1: "EINVAL", 2: "ERANGE", 3: "EDUP", 4: "ENOMEM", 7: "EOVERFLOW", 8: "ESMALL"}


class OracleError(RuntimeError):
    def __init__(self, rc: int):
        super().__init__(f"oracle rc={rc} ({_ERR.get(rc, '?')})")
        self.rc = rc
        self.name = _ERR.get(rc, "?")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C11, -O2, pthreads)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-shared", "-fPIC", "-pthread",
                               "-o", _LIB, _SRC])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(_LIB)
        P = C.c_void_p
        u32, u64, i32 = C.c_uint32, C.c_uint64, C.c_int
        lib.oracle_brute.argtypes = [u32, u32, P, P, P, P, P, P, P, P, P]
        lib.oracle_route_g.argtypes = [u32, u32, P, P, P, P, u64, i32, P]
        lib.oracle_route_s.argtypes = [u32, u32, P, P, P, P, u64, i32, P, P]
        lib.oracle_route_g_pv.argtypes = [u32, u32, P, P, P, P, u64, i32, P, P, P]
        lib.oracle_route_g_pv.restype = i32
        lib.oracle_prepare.argtypes = [u32, u32, P, P, P, P]
        lib.oracle_prepare.restype = P
        lib.oracle_release.argtypes = [P]
        lib.oracle_release.restype = None
        lib.oracle_route_g_pv_h.argtypes = [P, P, u64, i32, P, P, P]
        lib.oracle_route_g_pv_h.restype = i32
        lib.oracle_edge_brute.argtypes = [u32, u32, P, P, P, P, P]
        lib.oracle_edge_brute.restype = i32
        lib.oracle_edge.argtypes = [u32, u32, P, P, P, i32, P, P]
        lib.oracle_edge.restype = i32
        lib.oracle_bb_base.argtypes = [u32, u32, P, P, P, i32, P]
        lib.oracle_bb_base.restype = i32
        lib.oracle_pairs.argtypes = [u32, u32, P, P, P, i32, i32, P, P, P, P, u64, P]
        lib.oracle_priority_order.argtypes = [u32, u32, P, P, P, P]
        lib.oracle_sm64.argtypes = [u64]
        lib.oracle_sm64.restype = u64
        lib.oracle_sparsify.argtypes = [u32, P, P, P, C.c_double, u64, u32, P, P, P, P]
        lib.oracle_sparsify.restype = i32
        for f in (lib.oracle_brute, lib.oracle_route_g, lib.oracle_route_s, lib.oracle_pairs,
                  lib.oracle_priority_order):
            f.restype = i32
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _graph_args(g):
    rp = np.ascontiguousarray(g.row_ptr, dtype=np.uint64)
    col = np.ascontiguousarray(g.col, dtype=np.uint32)
    sg = np.ascontiguousarray(g.sign, dtype=np.uint8)
    # keep the arrays alive alongside the pointers
    return (rp, col, sg), (C.c_uint32(g.n_u), C.c_uint32(g.n_v), _ptr(rp), _ptr(col), _ptr(sg))


def _threads(t):
    return int(t) if t else (os.cpu_count() or 1)


def brute(g, pairs: bool = False):
    """Definition-level count over all 4-tuples.  Returns dict with B, N, per-vertex arrays
    (bal_u, unb_u, bal_v, unb_v) and, if pairs, the n_u x n_u upper-triangular pair matrix."""
    lib = _load()
    keep, a = _graph_args(g)
    out = np.zeros(2, np.uint64)
    bu, nu = np.zeros(g.n_u, np.uint64), np.zeros(g.n_u, np.uint64)
    bv, nv = np.zeros(g.n_v, np.uint64), np.zeros(g.n_v, np.uint64)
    pm = np.zeros((g.n_u, g.n_u), np.uint64) if pairs else None
    rc = lib.oracle_brute(*a, _ptr(out), _ptr(bu), _ptr(nu), _ptr(bv), _ptr(nv), _ptr(pm))
    if rc:
        raise OracleError(rc)
    r = dict(B=int(out[0]), N=int(out[1]), bal_u=bu, unb_u=nu, bal_v=bv, unb_v=nv)
    if pairs:
        r["pairs_u"] = pm
    return r


def route_g(g, starts=None, threads=None):
    """Alg. 2 BB-Bucket / ParBB-Bucket.  starts: optional global ids (U: u, V: n_u + v).
    Returns dict(B, N, W_G)."""
    lib = _load()
    keep, a = _graph_args(g)
    st = None if starts is None else np.ascontiguousarray(starts, dtype=np.uint32)
    out = np.zeros(4, np.uint64)
    rc = lib.oracle_route_g(*a, _ptr(st), C.c_uint64(0 if st is None else st.size),
                            _threads(threads), _ptr(out))
    if rc:
        raise OracleError(rc)
    return dict(B=int(out[0]), N=int(out[1]), W_G=int(out[2]), count_s=float(out[3]) * 1e-9)


def route_g_pv(g, threads=None, starts=None):
    """Alg. 2 BB-Bucket plus the 4-role scatter (bbf_oracle.c oracle_route_g_pv): global counts
    and the per-vertex arrays of both sides.  starts: optional global ids (the butterflies
    counted at those starts only).  Returns dict(B, N, W_G, count_s, bal_u, unb_u, bal_v,
    unb_v)."""
    lib = _load()
    keep, a = _graph_args(g)
    out = np.zeros(4, np.uint64)
    n = g.n_u + g.n_v
    bal, unb = np.zeros(n, np.uint64), np.zeros(n, np.uint64)
    st = None if starts is None else np.ascontiguousarray(starts, dtype=np.uint32)
    rc = lib.oracle_route_g_pv(*a, _ptr(st), C.c_uint64(0 if st is None else st.size),
                               _threads(threads), _ptr(out), _ptr(bal), _ptr(unb))
    if rc:
        raise OracleError(rc)
    return dict(B=int(out[0]), N=int(out[1]), W_G=int(out[2]), count_s=float(out[3]) * 1e-9,
                bal_u=bal[:g.n_u], unb_u=unb[:g.n_u], bal_v=bal[g.n_u:], unb_v=unb[g.n_u:])


class Prepared:
    """A graph preprocessed once (Alg. 2 lines 2-3: adjacency built, validated, sorted by
    priority) for repeated route-G counts over start subsets."""

    def __init__(self, g):
        lib = _load()
        self._keep, a = _graph_args(g)
        rc = C.c_int(0)
        self.h = lib.oracle_prepare(*a, C.byref(rc))
        if not self.h:
            raise OracleError(rc.value)
        self.n_u, self.n_v = g.n_u, g.n_v

    def route_g_pv(self, starts=None, threads=None):
        lib = _load()
        out = np.zeros(4, np.uint64)
        n = self.n_u + self.n_v
        bal, unb = np.zeros(n, np.uint64), np.zeros(n, np.uint64)
        st = None if starts is None else np.ascontiguousarray(starts, dtype=np.uint32)
        rc = lib.oracle_route_g_pv_h(C.c_void_p(self.h), _ptr(st), C.c_uint64(0 if st is None else st.size),
                                     _threads(threads), _ptr(out), _ptr(bal), _ptr(unb))
        if rc:
            raise OracleError(rc)
        return dict(B=int(out[0]), N=int(out[1]), W_G=int(out[2]), count_s=float(out[3]) * 1e-9,
                    bal_u=bal[:self.n_u], unb_u=unb[:self.n_u], bal_v=bal[self.n_u:], unb_v=unb[self.n_u:])

    def close(self):
        if self.h:
            _load().oracle_release(C.c_void_p(self.h))
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def edge_brute(g):
    """Per-edge (balanced, unbalanced) counts by brute force over 4-tuples, input CSR order."""
    lib = _load()
    keep, a = _graph_args(g)
    bal, unb = np.zeros(max(g.nnz, 1), np.uint64), np.zeros(max(g.nnz, 1), np.uint64)
    rc = lib.oracle_edge_brute(*a, _ptr(bal), _ptr(unb))
    if rc:
        raise OracleError(rc)
    return bal[:g.nnz], unb[:g.nnz]


def edge_counts(g, threads=None):
    """Per-edge (balanced, unbalanced) counts by the definition, edge by edge,
    input CSR order."""
    lib = _load()
    keep, a = _graph_args(g)
    bal, unb = np.zeros(max(g.nnz, 1), np.uint64), np.zeros(max(g.nnz, 1), np.uint64)
    rc = lib.oracle_edge(*a, _threads(threads), _ptr(bal), _ptr(unb))
    if rc:
        raise OracleError(rc)
    return bal[:g.nnz], unb[:g.nnz]


def bb_base(g, threads=None):
    """Alg. 1 BB-Base: explicit balance check of every pair in each H(w).
    Returns dict(B, N, W_G, count_s)."""
    lib = _load()
    keep, a = _graph_args(g)
    out = np.zeros(4, np.uint64)
    rc = lib.oracle_bb_base(*a, _threads(threads), _ptr(out))
    if rc:
        raise OracleError(rc)
    return dict(B=int(out[0]), N=int(out[1]), W_G=int(out[2]), count_s=float(out[3]) * 1e-9)


def route_s(g, verts=None, threads=None):
    """vBBFC per vertex.  verts: optional global ids (default all n_u + n_v).
    Returns (bal, unb) uint64 arrays aligned with verts."""
    lib = _load()
    keep, a = _graph_args(g)
    vs = None if verts is None else np.ascontiguousarray(verts, dtype=np.uint32)
    cnt = g.n_u + g.n_v if vs is None else vs.size
    bal, unb = np.zeros(cnt, np.uint64), np.zeros(cnt, np.uint64)
    rc = lib.oracle_route_s(*a, _ptr(vs), C.c_uint64(0 if vs is None else vs.size),
                            _threads(threads), _ptr(bal), _ptr(unb))
    if rc:
        raise OracleError(rc)
    return bal, unb


def pairs(g, side: int = 0, threads=None, cap: int | None = None):
    """Every same-side pair {z<y} (side-local ids) with a positive balanced count (Lemma 2).
    Returns (z, y, bal, unb) arrays, unsorted."""
    lib = _load()
    keep, a = _graph_args(g)
    cap = cap or max(1024, 4 * g.nnz)
    while True:
        pz, py = np.zeros(cap, np.uint32), np.zeros(cap, np.uint32)
        pb, pn = np.zeros(cap, np.uint64), np.zeros(cap, np.uint64)
        n = np.zeros(1, np.uint64)
        rc = lib.oracle_pairs(*a, int(side), _threads(threads), _ptr(pz), _ptr(py), _ptr(pb),
                              _ptr(pn), C.c_uint64(cap), _ptr(n))
        if rc == 8:
            cap = int(n[0]) + 16
            continue
        if rc:
            raise OracleError(rc)
        k = int(n[0])
        return pz[:k], py[:k], pb[:k], pn[:k]


def topk_pairs(g, k: int, side: int = 0, threads=None):
    """Top-k same-side pairs by balanced count (reading R11): order by balanced desc,
    then smaller id asc, then larger id asc; zero-score pairs excluded.
    Returns a list of (a, b, balanced, unbalanced) with a < b."""
    z, y, b, n = pairs(g, side, threads)
    order = np.lexsort((y, z, -b.astype(np.float64)))  # primary key last
    # exact tie-break on the uint64 score (float key above only pre-sorts)
    idx = sorted(order.tolist(), key=lambda i: (-int(b[i]), int(z[i]), int(y[i])))
    return [(int(z[i]), int(y[i]), int(b[i]), int(n[i])) for i in idx[:k]]


def priority_order(g):
    """Position of every global id in descending Def.-Vertex-Priority order (0 = highest)."""
    lib = _load()
    keep, a = _graph_args(g)
    pos = np.zeros(g.n_u + g.n_v, np.uint32)
    rc = lib.oracle_priority_order(*a, _ptr(pos))
    if rc:
        raise OracleError(rc)
    return pos


def sm64(x: int) -> int:
    """The generator of the sparsification draws (SplitMix64 output for state x)."""
    return int(_load().oracle_sm64(C.c_uint64(x & (2**64 - 1))))


def sparsify(g, rho: float, seed: int, trial: int = 0):
    """SBESPAR sample: each edge kept independently w.p. rho (documented
    counter-based draws, see bbf_oracle.c).  Returns a synth.graphs.SignedBipartite."""
    from synth.graphs import SignedBipartite
    lib = _load()
    keep, a = _graph_args(g)
    rp = np.zeros(g.n_u + 1, np.uint64)
    col = np.zeros(max(g.nnz, 1), np.uint32)
    sg = np.zeros(max(g.nnz, 1), np.uint8)
    k = np.zeros(1, np.uint64)
    rc = lib.oracle_sparsify(a[0], a[2], a[3], a[4], C.c_double(rho), C.c_uint64(seed),
                             C.c_uint32(trial), _ptr(rp), _ptr(col), _ptr(sg), _ptr(k))
    if rc:
        raise OracleError(rc)
    m = int(k[0])
    return SignedBipartite(g.n_u, g.n_v, rp, col[:m].copy(), sg[:m].copy())


def estimate(g, rho: float, trials: int, seed: int = 0, threads=None):
    """SBESPAR estimate of the global balanced count: per trial, the exact Alg.-2 count of the
    sample scaled by rho^-4 (reading R18).  Returns dict(sampled_B, sampled_N, estimates)."""
    sb, sn, est = [], [], []
    for t in range(trials):
        r = route_g(sparsify(g, rho, seed, t), threads=threads)
        sb.append(r["B"])
        sn.append(r["N"])
        est.append(r["B"] / rho ** 4)
    return dict(sampled_B=sb, sampled_N=sn, estimates=est)


def positive_subgraph(g):
    """Case-study restriction ("only formed by the edges with sign/weight as 1";
    SPEC.md:449): the graph with its positive edges only, vertex sets unchanged."""
    from synth.graphs import SignedBipartite
    keep = g.sign == 1
    u = np.repeat(np.arange(g.n_u), np.diff(g.row_ptr.astype(np.int64)))[keep]
    rp = np.zeros(g.n_u + 1, np.uint64)
    np.add.at(rp, u + 1, 1)
    return SignedBipartite(g.n_u, g.n_v, np.cumsum(rp).astype(np.uint64), g.col[keep].copy(),
                           g.sign[keep].copy())


def topk_vertices(g, k: int, side: int = 0, metric: str = "balanced", threads=None):
    """Top-k vertices of a side: by per-vertex balanced count (vBBFC) or by
    degree, score desc then id asc, all vertices ranked.  Returns [(id, score)]."""
    cnt = g.n_u if side == 0 else g.n_v
    if metric == "degree":
        if side == 0:
            score = np.diff(g.row_ptr.astype(np.int64))
        else:
            score = np.bincount(g.col.astype(np.int64), minlength=g.n_v)
    else:
        verts = np.arange(cnt, dtype=np.uint32) + (0 if side == 0 else g.n_u)
        score = route_s(g, verts=verts, threads=threads)[0].astype(np.int64)
    order = sorted(range(cnt), key=lambda i: (-int(score[i]), i))
    return [(i, int(score[i])) for i in order[:k]]
