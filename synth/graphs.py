"""Seeded synthetic signed bipartite graphs — the inputs both sides are tested on.

This module is shared by the CUDA path's tests/bench AND the CPU oracle's tests,
so it holds NONE of the method's arithmetic (no wedges, no butterflies, no
priorities): it only draws graphs.  Every graph is returned as a U-side CSR

    row_ptr : uint64[n_u + 1]   (row_ptr[0] == 0)
    col     : uint32[nnz]       V-side index of each edge, ascending inside a row
    sign    : uint8[nnz]        1 = positive, 0 = negative  ("weight 1
                                 ... positive", the sign protocol of §Datasets)

The five recipes are BASELINE.json `configs[0..4]`, with the exact draw order
pinned in DESIGN.md §"Input recipe".  The paper's datasets
are not available; these synthetic graphs stand in for them.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np


@dataclass
class SignedBipartite:
    n_u: int
    n_v: int
    row_ptr: np.ndarray  # uint64 [n_u+1]
    col: np.ndarray      # uint32 [nnz]
    sign: np.ndarray     # uint8  [nnz]
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.col.shape[0])

    def edges(self):
        """(u, v, sign) arrays in CSR order."""
        u = np.repeat(np.arange(self.n_u, dtype=np.int64), np.diff(self.row_ptr.astype(np.int64)))
        return u, self.col.astype(np.int64), self.sign.copy()

    def dense_sign(self) -> np.ndarray:
        """n_u x n_v int8 matrix: +1 positive edge, -1 negative edge, 0 no edge."""
        m = np.zeros((self.n_u, self.n_v), dtype=np.int8)
        u, v, s = self.edges()
        m[u, v] = np.where(s == 1, 1, -1).astype(np.int8)
        return m

    def sha256(self) -> str:
        h = hashlib.sha256()
        h.update(np.array([self.n_u, self.n_v], dtype=np.uint64).tobytes())
        for a in (self.row_ptr, self.col, self.sign):
            h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()


def from_edges(n_u: int, n_v: int, u, v, s, name: str = "", check_dup: bool = True) -> SignedBipartite:
    """Build the U-side CSR from an edge list (any order). Rows sorted by v."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    s = np.asarray(s, dtype=np.uint8)
    key = u * max(n_v, 1) + v
    order = np.argsort(key, kind="stable")
    key, u, v, s = key[order], u[order], v[order], s[order]
    if check_dup and key.size and np.any(key[1:] == key[:-1]):
        raise ValueError("duplicate edge")
    row_ptr = np.zeros(n_u + 1, dtype=np.uint64)
    if u.size:
        row_ptr[1:] = np.cumsum(np.bincount(u, minlength=n_u)).astype(np.uint64)
    return SignedBipartite(n_u, n_v, row_ptr, v.astype(np.uint32), s, name)


def _from_sorted_keys(n_u: int, n_v: int, key: np.ndarray, sign: np.ndarray, name: str) -> SignedBipartite:
    u = key // n_v
    v = (key % n_v).astype(np.uint32)
    row_ptr = np.zeros(n_u + 1, dtype=np.uint64)
    row_ptr[1:] = np.cumsum(np.bincount(u, minlength=n_u)).astype(np.uint64)
    return SignedBipartite(n_u, n_v, row_ptr, v, sign.astype(np.uint8), name)


# ----------------------------------------------------------------------------- small graphs

def random_bipartite(n_u: int, n_v: int, p_edge: float, p_pos: float, seed: int) -> SignedBipartite:
    """SPEC corpus graph: each of the n_u*n_v pairs present w.p. p_edge,
    each present edge positive w.p. p_pos. Draw order: presence matrix, then signs."""
    rng = np.random.default_rng(seed)
    present = rng.random((n_u, n_v)) < p_edge
    u, v = np.nonzero(present)
    s = (rng.random(u.size) < p_pos).astype(np.uint8)
    return from_edges(n_u, n_v, u, v, s, name=f"rand{n_u}x{n_v}_p{p_edge}_q{p_pos}_s{seed}")


def complete(m: int, n: int, sign_fn=None) -> SignedBipartite:
    """K_{m,n}; sign_fn(u, v) -> 0/1 (default all positive)."""
    u, v = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    u, v = u.ravel(), v.ravel()
    s = np.ones(u.size, dtype=np.uint8) if sign_fn is None else np.array(
        [sign_fn(a, b) for a, b in zip(u, v)], dtype=np.uint8)
    return from_edges(m, n, u, v, s, name=f"K{m},{n}")


# ----------------------------------------------------------------------------- BASELINE configs

def config1(seed: int = 1) -> SignedBipartite:
    """configs[0]: |U|=200, |V|=150, 2,000 distinct edges uniformly at random, sign + w.p. 0.7.
    Draw order: rng.choice(200*150, 2000, replace=False) -> pair ids; then U(0,1)<0.7 signs."""
    n_u, n_v, m = 200, 150, 2000
    rng = np.random.default_rng(seed)
    ids = rng.choice(n_u * n_v, size=m, replace=False)
    s = (rng.random(m) < 0.7).astype(np.uint8)
    order = np.argsort(ids)
    return _from_sorted_keys(n_u, n_v, ids[order].astype(np.int64), s[order], "config1")


def config2(seed: int = 2) -> SignedBipartite:
    """configs[1]: actor-movie-shaped graph (IMDb rating >= 6 -> positive).
    U = 5,000 actors, V = 4,800 movies.  Draw order:
      1. actor weight d_i ~ Zipf(1.8), values > 80 redrawn until in [1, 80];
      2. cast size c_j ~ Poisson(5) for every movie j;
      3. for j = 0..4799: cast = c_j distinct actors drawn without replacement prop. to d;
      4. movie score ~ N(6.4, 1.0); every edge of movie j is positive iff score_j >= 6;
      5. actor degree capped at 80 by dropping that actor's edges to the highest movie ids."""
    n_u, n_v = 5000, 4800
    rng = np.random.default_rng(seed)
    d = rng.zipf(1.8, size=n_u)
    bad = d > 80
    while bad.any():
        d[bad] = rng.zipf(1.8, size=int(bad.sum()))
        bad = d > 80
    c = rng.poisson(5.0, size=n_v)
    p = d / d.sum()
    us, vs = [], []
    for j in range(n_v):
        k = int(min(c[j], n_u))
        if k == 0:
            continue
        cast = rng.choice(n_u, size=k, replace=False, p=p)
        us.append(cast)
        vs.append(np.full(k, j, dtype=np.int64))
    score = rng.normal(6.4, 1.0, size=n_v)
    u = np.concatenate(us).astype(np.int64)
    v = np.concatenate(vs)
    # cap actor degree at 80: keep each actor's 80 lowest movie ids
    key = u * n_v + v
    order = np.argsort(key)
    u, v = u[order], v[order]
    first = np.searchsorted(u, u, side="left")
    keep = (np.arange(u.size) - first) < 80
    u, v = u[keep], v[keep]
    s = (score[v] >= 6.0).astype(np.uint8)
    return _from_sorted_keys(n_u, n_v, u * n_v + v, s, "config2")


def chung_lu_weights(n: int, mean: float, wmax: float, gamma: float) -> np.ndarray:
    """w_i = c (i + i0)^(-1/(gamma-1)), with c, i0 solved so that w_0 = wmax and mean(w) = mean."""
    alpha = 1.0 / (gamma - 1.0)
    idx = np.arange(n, dtype=np.float64)

    def total(i0):
        return float(np.sum(wmax * (i0 / (idx + i0)) ** alpha))

    lo, hi = 1e-9, 1e12
    target = mean * n
    for _ in range(64):
        mid = np.sqrt(lo * hi)
        if total(mid) < target:
            lo = mid
        else:
            hi = mid
    i0 = np.sqrt(lo * hi)
    return wmax * (i0 / (idx + i0)) ** alpha


def _accel():
    """torch CUDA device for the exact, order-free primitives below (searchsorted of float64
    keys, sort-based unique) when a GPU is present; results are identical to numpy's."""
    try:
        import torch
        if torch.cuda.is_available():
            return torch
    except Exception:
        pass
    return None


def _searchsorted_right(cdf: np.ndarray, r: np.ndarray) -> np.ndarray:
    t = _accel()
    if t is None:
        return np.searchsorted(cdf, r, side="right")
    out = t.searchsorted(t.from_numpy(cdf).cuda(), t.from_numpy(r).cuda(), right=True)
    return out.cpu().numpy()


def _unique_first(keys: np.ndarray):
    """np.unique(keys, return_index=True): sorted distinct keys and first occurrence index."""
    t = _accel()
    if t is None:
        return np.unique(keys, return_index=True)
    k = t.from_numpy(keys).cuda()
    uniq, inv = t.unique(k, sorted=True, return_inverse=True)
    pos = t.arange(k.numel(), device=k.device)
    first = t.full((uniq.numel(),), k.numel(), dtype=t.int64, device=k.device)
    first.scatter_reduce_(0, inv, pos, reduce="amin")
    return uniq.cpu().numpy(), first.cpu().numpy()


def chung_lu(n_u: int, n_v: int, m: int, gamma: float, wmax_u: float, wmax_v: float, seed: int):
    """Distinct (u, v) pairs, endpoints drawn independently prop. to Chung-Lu weights.
    Draw order: batch 0 of ceil(1.2 m) draws, then batches of ceil(0.1 m) draws, each batch
    drawing all its u endpoints then all its v endpoints, until >= m distinct pairs exist;
    the first m distinct pairs in draw order are kept.  Returns the sorted int64 keys
    u * n_v + v and the rng (the sign draws continue from it)."""
    rng = np.random.default_rng(seed)
    wu = chung_lu_weights(n_u, m / n_u, wmax_u, gamma)
    wv = chung_lu_weights(n_v, m / n_v, wmax_v, gamma)
    cu = np.cumsum(wu); cu /= cu[-1]
    cv = np.cumsum(wv); cv /= cv[-1]
    chunks = []
    batch = int(np.ceil(1.2 * m))
    while True:
        bu = _searchsorted_right(cu, rng.random(batch)).clip(0, n_u - 1)
        bv = _searchsorted_right(cv, rng.random(batch)).clip(0, n_v - 1)
        chunks.append(bu.astype(np.int64) * n_v + bv)
        keys = np.concatenate(chunks) if len(chunks) > 1 else chunks[0]
        uniq, first = _unique_first(keys)
        if uniq.size >= m:
            break
        batch = int(np.ceil(0.1 * m))
    if uniq.size == m:
        return uniq, rng
    keep = np.sort(first)[:m]              # first m distinct pairs in draw order
    return np.sort(keys[keep]), rng


def config3(seed: int = 3) -> SignedBipartite:
    """configs[2]: Chung-Lu power-law, |U|=1,000,000, |V|=200,000, 10M distinct edges,
    exponent 2.1 both sides, weight max 20,000; signs iid positive w.p. 0.8."""
    n_u, n_v, m = 1_000_000, 200_000, 10_000_000
    key, rng = chung_lu(n_u, n_v, m, 2.1, 20_000.0, 20_000.0, seed)
    s = rng.random(m) < 0.8
    return _from_sorted_keys(n_u, n_v, key, s, "config3")


def config4(seed: int = 4) -> SignedBipartite:
    """configs[3]: dense block graph |U|=|V|=16,384, each pair iid present w.p. 0.05,
    drawn in row blocks of 1,024; then signs iid positive w.p. 0.5 (CSR order)."""
    n = 16384
    rng = np.random.default_rng(seed)
    keys = []
    for r0 in range(0, n, 1024):
        blk = rng.random((1024, n)) < 0.05
        uu, vv = np.nonzero(blk)
        keys.append((uu.astype(np.int64) + r0) * n + vv)
    key = np.concatenate(keys)
    s = rng.random(key.size) < 0.5
    return _from_sorted_keys(n, n, key, s, "config4")


def config5(seed: int = 5) -> SignedBipartite:
    """configs[4]: large skewed graph, |U|=8,000,000, |V|=2,000,000, 50M distinct edges,
    Chung-Lu exponent 1.9, weight max 100,000; per-V bias b_v ~ Beta(3,1) (drawn for all V
    first), then edge sign positive w.p. b_v (CSR order)."""
    n_u, n_v, m = 8_000_000, 2_000_000, 50_000_000
    key, rng = chung_lu(n_u, n_v, m, 1.9, 100_000.0, 100_000.0, seed)
    b = rng.beta(3.0, 1.0, size=n_v)
    v = key % n_v
    s = rng.random(m) < b[v]
    return _from_sorted_keys(n_u, n_v, key, s, "config5")


def core_periphery(n_u: int, n_v: int, m: int, gamma: float, wmax_u: float, wmax_v: float, core_u: int,
                   core_v: int, p_core: float, p_pos: float, seed: int, name: str = "",
                   core_random: bool = False) -> SignedBipartite:
    """A Chung-Lu power-law periphery (chung_lu above, m distinct pairs) plus a planted dense core
    of core_u x core_v vertices, each of its pairs present w.p. p_core (drawn in row blocks of
    1,024 after the periphery); the core sits on the highest-weight ids [0, core_u) x [0, core_v),
    or (core_random) on ids drawn without replacement after the block (a dense community away from
    the periphery's hubs).  Then every edge of the union positive w.p. p_pos (CSR order).  Stands
    in for the dense-core / sparse-remainder regime of NEXT-3 (the Senate/House-like dense
    blocks, inside a power-law graph)."""
    key, rng = chung_lu(n_u, n_v, m, gamma, wmax_u, wmax_v, seed)
    blocks = []
    for r0 in range(0, core_u, 1024):
        rows = min(1024, core_u - r0)
        uu, vv = np.nonzero(rng.random((rows, core_v)) < p_core)
        blocks.append((uu.astype(np.int64) + r0, vv.astype(np.int64)))
    bu = np.concatenate([b[0] for b in blocks]) if blocks else np.zeros(0, np.int64)
    bv = np.concatenate([b[1] for b in blocks]) if blocks else np.zeros(0, np.int64)
    if core_random:
        bu = rng.choice(n_u, size=core_u, replace=False)[bu]
        bv = rng.choice(n_v, size=core_v, replace=False)[bv]
    key = np.unique(np.concatenate([key, bu * n_v + bv]))
    s = rng.random(key.size) < p_pos
    return _from_sorted_keys(n_u, n_v, key, s, name or f"cp{n_u}x{n_v}_c{core_u}x{core_v}_s{seed}")


def config_hybrid(seed: int = 6) -> SignedBipartite:
    """The NEXT-3 hybrid workload (not a BASELINE config): a dense community of 8,192 x 8,192
    vertices at density 0.2 (~13.4M edges, degrees ~1,640; placed on random ids) inside a Chung-Lu
    power-law periphery of |U|=1M, |V|=200K, 5M distinct pairs, exponent 2.1, weight max 1,000
    (so the community is the top of the priority order); signs iid positive w.p. 0.8."""
    return core_periphery(1_000_000, 200_000, 5_000_000, 2.1, 1_000.0, 1_000.0, 8192, 8192, 0.2, 0.8, seed,
                          "config_hybrid", core_random=True)


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5, 6: config_hybrid}  # 6: NEXT-3 workload


def make_config(i: int) -> SignedBipartite:
    return CONFIGS[i]()
