// plan.cu — S5 of the hot path: per eligible middle entry (x -> v) the first eligible end
// ub = upper_bound(N(v), l(x)) (Alg. 2 line 10 "w in Γ(v) | p(w) < p(u)", as a
// suffix of the priority-sorted list), the per-start work, the wedge count W of the route,
// tiering of starts by work, and the split of hub starts into end-range units.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "bbf_internal.cuh"

namespace bbf {

constexpr uint32_t kT1Max = 512;  // starts with at most this many (pruned) wedges -> warp hash
// starts with (kT1Max, kT2Max] wedges -> one CTA with a shared hash (k_t2); above -> hub units
// (k_t3).  Env BBF_T2_MAX overrides (0 disables the T2 tier).

namespace {

struct RouteRows {
  int route;  // 0 G, 1 S(U), 2 S(V), 3 S(U) with the ends BEFORE the start (per-edge counts)
  uint32_t n_u, n;
  // hybrid core (route G only): rows of side-local rank < nc[side] are core; ccnt[row] = the
  // row's entries inside the other side's core (a prefix: rows are sorted by local rank)
  uint32_t nc0, nc1;
  const uint32_t* ccnt;
  __device__ __forceinline__ bool core(uint32_t x) const {
    return x < n_u ? x < nc0 : x - n_u < nc1;
  }
  __device__ __forceinline__ bool in_route(uint32_t x) const {
    return route == 0 || (route == 1 || route == 3 ? x < n_u : x >= n_u);
  }
};

// rsafe[side] = 1 + the largest local rank of an end whose end-role totals could reach 2^32:
// sum_x C(c_xw, 2) <= min(C(W, 2), W * (deg(w) - 1) / 2) with W = the wedges ending at w
// rmid[side] likewise for the middle role: a middle's totals are at most (wedges through it) x
// (the largest pair count c_xw) <= C(deg, 2) x (the largest degree on the other side)
__global__ void k_rsafe(const unsigned long long* __restrict__ win, const uint32_t* __restrict__ degs, uint32_t n_u,
                        uint32_t n, uint32_t* __restrict__ rsafe) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const unsigned long long W = win[r], d = degs[r];
  const bool safe = W <= 92681ull || W * d < (1ull << 33);
  const uint32_t side = r < n_u ? 0 : 1, lr = r < n_u ? r : r - n_u;
  if (!safe) atomicMax(&rsafe[side], lr + 1u);
  const unsigned long long dmax = n_u < n ? degs[side ? 0 : n_u] : 0ull;  // other side's rank 0
  const unsigned long long pairs = d * (d - (d ? 1ull : 0ull)) / 2ull;
  if (d > 1 && (pairs >= (1ull << 32) || pairs * dmax >= (1ull << 32))) atomicMax(&rsafe[2 + side], lr + 1u);
}

// one thread per adjacency entry: if the entry is a middle of its row for this route, compute
// ub, the pruned segment length (ends of degree >= 2) and the full count (all ends; W_G)
// (win != nullptr, route G) also the per-end bound of incoming wedges (see make_plan): the same entry's
// middle and reverse position give the eligible starts before it (one pass over erow/adj/rev)
// the middle row's (off, off + 1, end1, mid) in one 16-byte record: one random sector per entry
// instead of four
__global__ void k_rowinfo(const uint32_t* __restrict__ off, const uint32_t* __restrict__ end1,
                          const uint32_t* __restrict__ mid, uint32_t n, uint4* __restrict__ ri) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) ri[r] = make_uint4(off[r], off[r + 1], end1[r], mid[r]);
}

__global__ void k_plan_entries(RouteRows rr, const uint32_t* __restrict__ off,
                               const uint32_t* __restrict__ adj, const uint32_t* __restrict__ rev,
                               const uint32_t* __restrict__ erow,
                               const uint32_t* __restrict__ mid,
                               const uint32_t* __restrict__ end1, const uint4* __restrict__ rowinfo, uint64_t m,
                               uint32_t* __restrict__ ub, unsigned long long* __restrict__ work,
                               unsigned long long* __restrict__ w_full, unsigned long long* __restrict__ win) {
  unsigned long long full = 0;
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t e0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) & ~31ull; e0 < m;
       e0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t e64 = e0 + lane;
    uint32_t x = 0xffffffffu;
    unsigned long long c = 0, l_seg = 0;
    if (e64 < m) {
      const uint32_t e = (uint32_t)e64;
      x = erow[e];
      const uint32_t ob = x < rr.n_u ? rr.n_u : 0;
      const uint32_t rv = ob + (adj[e] & kMask);
      const uint32_t r = rev[e];
      const uint32_t lo = rr.route == 0 ? mid[x] : off[x];
      const bool mid_entry = rr.in_route(x) && e >= lo && e < end1[x];
      uint4 rvi = make_uint4(0, 0, 0, 0);  // off[rv], off[rv + 1], end1[rv], mid[rv]
      if (mid_entry || win) rvi = rowinfo[rv];
      if (mid_entry) {
        if (rr.route == 3) {  // ends before x in N(v): [off(v), r), of degree >= 2
          const uint32_t u = rvi.x, en = min(rvi.z, r);
          ub[e] = u;
          full += r - u;
          l_seg = en > u ? en - u : 0;
        } else {
          const uint32_t f = rvi.y;
          const uint32_t u = r + 1;  // x's entry in its middle's row is the reverse entry
          const uint32_t en = rvi.z;
          // hybrid: a core start's wedges through a core middle skip the core ends (counted by
          // the dense core, hybrid.cu); W_G (full) stays the paper's count
          const uint32_t u2 = (rr.ccnt && rr.core(x) && rr.core(rv)) ? max(u, rvi.x + rr.ccnt[rv]) : u;
          ub[e] = u2;
          full += f - u;
          l_seg = en > u2 ? en - u2 : 0;
        }
      }
      if (win) {
        const uint32_t o = rvi.x, pos = r - o, hi = rvi.w - o;
        c = pos < hi ? pos : hi;
      }
    }
    // per-row sums (work: pruned segment lengths; win: the end bound) over runs of equal rows in
    // the warp, one atomic per run
    const uint32_t xp = __shfl_up_sync(0xffffffffu, x, 1);
    const uint32_t starts = __ballot_sync(0xffffffffu, lane == 0 || xp != x);
    const int gs = 31 - __clz(starts & (0xffffffffu >> (31 - lane)));
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(0xffffffffu, l_seg, o);
      const unsigned long long t2 = __shfl_up_sync(0xffffffffu, c, o);
      if ((int)lane - o >= gs) { l_seg += t; c += t2; }
    }
    const bool last = lane == 31 || ((starts >> (lane + 1)) & 1u);
    if (last && x != 0xffffffffu) {
      if (l_seg) atomicAdd(&work[x], l_seg);
      if (win && c) atomicAdd(&win[x], c);
    }
  }
  for (int o = 16; o; o >>= 1) full += __shfl_xor_sync(0xffffffffu, full, o);
  if ((threadIdx.x & 31) == 0 && full) atomicAdd(w_full, full);
}

__global__ void k_seg_bounds(RouteRows rr, const uint32_t* __restrict__ off,
                             const uint32_t* __restrict__ mid, const uint32_t* __restrict__ end1,
                             uint32_t* __restrict__ b, uint32_t* __restrict__ e) {
  uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= rr.n) return;
  if (!rr.in_route(x)) { b[x] = e[x] = 0; return; }
  uint32_t lo = rr.route == 0 ? mid[x] : off[x];
  uint32_t hi = end1[x];
  b[x] = lo;
  e[x] = hi > lo ? hi : lo;
}

// count T1 / T3 rows, W per tier, units per T3 row
// w_target = max(W_pruned / (nranks * SMs * 6 + 1), 2^16), from the device-side W_pruned (no host
// round trip between the work reduction and the tiers)
__global__ void k_tier(uint32_t n, const uint64_t* __restrict__ work, const unsigned long long* __restrict__ d_wp,
                       uint64_t w_div, uint64_t t1max, uint64_t t2max, const uint32_t* __restrict__ mlo,
                       const uint32_t* __restrict__ mhi, uint32_t* __restrict__ nunits,
                       unsigned long long* __restrict__ acc) {
  const uint64_t wt = *d_wp / w_div, w_target = wt > (1ull << 16) ? wt : (1ull << 16);
  uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long w1 = 0, w3 = 0, m3 = 0, w2 = 0, s3 = 0;  // s3: starts with hub units
  uint32_t u = 0;
  if (x < n) {
    uint64_t w = work[x];
    if (w > 0 && w <= t1max) w1 = w;
    if (w > t1max && w <= t2max) w2 = w;
    if (w > t1max && w > t2max) {
      w3 = w;
      m3 = mhi[x] - mlo[x];
      u = (uint32_t)std::min<uint64_t>((w + w_target - 1) / w_target, 4096);
      s3 = 1;
    }
    nunits[x] = u;
  }
  for (int o = 16; o; o >>= 1) {
    w1 += __shfl_xor_sync(0xffffffffu, w1, o);
    w3 += __shfl_xor_sync(0xffffffffu, w3, o);
    m3 += __shfl_xor_sync(0xffffffffu, m3, o);
    w2 += __shfl_xor_sync(0xffffffffu, w2, o);
    s3 += __shfl_xor_sync(0xffffffffu, s3, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (w1) atomicAdd(&acc[0], w1);
    if (w3) atomicAdd(&acc[1], w3);
    if (m3) atomicAdd(&acc[2], m3);
    if (w2) atomicAdd(&acc[3], w2);
    if (s3) atomicAdd(&acc[4], s3);
  }
}

struct IsT2 {  // lo < work <= hi
  const uint64_t* work;
  uint64_t lo, hi;
  __device__ __forceinline__ bool operator()(uint32_t x) const {
    uint64_t w = work[x];
    return w > lo && w <= hi;
  }
};



// fill the units of every T3 row: split [l(x)+1, L4) into nunits pieces of ~equal sum of end
// degrees (expected wedges per end rank are proportional to the end's degree)
__global__ void k_units(int route, uint32_t n, uint32_t n_u, const uint32_t* __restrict__ nunits,
                        const uint32_t* __restrict__ ustart, const uint64_t* __restrict__ degpre,
                        uint32_t L4u, uint32_t L4v, const uint32_t* __restrict__ mid_lo,
                        const uint32_t* __restrict__ end1, const uint64_t* __restrict__ work,
                        Unit* __restrict__ units, unsigned int* __restrict__ max_mid,
                        unsigned long long* __restrict__ max_work) {
  uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  uint32_t k = nunits[x];
  if (!k) return;
  uint32_t sb = x < n_u ? 0 : n_u;
  uint32_t L4 = x < n_u ? L4u : L4v;
  uint32_t lx = x - sb;
  // ends after x (routes G, S) or before x (route 3, per-edge counts), of degree >= 2
  uint32_t lo = route == 3 ? 0u : lx + 1, hi = route == 3 ? (lx < L4 ? lx : L4) : (L4 > lo ? L4 : lo);
  atomicMax(max_mid, end1[x] - mid_lo[x]);
  atomicMax(max_work, (unsigned long long)work[x]);
  uint32_t base = ustart[x];
  // prefix over rows: P(r) = sum degs[0..r]; sum over side-local [a, b) = P(sb+b-1) - P(sb+a-1)
  auto pre = [&](uint32_t l) -> uint64_t {  // sum of degs of side-local ranks [0, l)
    uint32_t r = sb + l;
    uint64_t at = r ? degpre[r - 1] : 0;
    uint64_t base0 = sb ? degpre[sb - 1] : 0;
    return at - base0;
  };
  uint64_t s0 = pre(lo), s1 = pre(hi);
  uint32_t prev = lo;
  for (uint32_t j = 0; j < k; ++j) {
    uint32_t cut;
    if (j + 1 == k) {
      cut = hi;
    } else {
      uint64_t t = s0 + (s1 - s0) * (uint64_t)(j + 1) / k;
      uint32_t a = prev, b = hi;  // smallest l in [prev, hi] with pre(l) >= t
      while (a < b) {
        uint32_t m = a + (b - a) / 2;
        if (pre(m) < t) a = m + 1; else b = m;
      }
      cut = a;
    }
    units[base + j] = Unit{x, prev, cut, 0};
    prev = cut;
  }
}

// middle counts of the listed starts (the split starts' boundaries)
__global__ void k_gather_m(const uint32_t* __restrict__ xs, uint32_t cnt, const uint32_t* __restrict__ mid_lo,
                           const uint32_t* __restrict__ end1, uint32_t* __restrict__ m) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) m[i] = end1[xs[i]] > mid_lo[xs[i]] ? end1[xs[i]] - mid_lo[xs[i]] : 0u;
}

// one CTA per boundary between two units of a split start: for each middle entry of the start, the
// first entry of its end segment [ub, en) with rank >= the boundary (the search the hub kernel's
// pre-scan would otherwise repeat in both units)
struct CutDesc {
  uint32_t x, cut;
  unsigned long long off;
};
__global__ void k_split_cuts(const CutDesc* __restrict__ d, const uint32_t* __restrict__ mid_lo,
                             const uint32_t* __restrict__ end1, const uint32_t* __restrict__ adj,
                             const uint32_t* __restrict__ ub, const uint32_t* __restrict__ ue, uint32_t n_u,
                             uint32_t* __restrict__ tab) {
  const CutDesc c = d[blockIdx.x];
  const uint32_t ob = c.x < n_u ? n_u : 0;
  const uint32_t m_lo = mid_lo[c.x], m = end1[c.x] - m_lo;
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
    const uint32_t e = m_lo + i;
    const uint32_t v = adj[e] & kMask;
    uint32_t b = ub[e], f = end1[ob + v];
    if (ue) f = min(f, ue[e]);
    while (b < f) {
      const uint32_t md = b + (f - b) / 2;
      if ((adj[md] & kMask) < c.cut) b = md + 1; else f = md;
    }
    tab[c.off + i] = b;
  }
}

inline unsigned grid_for(uint64_t n, unsigned block, unsigned cap = 148u * 64u) {
  uint64_t g = (n + block - 1) / block;
  if (g == 0) g = 1;
  return (unsigned)std::min<uint64_t>(g, cap);
}

}  // namespace

void free_plan(Plan* p, cudaStream_t st) {
  if (p->ub) dfree(p->ub, st);
  if (p->work) dfree(p->work, st);
  if (p->t1) dfree(p->t1, st);
  if (p->t2) dfree(p->t2, st);
  if (p->t2s) dfree(p->t2s, st);
  if (p->t1b) dfree(p->t1b, st);
  if (p->t2h) dfree(p->t2h, st);
  if (p->units) dfree(p->units, st);
  if (p->cut_tab) dfree(p->cut_tab, st);
  if (p->unit_cut) dfree(p->unit_cut, st);

  *p = Plan{};
}

bbf_status make_plan(bbf_graph* g, int route, Plan* p, bool all_t3, const uint32_t* nc) {
  NvtxRange nvtx_("bbf::make_plan");
  cudaStream_t st = g->stream;
  const uint32_t n = g->n;
  const uint64_t m = 2 * g->nnz;
  free_plan(p, st);
  p->route = route;
  const bool hyb = route == 0 && nc && nc[0] && nc[1] && g->hyb.ccnt;
  p->nc[0] = hyb ? nc[0] : 0u;
  p->nc[1] = hyb ? nc[1] : 0u;
  RouteRows rr{route, g->n_u, n, p->nc[0], p->nc[1], hyb ? g->hyb.ccnt : nullptr};
  BBF_CUDA(dmalloc(&p->ub, 4ull * (m + 1), st));
  BBF_CUDA(dmalloc(&p->work, 8ull * (n + 1), st));
  uint32_t *sb, *se, *nunits, *ustart;
  unsigned long long* acc;
  BBF_CUDA(dmalloc(&sb, 4ull * (n + 1), st));
  BBF_CUDA(dmalloc(&se, 4ull * (n + 1), st));
  BBF_CUDA(dmalloc(&nunits, 4ull * (n + 1), st));
  BBF_CUDA(dmalloc(&ustart, 4ull * (n + 1), st));
  BBF_CUDA(dmalloc(&acc, 8 * sizeof(unsigned long long), st));
  BBF_CUDA(cudaMemsetAsync(acc, 0, 8 * sizeof(unsigned long long), st));
  BBF_CUDA(cudaMemsetAsync(p->work, 0, 8ull * (n + 1), st));
  // per-end bound of incoming wedges (route G, per-vertex REDs packing):
  // the wedges ending at w from starts before both w and the middle v, per entry (w -> v):
  // min(position of w in N(v), mid(v) - off(v))
  const bool want_pack = route == 0 && m && !getenv("BBF_NO_PACKED_END");  // env: test hook
  unsigned long long* win = nullptr;
  if (want_pack) {
    BBF_CUDA(dmalloc(&win, 8ull * (n + 1), st));
    BBF_CUDA(cudaMemsetAsync(win, 0, 8ull * (n + 1), st));
  }
  if (m) {
    uint4* rowinfo;
    BBF_CUDA(dmalloc(&rowinfo, 16ull * n, st));
    k_rowinfo<<<(n + 255) / 256, 256, 0, st>>>(g->off, g->end1, g->mid, n, rowinfo);
    k_plan_entries<<<grid_for(m, 256), 256, 0, st>>>(rr, g->off, g->adj, g->rev, g->erow, g->mid, g->end1, rowinfo,
                                                   m, p->ub, (unsigned long long*)p->work, &acc[0], win);
    g->launches += 2;
    dfree(rowinfo, st);
  }
  if (n) {
    k_seg_bounds<<<grid_for(n, 256, 1u << 30), 256, 0, st>>>(rr, g->off, g->mid, g->end1, sb, se);
    g->launches += 1;
  }
  uint32_t h_rs[4] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu};  // no packing (route S, empty graph)
  if (want_pack) {  // (env BBF_NO_PACKED_END: every end / middle takes two REDs)
    uint32_t* d_rs;
    BBF_CUDA(dmalloc(&d_rs, 16, st));
    BBF_CUDA(cudaMemsetAsync(d_rs, 0, 16, st));
    k_rsafe<<<(n + 255) / 256, 256, 0, st>>>(win, g->degs, g->n_u, n, d_rs);
    g->launches += 1;
    BBF_CUDA(rb_add(h_rs, d_rs, 16, st)); g->launches++;  // delivered by the next rb_sync
    dfree(win, st);
    dfree(d_rs, st);
  }
  // pruned total, to size units
  unsigned long long* d_wp;
  BBF_CUDA(dmalloc(&d_wp, 8, st));
  {
    size_t tb = 0;
    cub::DeviceReduce::Sum(nullptr, tb, p->work, d_wp, (int)n, st);
    void* tmp;
    BBF_CUDA(dmalloc(&tmp, tb + 16, st));
    BBF_CUDA(cub::DeviceReduce::Sum(tmp, tb, p->work, d_wp, (int)n, st));
    g->launches += kCubReduceKernels;
    dfree(tmp, st);
  }
  unsigned long long h_wp = 0, h_wf = 0;
  BBF_CUDA(rb_add(&h_wp, d_wp, 8, st)); g->launches++;  // delivered by the next rb_sync
  BBF_CUDA(rb_add(&h_wf, &acc[0], 8, st)); g->launches++;
  // hub units of ~1/6 of one SM's share of the whole job: with N ranks the share is W / (N * SMs),
  // so a rank's largest unit stays well below its per-SM work at any N
  int shard_rank = 0, shard_n = 1;
  shard_of(g, &shard_rank, &shard_n);
  (void)shard_rank;  // every rank builds the same plan
  p->nranks = shard_n;
  const uint64_t nranks = (uint64_t)shard_n;
  // hub units of ~1/3 of an SM share (BBF_UNIT_DIV tunes it; 3 measured best at N = 1 and 8:
  // finer units repeat the unit pre-scan of the hub's middles, coarser ones leave a tail)
  const uint64_t udiv = getenv("BBF_UNIT_DIV") ? std::max<uint64_t>(1, strtoull(getenv("BBF_UNIT_DIV"), nullptr, 10)) : 3ull;
  const uint64_t w_div = nranks * (uint64_t)g->num_sms * udiv + 1;

  // tiers and units
  // a T2 start's distinct ends (<= its wedges) must fit the k_t2 hash at load <= 1/2
  // all_t3: every start with work goes to the hub kernel (the per-edge counts need its records)
  const uint64_t t1max = all_t3 ? 0ull : (uint64_t)kT1Max;
  const uint64_t t2max = all_t3 ? 0ull : std::min<uint64_t>(
      getenv("BBF_T2_MAX") ? (uint64_t)atoll(getenv("BBF_T2_MAX")) : kT2MaxDefault, kT2HugeSlots * 3 / 4);
  BBF_CUDA(cudaMemsetAsync(acc, 0, 8 * sizeof(unsigned long long), st));
  if (n) {
    k_tier<<<grid_for(n, 256, 1u << 30), 256, 0, st>>>(n, p->work, d_wp, w_div, t1max, t2max, sb, se, nunits, acc);
    g->launches += 1;
  }
  BBF_CUDA(dmalloc(&p->t1, 4ull * (n + 1), st));
  BBF_CUDA(dmalloc(&p->t2, 4ull * (n + 1), st));
  BBF_CUDA(dmalloc(&p->t2s, 4ull * (n + 1), st));
  BBF_CUDA(dmalloc(&p->t1b, 4ull * (n + 1), st));
  BBF_CUDA(dmalloc(&p->t2h, 4ull * (n + 1), st));
  uint32_t* d_nsel;
  BBF_CUDA(dmalloc(&d_nsel, 20, st));
  const uint64_t t2mid = std::min<uint64_t>(kT2SmallMax, t2max), t2big = std::min<uint64_t>(kT2Slots * 3 / 4, t2max);
  const IsT2 big{p->work, t2mid, t2big}, small{p->work, t1max, std::max(t1max, t2mid)}, huge{p->work, t2big, t2max};
  const IsT2 t1s{p->work, 0, std::min<uint64_t>(kT1SmallMax, t1max)}, t1b{p->work, std::min<uint64_t>(kT1SmallMax, t1max), t1max};
  {
    cub::CountingInputIterator<uint32_t> it(0);
    size_t tb = 0, tb3 = 0;
    cub::DeviceSelect::If(nullptr, tb, it, p->t1, d_nsel, (int)n, t1s, st);
    cub::DeviceSelect::If(nullptr, tb3, it, p->t2, d_nsel + 1, (int)n, big, st);
    size_t tb2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb2, nunits, ustart, (int)(n + 1), st);
    tb = std::max(std::max(tb, tb2), tb3);
    void* tmp;
    BBF_CUDA(dmalloc(&tmp, tb + 16, st));
    BBF_CUDA(cub::DeviceSelect::If(tmp, tb, it, p->t1, d_nsel, (int)n, t1s, st));
    BBF_CUDA(cub::DeviceSelect::If(tmp, tb, it, p->t1b, d_nsel + 3, (int)n, t1b, st));
    BBF_CUDA(cub::DeviceSelect::If(tmp, tb, it, p->t2h, d_nsel + 4, (int)n, huge, st));
    BBF_CUDA(cub::DeviceSelect::If(tmp, tb, it, p->t2, d_nsel + 1, (int)n, big, st));
    BBF_CUDA(cub::DeviceSelect::If(tmp, tb, it, p->t2s, d_nsel + 2, (int)n, small, st));
    BBF_CUDA(cudaMemsetAsync(nunits + n, 0, 4, st));
    BBF_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, nunits, ustart, (int)(n + 1), st));
    g->launches += 5 * kCubSelectKernels + kCubScanKernels;
    dfree(tmp, st);
  }
  uint32_t h_nsel[5] = {0, 0, 0, 0, 0}, h_nunits = 0;
  unsigned long long h_acc[5];
  BBF_CUDA(rb_add(h_nsel, d_nsel, 20, st)); g->launches++;
  BBF_CUDA(rb_add(&h_nunits, ustart + n, 4, st)); g->launches++;
  BBF_CUDA(rb_add(h_acc, acc, 40, st)); g->launches++;
  BBF_CUDA(rb_sync(st));
  p->W_pruned = h_wp;
  p->W_full = h_wf;
  p->rsafe[0] = h_rs[0]; p->rsafe[1] = h_rs[1]; p->rmid[0] = h_rs[2]; p->rmid[1] = h_rs[3];
  const uint64_t w_target = std::max<uint64_t>(h_wp / w_div, 1ull << 16);  // (debug print)
  p->n_t1 = h_nsel[0];
  p->n_t2 = h_nsel[1];
  p->n_t2s = h_nsel[2];
  p->n_t1b = h_nsel[3];
  p->n_t2h = h_nsel[4];
  p->n_units = h_nunits;
  p->W_t1 = h_acc[0];
  p->W_t3 = h_acc[1];
  p->M_t3 = h_acc[2];
  p->W_t2 = h_acc[3];
  BBF_CUDA(dmalloc(&p->units, sizeof(Unit) * (h_nunits + 1), st));
  unsigned int* d_maxmid;  // [0] max middles, [2..3] max work (u64)
  BBF_CUDA(dmalloc(&d_maxmid, 16, st));
  BBF_CUDA(cudaMemsetAsync(d_maxmid, 0, 16, st));
  if (n && h_nunits) {
    k_units<<<grid_for(n, 256, 1u << 30), 256, 0, st>>>(route, n, g->n_u, nunits, ustart, g->degpre,
                                                      g->L4[0], g->L4[1], sb, g->end1, p->work,
                                                      p->units, d_maxmid, (unsigned long long*)(d_maxmid + 2));
    g->launches += 1;
  }
  unsigned int h_maxmid[4] = {0, 0, 0, 0};
  BBF_CUDA(rb_add(h_maxmid, d_maxmid, 16, st)); g->launches++;
  BBF_CUDA(rb_sync(st));
  p->max_mid = h_maxmid[0];
  p->max_work = *(unsigned long long*)(h_maxmid + 2);
  // cut tables of the split starts (consecutive units of one start share a boundary), when some
  // start has more than one unit
  if (h_nunits > h_acc[4]) {
    std::vector<Unit> hu(h_nunits);
    BBF_CUDA(cudaMemcpyAsync(hu.data(), p->units, sizeof(Unit) * h_nunits, cudaMemcpyDeviceToHost, st));
    std::vector<CutDesc> cd;
    std::vector<unsigned long long> uc(2ull * h_nunits, ~0ull);
    BBF_CUDA(cudaStreamSynchronize(st));
    bool any = false;
    for (uint32_t i = 0; i + 1 < h_nunits; ++i) any |= hu[i].x == hu[i + 1].x;
    if (any) {
      // the boundaries' starts, and their middle counts gathered on the device (no n-sized copy)
      std::vector<uint32_t> bx;
      for (uint32_t i = 0; i + 1 < h_nunits; ++i)
        if (hu[i].x == hu[i + 1].x) bx.push_back(hu[i].x);
      uint32_t* d_bx;
      BBF_CUDA(dmalloc(&d_bx, 8ull * bx.size(), st));
      BBF_CUDA(cudaMemcpyAsync(d_bx, bx.data(), 4ull * bx.size(), cudaMemcpyHostToDevice, st));
      k_gather_m<<<(unsigned)((bx.size() + 255) / 256), 256, 0, st>>>(d_bx, (uint32_t)bx.size(), sb, g->end1,
                                                                     d_bx + bx.size());
      g->launches += 1;
      std::vector<uint32_t> bm(bx.size());
      BBF_CUDA(cudaMemcpyAsync(bm.data(), d_bx + bx.size(), 4ull * bx.size(), cudaMemcpyDeviceToHost, st));
      BBF_CUDA(cudaStreamSynchronize(st));
      dfree(d_bx, st);
      unsigned long long off = 0;
      size_t b = 0;
      for (uint32_t i = 0; i + 1 < h_nunits; ++i) {
        if (hu[i].x != hu[i + 1].x) continue;
        cd.push_back(CutDesc{hu[i].x, hu[i].hi, off});
        uc[2ull * i + 1] = off;  // unit i's upper cut, unit i + 1's lower cut
        uc[2ull * (i + 1)] = off;
        off += bm[b++];
      }
      BBF_CUDA(dmalloc(&p->cut_tab, 4ull * (off + 1), st));
      BBF_CUDA(dmalloc(&p->unit_cut, 8ull * uc.size(), st));
      CutDesc* dcd;
      BBF_CUDA(dmalloc(&dcd, sizeof(CutDesc) * cd.size(), st));
      BBF_CUDA(cudaMemcpyAsync(dcd, cd.data(), sizeof(CutDesc) * cd.size(), cudaMemcpyHostToDevice, st));
      BBF_CUDA(cudaMemcpyAsync(p->unit_cut, uc.data(), 8ull * uc.size(), cudaMemcpyHostToDevice, st));
      k_split_cuts<<<(unsigned)cd.size(), 256, 0, st>>>(dcd, sb, g->end1, g->adj, p->ub, route == 3 ? g->rev : nullptr,
                                                        g->n_u, p->cut_tab);
      g->launches += 1;
      dfree(dcd, st);
    }
  }
  if (getenv("BBF_DEBUG") && atoi(getenv("BBF_DEBUG")) >= 2) {  // work histogram by log2 bucket
    std::vector<uint64_t> hw(n);
    cudaMemcpy(hw.data(), p->work, 8ull * n, cudaMemcpyDeviceToHost);
    unsigned long long cnt[40] = {0}, sum[40] = {0};
    for (uint32_t x = 0; x < n; ++x) {
      if (!hw[x]) continue;
      int b = 0;
      while ((2ull << b) <= hw[x]) ++b;
      cnt[b]++;
      sum[b] += hw[x];
    }
    for (int b = 0; b < 40; ++b)
      if (cnt[b]) fprintf(stderr, "[bbf]   work [2^%d, 2^%d): %llu starts, %llu wedges\n", b, b + 1, cnt[b], sum[b]);
  }
  if (getenv("BBF_DEBUG"))
    fprintf(stderr,
            "[bbf] plan route=%d W_full=%llu W_pruned=%llu W_t1=%llu (%u starts) W_t2=%llu (%u starts) W_t3=%llu (%u units) "
            "M_t3=%llu max_mid=%u w_target=%llu words U=%u V=%u\n",
            route, (unsigned long long)p->W_full, (unsigned long long)p->W_pruned,
            (unsigned long long)p->W_t1, p->n_t1, (unsigned long long)p->W_t2, p->n_t2,
            (unsigned long long)p->W_t3, p->n_units,
            (unsigned long long)p->M_t3, p->max_mid, (unsigned long long)w_target, g->zones[0].WB[5],
            g->zones[1].WB[5]);
  dfree(sb, st);
  dfree(se, st);
  dfree(nunits, st);
  dfree(ustart, st);
  dfree(acc, st);
  dfree(d_wp, st);
  dfree(d_nsel, st);
  dfree(d_maxmid, st);
  BBF_CUDA(cudaGetLastError());
  p->valid = true;
  return BBF_OK;
}

}  // namespace bbf
