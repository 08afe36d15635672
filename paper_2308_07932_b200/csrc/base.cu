// base.cu — Alg. 1 BB-Base on the GPU: the paper's baseline, kept to
// reproduce its BB-Base vs BB-Bucket regime.
//
// Same priority-eligible wedges as Alg. 2 (rank-space CSR, route-G plan: middles from mid[x],
// ends from ub[e]; ends of degree 1 are pruned as everywhere else: their H(w) has one entry
// and no pair).  Per start x (one 1024-thread CTA):
//   sweep 1  |H(w)| per end w in a shared open-addressing table (lines 7-9);
//   scan     list offsets;
//   sweep 2  H(w).add(v): each wedge stores its two sign bits (neg(x,v) << 1 | neg(v,w)) in its
//            end's list in a per-CTA global scratch area;
//   pairs    every unordered pair (v1, v2) of every list is checked explicitly (lines 10-13):
//            balanced iff the four edges hold an even number of negative signs (Def. Balanced
//            butterfly), i.e. the XOR of the two entries has even parity.
// Cost Σ_(x,w) C(|H(w)|, 2) = the number of butterflies — the explicit enumeration Alg. 2's
// buckets avoid.  Warp per list, rows of the pair triangle folded (row q with row c-2-q) so
// the lanes' loops have equal length.
#include <algorithm>

#include <cub/cub.cuh>

#include "bbf_internal.cuh"

namespace bbf {
namespace {

constexpr int kBaseThreads = 1024, kBaseWarps = kBaseThreads / 32;
constexpr uint32_t kBaseSlots = 8192;  // distinct ends per start (shared table)

struct BaseArgs {
  const uint32_t* adj;
  const uint32_t* mid;
  const uint32_t* end1;
  const uint32_t* ub;
  const uint64_t* work;
  uint32_t n, n_u;
  int rank, nranks;
  uint8_t* scratch;
  uint64_t per_cta;
  unsigned long long* acc;  // [0] balanced, [1] unbalanced, [2] start counter, [3] error flags
};

__device__ __forceinline__ uint32_t base_slot(uint32_t key, uint32_t mask) {
  return (key * 2654435761u >> 11) & mask;
}

// slot of key (inserting it when `insert`); 0xffffffff if the table is full
__device__ __forceinline__ uint32_t base_find(uint32_t* keys, uint32_t key, uint32_t mask, bool insert) {
  uint32_t h = base_slot(key, mask);
  for (uint32_t probes = 0; probes <= mask; ++probes) {
    uint32_t k = *reinterpret_cast<volatile uint32_t*>(&keys[h]);
    if (k == key) return h;
    if (k == 0 && insert) {
      k = atomicCAS(&keys[h], 0u, key);
      if (k == 0 || k == key) return h;
    }
    h = (h + 1) & mask;
  }
  return 0xffffffffu;
}

__global__ void __launch_bounds__(kBaseThreads) k_bb_base(const BaseArgs a) {
  extern __shared__ uint32_t smem[];
  uint32_t* keys = smem;              // end row + 1, 0 = empty
  uint32_t* cnt = keys + kBaseSlots;  // |H(w)|; the list cursor during sweep 2
  uint32_t* pos = cnt + kBaseSlots;   // list start in the scratch area
  __shared__ uint32_t sh_x, sh_err, sh_wsum[kBaseWarps];
  __shared__ unsigned long long sh_red[2][kBaseWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (uint32_t i = tid; i < kBaseSlots; i += kBaseThreads) { keys[i] = 0; cnt[i] = 0; }
  uint8_t* H = a.scratch + (uint64_t)blockIdx.x * a.per_cta;
  unsigned long long nb = 0, nn = 0;
  if (tid == 0) sh_err = 0;
  __syncthreads();
  while (true) {
    if (tid == 0) sh_x = (uint32_t)atomicAdd(&a.acc[2], 1ull);
    __syncthreads();
    const uint64_t xi = (uint64_t)sh_x * a.nranks + a.rank;
    if (xi >= a.n) break;
    const uint32_t x = (uint32_t)xi;
    const uint64_t W = a.work[x];
    if (W == 0 || W > a.per_cta) {  // (the host sizes per_cta to the largest start)
      if (W > a.per_cta && tid == 0) atomicOr(&sh_err, 2u);
      __syncthreads();
      continue;
    }
    const uint32_t ob = x < a.n_u ? a.n_u : 0;
    const uint32_t m_lo = a.mid[x], m_hi = a.end1[x];
    uint32_t S = 64;
    while (S < 2 * W && S < kBaseSlots) S <<= 1;
    const uint32_t mask = S - 1;
    // sweep 1 (lines 7-9): |H(w)|
    for (uint32_t e = m_lo + warp; e < m_hi; e += kBaseWarps) {
      const uint32_t wv = a.adj[e];
      const uint32_t en = a.end1[ob + (wv & kMask)];
      for (uint32_t p = a.ub[e] + lane; p < en; p += 32) {
        const uint32_t h = base_find(keys, (a.adj[p] & kMask) + 1, mask, true);
        if (h == 0xffffffffu) atomicOr(&sh_err, 1u);
        else atomicAdd(&cnt[h], 1u);
      }
    }
    __syncthreads();
    // list offsets: exclusive scan of cnt[0..S), one contiguous run of slots per thread
    {
      const uint32_t per = (S + kBaseThreads - 1) / kBaseThreads;
      const uint32_t i0 = min(S, tid * per), i1 = min(S, i0 + per);
      uint32_t loc = 0;
      for (uint32_t i = i0; i < i1; ++i) loc += cnt[i];
      uint32_t inc = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
      }
      if (lane == 31) sh_wsum[warp] = inc;
      __syncthreads();
      uint32_t base = 0;
      for (int w2 = 0; w2 < warp; ++w2) base += sh_wsum[w2];
      uint32_t run = base + inc - loc;
      for (uint32_t i = i0; i < i1; ++i) { pos[i] = run; run += cnt[i]; cnt[i] = 0; }
    }
    __syncthreads();
    // sweep 2 (line 9, H(w).add(v)): the two sign bits of each wedge in its end's list
    for (uint32_t e = m_lo + warp; e < m_hi; e += kBaseWarps) {
      const uint32_t wv = a.adj[e];
      const uint32_t en = a.end1[ob + (wv & kMask)];
      const uint32_t sxv = wv >> 31;  // 1 = negative (x, v)
      for (uint32_t p = a.ub[e] + lane; p < en; p += 32) {
        const uint32_t ew = a.adj[p];
        const uint32_t h = base_find(keys, (ew & kMask) + 1, mask, false);
        if (h == 0xffffffffu) continue;  // (table overflow, already flagged)
        H[pos[h] + atomicAdd(&cnt[h], 1u)] = (uint8_t)((sxv << 1) | (ew >> 31));
      }
    }
    __syncthreads();
    // lines 10-13: every pair of every list with |H(w)| > 1, checked one by one
    for (uint32_t sl = warp; sl < S; sl += kBaseWarps) {
      const uint32_t c = cnt[sl];
      if (c < 2) continue;
      const uint8_t* L = H + pos[sl];
      for (uint32_t q = lane; q < c / 2; q += 32) {
        const uint32_t r1 = q, r2 = c - 2 - q;  // triangle rows q and c-2-q: c-1 pairs together
#pragma unroll 1
        for (int k = 0; k < 2; ++k) {
          const uint32_t i = k ? r2 : r1;
          if (k && r2 <= r1) break;
          const uint32_t bi = L[i];
          for (uint32_t j = i + 1; j < c; ++j) {
            if (__popc(bi ^ L[j]) & 1u) ++nn;  // odd number of negative edges: unbalanced
            else ++nb;                         // is_Balanced
          }
        }
      }
    }
    __syncthreads();
    for (uint32_t i = tid; i < S; i += kBaseThreads) { keys[i] = 0; cnt[i] = 0; }
    __syncthreads();
  }
  for (int o = 16; o; o >>= 1) {
    nb += __shfl_xor_sync(0xffffffffu, nb, o);
    nn += __shfl_xor_sync(0xffffffffu, nn, o);
  }
  if (lane == 0) { sh_red[0][warp] = nb; sh_red[1][warp] = nn; }
  __syncthreads();
  if (warp == 0) {
    nb = sh_red[0][lane];
    nn = sh_red[1][lane];
    for (int o = 16; o; o >>= 1) {
      nb += __shfl_xor_sync(0xffffffffu, nb, o);
      nn += __shfl_xor_sync(0xffffffffu, nn, o);
    }
    if (lane == 0) {
      if (nb) atomicAdd(&a.acc[0], nb);
      if (nn) atomicAdd(&a.acc[1], nn);
      if (sh_err) atomicOr(&a.acc[3], (unsigned long long)sh_err);
    }
  }
}

}  // namespace

// Alg. 1 over this rank's share of the starts (start x on rank x mod nranks); host_BN receives
// this rank's (balanced, unbalanced).  Scratch: one area of max-work bytes per CTA.
bbf_status run_base(bbf_graph* g, Plan* p, int rank, int nranks, unsigned long long* host_BN) {
  NvtxRange nvtx_("bbf::bb_base");
  cudaStream_t st = g->stream;
  const uint32_t n = g->n;
  host_BN[0] = host_BN[1] = 0;
  if (!n) return BBF_OK;
  unsigned long long* d;  // acc[4] + max work
  BBF_CUDA(dmalloc(&d, 5 * sizeof(unsigned long long), st));
  BBF_CUDA(cudaMemsetAsync(d, 0, 5 * sizeof(unsigned long long), st));
  {
    size_t tb = 0;
    cub::DeviceReduce::Max(nullptr, tb, p->work, d + 4, (int)n, st);
    void* tmp;
    BBF_CUDA(dmalloc(&tmp, tb + 16, st));
    BBF_CUDA(cub::DeviceReduce::Max(tmp, tb, p->work, d + 4, (int)n, st));
    g->launches += kCubReduceKernels;
    dfree(tmp, st);
  }
  unsigned long long max_work = 0;
  BBF_CUDA(rb_add(&max_work, d + 4, 8, st)); g->launches++;
  BBF_CUDA(rb_sync(st));
  if (max_work == 0) { dfree(d, st); return BBF_OK; }
  const uint64_t budget = 8ull << 30;  // scratch bytes
  // the per-start list offsets (pos, cnt, the CTA scan) are 32-bit: a start's wedges must stay
  // below 2^32 as well as within the scratch
  if (max_work > budget || max_work >= (1ull << 32)) {
    dfree(d, st);
    set_error("BB-Base: a start has more wedges than the list scratch holds (8 GiB, 2^32 - 1 entries)");
    return BBF_ENOMEM;
  }
  const uint64_t per_cta = (max_work + 15) & ~15ull;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g->num_sms, budget / per_cta));
  uint8_t* scratch;
  BBF_CUDA(dmalloc(&scratch, per_cta * grid, st));
  BaseArgs a{};
  a.adj = g->adj; a.mid = g->mid; a.end1 = g->end1; a.ub = p->ub; a.work = p->work;
  a.n = n; a.n_u = g->n_u; a.rank = rank; a.nranks = nranks;
  a.scratch = scratch; a.per_cta = per_cta; a.acc = d;
  const int smem = (int)(3 * kBaseSlots * sizeof(uint32_t));
  BBF_CUDA(cudaFuncSetAttribute(k_bb_base, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_bb_base<<<grid, kBaseThreads, smem, st>>>(a);
  g->launches++;
  BBF_CUDA(cudaGetLastError());
  unsigned long long h[4] = {0, 0, 0, 0};
  BBF_CUDA(rb_add(h, d, sizeof(h), st)); g->launches++;
  BBF_CUDA(rb_sync(st));
  dfree(scratch, st);
  dfree(d, st);
  if (h[3] & 1u) {
    set_error("BB-Base: a start has more distinct ends than the 8,192-slot table holds");
    return BBF_EINVAL;
  }
  if (h[3] & 2u) {
    set_error("internal: BB-Base scratch smaller than a start's wedges");
    return BBF_ECUDA;
  }
  host_BN[0] = h[0];
  host_BN[1] = h[1];
  return BBF_OK;
}

}  // namespace bbf
