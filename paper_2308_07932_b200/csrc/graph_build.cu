// graph_build.cu — S1-S4 of the hot path: validate the input CSR, degrees,
// vertex priority ranks (Def. Vertex Priority), both-direction adjacency in
// rank space sorted by priority (Alg. 2 line 3) with the sign packed into bit 31,
// duplicate detection, and the per-row cut points mid_start / end1.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "bbf_internal.cuh"

namespace bbf {
namespace {

enum : uint32_t { kErrRowPtr = 1, kErrCol = 2, kErrSign = 4, kErrDup = 8 };

__global__ void k_validate_rows(const uint64_t* __restrict__ rp, uint32_t n_u, uint32_t* err) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i == 0 && rp[0] != 0) atomicOr(err, kErrRowPtr);
  if (i < n_u && rp[i + 1] < rp[i]) atomicOr(err, kErrRowPtr);
}

__global__ void k_validate_edges(const uint32_t* __restrict__ col, const uint8_t* __restrict__ sg,
                                 uint64_t nnz, uint32_t n_v, uint32_t* err) {
  uint32_t bad = 0;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (uint64_t)gridDim.x * blockDim.x) {
    if (col[e] >= n_v) bad |= kErrCol;
    if (sg[e] > 1) bad |= kErrSign;
  }
  if (bad) atomicOr(err, bad);
}

// priority sort items (Def. Vertex Priority: degree desc, then gid desc; gid: U -> u, V -> n_u + v,
// SPEC.md:100): the degree is the key, the gid the value, written in DESCENDING gid order so the
// stable radix sort by degree keeps equal degrees in descending gid order — a sort over the
// degree bits only instead of 64-bit (deg << 32 | gid) keys
__global__ void k_keys_u(const uint64_t* __restrict__ rp, uint32_t n_u, uint32_t* __restrict__ kdeg,
                         uint32_t* __restrict__ kid) {
  uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < n_u) {
    kdeg[n_u - 1 - u] = (uint32_t)(rp[u + 1] - rp[u]);
    kid[n_u - 1 - u] = u;
  }
}

// V-side degrees.  Hub columns of a power-law graph serialise plain global atomics on their
// counters (1.8 ms for config 5 vs 0.24 ms for uniform ids), so each CTA first aggregates a
// chunk of edges in a shared open-addressing table (kHistSlots keys, 2 probes; a column that
// finds no slot goes straight to global memory) and flushes one atomic per distinct column.
constexpr int kHistSlots = 4096, kHistThreads = 1024;
constexpr uint32_t kHistChunk = 65536;
__global__ void __launch_bounds__(kHistThreads) k_hist_v(const uint32_t* __restrict__ col, uint64_t nnz,
                                                         uint32_t* __restrict__ dv) {
  __shared__ uint32_t key[kHistSlots], cnt[kHistSlots];
  for (uint64_t c0 = (uint64_t)blockIdx.x * kHistChunk; c0 < nnz; c0 += (uint64_t)gridDim.x * kHistChunk) {
    for (int i = threadIdx.x; i < kHistSlots; i += kHistThreads) { key[i] = 0xffffffffu; cnt[i] = 0; }
    __syncthreads();
    const uint64_t c1 = c0 + kHistChunk < nnz ? c0 + kHistChunk : nnz;
    for (uint64_t e = c0 + threadIdx.x; e < c1; e += kHistThreads) {
      const uint32_t v = col[e];
      const uint32_t h = (v * 2654435761u) >> 20;  // 12 bits
      bool done = false;
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        if (done) break;
        const uint32_t s = (h + p) & (kHistSlots - 1);
        uint32_t k = key[s];
        if (k == 0xffffffffu) k = atomicCAS(&key[s], 0xffffffffu, v);
        if (k == 0xffffffffu || k == v) { atomicAdd(&cnt[s], 1u); done = true; }
      }
      if (!done) atomicAdd(&dv[v], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kHistSlots; i += kHistThreads)
      if (cnt[i]) atomicAdd(&dv[key[i]], cnt[i]);
    __syncthreads();
  }
}

// Narrow V sides (n_v <= kHistDirectMax): one persistent CTA per SM keeps a private counter per
// column in shared memory over its whole share of the edges and flushes the non-zero ones once
// (uniform columns defeat the 4096-slot table above: most edges would miss it and contend on
// the global counters)
constexpr uint32_t kHistDirectMax = 49152;
__global__ void __launch_bounds__(kHistThreads) k_hist_v_direct(const uint32_t* __restrict__ col, uint64_t nnz,
                                                                uint32_t n_v, uint32_t* __restrict__ dv) {
  extern __shared__ uint32_t hcnt[];
  for (uint32_t i = threadIdx.x; i < n_v; i += kHistThreads) hcnt[i] = 0;
  __syncthreads();
  for (uint64_t e = blockIdx.x * (uint64_t)kHistThreads + threadIdx.x; e < nnz; e += (uint64_t)gridDim.x * kHistThreads)
    atomicAdd(&hcnt[col[e]], 1u);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < n_v; i += kHistThreads)
    if (hcnt[i]) atomicAdd(&dv[i], hcnt[i]);
}

__global__ void k_keys_v(const uint32_t* __restrict__ dv, uint32_t n_u, uint32_t n_v,
                         uint32_t* __restrict__ kdeg, uint32_t* __restrict__ kid) {
  uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n_v) {
    kdeg[n_v - 1 - v] = dv[v];
    kid[n_v - 1 - v] = n_u + v;
  }
}

// sorted (degree desc, gid desc) items -> row tables: the priority key skey (deg << 32 | gid, for
// cross-side comparisons), inv (row -> input id), degs, lr (input id -> local rank)
__global__ void k_rank_tables(const uint32_t* __restrict__ sdeg, const uint32_t* __restrict__ sid, uint32_t cnt,
                              uint32_t id_base, uint32_t row_base, uint64_t* __restrict__ skey,
                              uint32_t* __restrict__ inv, uint32_t* __restrict__ degs, uint32_t* __restrict__ lr) {
  uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= cnt) return;
  const uint32_t d = sdeg[l], gid = sid[l], id = gid - id_base;
  skey[l] = ((uint64_t)d << 32) | gid;
  inv[row_base + l] = id;
  degs[row_base + l] = d;
  lr[id] = l;
}

// Rank-space adjacency in three stable passes ("Build"):
//   A  k_entries: each input row u is copied to its rank row lr_u[u] (keys = lr_v[v],
//      values = lr_u[u] | neg << 31), so the entries are in U-rank-major order;
//   B  a stable radix sort by V rank (bits(n_v) bits) groups them into V rows whose entries keep
//      the U-rank order: the values are the V-side adjacency (l | neg << 31) as is;
//   C  k_transpose_keys + a stable radix sort by U rank (bits(n_u) bits) gives the U rows with
//      their entries in V-rank order; its 8-byte values carry the U-side adjacency word and the
//      V-side position of the same edge, from which k_u_adj writes both directions' reverse
//      positions (rev: the plan's upper bound of a start in its middle's row is rev + 1).
// Two sorts of 4+4-byte items over ~bits(n_side) bits replace one sort of 8-byte keys over
// bits(n) + bits(n_side) + 1 bits (half the radix traffic).
__global__ void k_entries(const uint64_t* __restrict__ rp, const uint32_t* __restrict__ col,
                          const uint8_t* __restrict__ sg, uint64_t nnz, uint32_t n_u,
                          const uint32_t* __restrict__ lr_u, const uint32_t* __restrict__ lr_v,
                          const uint32_t* __restrict__ off, uint32_t* __restrict__ key,
                          uint32_t* __restrict__ val) {
  // one warp per input row (no per-edge row search)
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n_u; u += (gridDim.x * blockDim.x) >> 5) {
    const uint64_t b = rp[u], e1 = rp[u + 1];
    const uint32_t a = lr_u[u];
    const uint64_t d0 = off[a];
    for (uint64_t e = b + lane; e < e1; e += 32) {
      const uint32_t neg = sg[e] ? 0u : kNegBit;  // weight 0 = negative
      key[d0 + (e - b)] = lr_v[col[e]];
      val[d0 + (e - b)] = a | neg;
    }
  }
}

// after B: V-side rows (erow), and the inputs of C (key = U rank, value = the U-side adjacency
// word (V rank | neg) << 32 | the V-side position)
__global__ void k_transpose_keys(const uint32_t* __restrict__ vkey, const uint32_t* __restrict__ vadj,
                                 uint64_t nnz, uint32_t n_u, uint32_t* __restrict__ verow,
                                 uint32_t* __restrict__ key, uint64_t* __restrict__ val) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t l = vkey[i], w = vadj[i];
    verow[i] = n_u + l;
    key[i] = w & kMask;
    val[i] = ((uint64_t)(l | (w & kNegBit)) << 32) | (uint64_t)i;
  }
}

// after C: U entry i -> its adjacency word and the reverse positions of both entries of the
// edge (absolute indices into adj)
__global__ void k_u_adj(const uint64_t* __restrict__ val, uint64_t nnz, const uint32_t* __restrict__ erow,
                        uint32_t* __restrict__ adj, uint32_t* __restrict__ rev, uint32_t* err) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = val[i];
    const uint64_t r = nnz + (uint32_t)v;
    adj[i] = (uint32_t)(v >> 32);
    rev[i] = (uint32_t)r;
    rev[r] = (uint32_t)i;
    // duplicate (u, v) edges are adjacent in the sorted U rows
    if (i > 0 && erow[i] == erow[i - 1] && (((uint32_t)(v >> 32) ^ (uint32_t)(val[i - 1] >> 32)) & kMask) == 0)
      atomicOr(err, kErrDup);
  }
}

// number of entries of the descending array a[0..cnt) that are > key
__device__ __forceinline__ uint32_t count_greater(const uint64_t* __restrict__ a, uint32_t cnt,
                                                  uint64_t key) {
  uint32_t lo = 0, hi = cnt;
  while (lo < hi) {
    uint32_t mid = lo + (hi - lo) / 2;
    if (a[mid] > key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// first index in adj[b, e) whose masked column >= t
__device__ __forceinline__ uint32_t lower_bound_col(const uint32_t* __restrict__ adj, uint32_t b,
                                                    uint32_t e, uint32_t t) {
  while (b < e) {
    uint32_t mid = b + (e - b) / 2;
    if ((adj[mid] & kMask) < t) b = mid + 1; else e = mid;
  }
  return b;
}

// mid_start[x]: first neighbour with lower priority than x; end1[x]: first neighbour of degree<=1
__global__ void k_cuts(const uint32_t* __restrict__ off, const uint32_t* __restrict__ adj,
                       const uint64_t* __restrict__ skey_u, const uint64_t* __restrict__ skey_v,
                       uint32_t n_u, uint32_t n_v, uint32_t L4u, uint32_t L4v,
                       uint32_t* __restrict__ mid, uint32_t* __restrict__ end1) {
  uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n_u + n_v) return;
  bool is_u = x < n_u;
  uint64_t kx = is_u ? skey_u[x] : skey_v[x - n_u];
  uint32_t higher = is_u ? count_greater(skey_v, n_v, kx) : count_greater(skey_u, n_u, kx);
  uint32_t b = off[x], e = off[x + 1];
  mid[x] = lower_bound_col(adj, b, e, higher);
  end1[x] = lower_bound_col(adj, b, e, is_u ? L4v : L4u);
}

// number of entries of the non-increasing degs[base, base+cnt) that are >= t
__global__ void k_count_ge(const uint32_t* __restrict__ degs, uint32_t base, uint32_t cnt,
                           unsigned long long* out) {
  const uint32_t th[6] = {65536u, 256u, 16u, 4u, 2u, 33u};  // zones; 33: "long" middles (deg > 32)
  int t = threadIdx.x;
  if (t >= 6) return;
  uint32_t lo = 0, hi = cnt;
  while (lo < hi) {
    uint32_t mid = lo + (hi - lo) / 2;
    if (degs[base + mid] >= th[t]) lo = mid + 1; else hi = mid;
  }
  out[t] = lo;
}

// sum over vertices of C(deg, 2) per side (overflow pre-check)
__global__ void k_ws(const uint32_t* __restrict__ degs, uint32_t n_u, uint32_t n,
                     unsigned long long* out) {
  unsigned long long su = 0, sv = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    unsigned long long d = degs[i];
    if (i < n_u) su += comb2(d); else sv += comb2(d);
  }
  for (int o = 16; o; o >>= 1) {
    su += __shfl_xor_sync(0xffffffffu, su, o);
    sv += __shfl_xor_sync(0xffffffffu, sv, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&out[0], su);
    atomicAdd(&out[1], sv);
  }
}

__global__ void k_u32_to_u64(const uint32_t* __restrict__ a, uint32_t n, uint64_t* __restrict__ b) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}

// counter address of each entry's end vertex (entries [0, nnz) are U rows -> V ends)
// counter address of each entry's end, and the window-run start flags: an entry starts a run if
// it starts its row or its counter window differs from the previous entry's
__device__ __forceinline__ uint32_t caddr_of(uint32_t w, const Zones& z, bool compact) {
  return compact ? encode_caddr_compact(z, w & kMask, w >> 31) : encode_caddr(z, w & kMask) | (w & kNegBit);
}
__global__ void k_caddr(const uint32_t* __restrict__ adj, const uint32_t* __restrict__ erow, uint64_t m,
                        uint64_t nnz, Zones zu, Zones zv, bool compact, uint32_t wshift, uint32_t wmask,
                        uint32_t* __restrict__ adjc, uint32_t* __restrict__ flag) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const Zones& z = e < nnz ? zv : zu;
    const uint32_t c = caddr_of(adj[e], z, compact);
    adjc[e] = c;
    uint32_t f = 1u;
    if (e > 0 && erow[e] == erow[e - 1]) {
      const uint32_t cp = caddr_of(adj[e - 1], z, compact);
      f = ((c >> wshift) & wmask) / kWin != ((cp >> wshift) & wmask) / kWin ? 1u : 0u;
    }
    flag[e] = f;
  }
}

__global__ void k_rlast(const uint32_t* __restrict__ off, const uint32_t* __restrict__ end1,
                        const uint32_t* __restrict__ runid, uint32_t n, uint32_t* __restrict__ rlast) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x < n) rlast[x] = end1[x] > off[x] ? runid[end1[x] - 1] : 0u;
}

__global__ void k_runs(const uint32_t* __restrict__ adjc, const uint32_t* __restrict__ flag,
                       uint64_t m, uint32_t wshift, uint32_t wmask, const uint32_t* __restrict__ runid,
                       uint2* __restrict__ runs) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
       e += (uint64_t)gridDim.x * blockDim.x)
    if (e == 0 || flag[e]) runs[runid[e]] = make_uint2((uint32_t)e, ((adjc[e] >> wshift) & wmask) / kWin);
}

inline unsigned grid_for(uint64_t n, unsigned block, unsigned cap = 148u * 64u) {
  uint64_t g = (n + block - 1) / block;
  if (g == 0) g = 1;
  return (unsigned)std::min<uint64_t>(g, cap);
}

inline int bits_for(uint64_t x) {
  int b = 0;
  while ((1ull << b) <= x) ++b;
  return b;
}

// BBF_POSITIVE_ONLY compaction: keep[e] = edge e is positive; pos = exclusive prefix
__global__ void k_keep_pos(const uint8_t* __restrict__ sg, uint64_t nnz, uint32_t* __restrict__ keep) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (uint64_t)gridDim.x * blockDim.x)
    keep[e] = sg[e] == 1 ? 1u : 0u;
}
__global__ void k_pos_rows(const uint64_t* __restrict__ rp, uint32_t n_u, const uint32_t* __restrict__ pos,
                           uint64_t* __restrict__ nrp) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u <= n_u;
       u += (uint64_t)gridDim.x * blockDim.x)
    nrp[u] = pos[rp[u]];
}
__global__ void k_pos_compact(uint64_t nnz, const uint32_t* __restrict__ keep, const uint32_t* __restrict__ pos,
                              const uint32_t* __restrict__ col, const uint8_t* __restrict__ sg,
                              uint32_t* __restrict__ ncol, uint8_t* __restrict__ nsg) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (uint64_t)gridDim.x * blockDim.x)
    if (keep[e]) {
      ncol[pos[e]] = col[e];
      nsg[pos[e]] = sg[e];
    }
}

// Paper wedge count W_G of Alg. 2 in O(nnz), without the sorted adjacency: for a
// middle v, the eligible starts are its m_v neighbours of higher priority, and the k-th of them
// (k = 0.. in priority order) sees deg(v) - 1 - k eligible ends, so v contributes
// m_v (deg v - 1) - m_v (m_v - 1) / 2.  (Cross-checked against the plan's per-entry count.)
// one warp per U row: the row's own count (eligible starts v of middle u) is a warp sum written
// once; middle v's counter gets an atomic per eligible start u (consecutive edges of a row share
// u, so per-edge atomics on mcnt[u] would serialise inside the warp)
__global__ void k_wg_m(const uint64_t* __restrict__ rp, const uint32_t* __restrict__ col, uint32_t n_u,
                       const uint64_t* __restrict__ key_u, const uint64_t* __restrict__ key_v,
                       uint32_t* __restrict__ mcnt) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n_u; u += (gridDim.x * blockDim.x) >> 5) {
    const uint64_t ku = key_u[u];
    uint32_t c = 0;
    for (uint64_t e = rp[u] + lane; e < rp[u + 1]; e += 32) {
      const uint32_t v = col[e];
      if (ku > key_v[v]) atomicAdd(&mcnt[n_u + v], 1u);  // u is an eligible start for middle v
      else ++c;
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) mcnt[u] = c;
  }
}

// k_wg_m with the V-side middle counters in shared memory (n_v <= kHistDirectMax): one CTA per
// SM, warp per start row, flushed once per CTA
__global__ void __launch_bounds__(1024) k_wg_m_direct(const uint64_t* __restrict__ rp,
                                                      const uint32_t* __restrict__ col, uint32_t n_u,
                                                      uint32_t n_v, const uint64_t* __restrict__ key_u,
                                                      const uint64_t* __restrict__ key_v,
                                                      uint32_t* __restrict__ mcnt) {
  extern __shared__ uint32_t vcnt[];
  for (uint32_t i = threadIdx.x; i < n_v; i += blockDim.x) vcnt[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n_u; u += (gridDim.x * blockDim.x) >> 5) {
    const uint64_t ku = key_u[u];
    uint32_t c = 0;
    for (uint64_t e = rp[u] + lane; e < rp[u + 1]; e += 32) {
      const uint32_t v = col[e];
      if (ku > key_v[v]) atomicAdd(&vcnt[v], 1u);  // u is an eligible start for middle v
      else ++c;
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) mcnt[u] = c;
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < n_v; i += blockDim.x)
    if (vcnt[i]) atomicAdd(&mcnt[n_u + i], vcnt[i]);
}

// priority keys by input id (deg << 32 | gid) for the load-time W_G pass of a dense candidate
__global__ void k_keys64(const uint64_t* __restrict__ rp, const uint32_t* __restrict__ dv, uint32_t n_u, uint32_t n,
                         uint64_t* __restrict__ key) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t d = i < n_u ? rp[i + 1] - rp[i] : (uint64_t)dv[i - n_u];
  key[i] = (d << 32) | i;
}

__global__ void k_wg_sum(const uint32_t* __restrict__ mcnt, const uint64_t* __restrict__ key_u,
                         const uint64_t* __restrict__ key_v, uint32_t n_u, uint32_t n,
                         unsigned long long* __restrict__ out) {
  unsigned long long s = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned long long mv = mcnt[i];
    const unsigned long long d = (i < n_u ? key_u[i] : key_v[i - n_u]) >> 32;
    if (mv) s += mv * (d - 1ull) - mv * (mv - 1ull) / 2ull;
  }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

}  // namespace

// S1-S3 and the row offsets / zones; then either the rank-space adjacency (S4, sparse path) or,
// for a graph the dispatch rule sends to the dense path, the dense operands (adjacency deferred
// until a sparse call needs it; the input CSR is then kept on the device).
// S1 validation of a device CSR on its own (bbf_estimate_global validates its input once before
// any sampling kernel reads it): the same checks and status codes as the load.
bbf_status validate_csr(const uint64_t* d_rp, uint32_t n_u, const uint32_t* d_col, const uint8_t* d_sg,
                        uint64_t nnz, uint32_t n_v, cudaStream_t st) {
  uint32_t* d_err;
  BBF_CUDA(dmalloc(&d_err, 4, st));
  BBF_CUDA(cudaMemsetAsync(d_err, 0, 4, st));
  k_validate_rows<<<grid_for(n_u + 1, 256, 1u << 30), 256, 0, st>>>(d_rp, n_u, d_err);
  if (nnz) k_validate_edges<<<grid_for(nnz, 256), 256, 0, st>>>(d_col, d_sg, nnz, n_v, d_err);
  uint32_t h_err = 0;
  BBF_CUDA(rb_add(&h_err, d_err, 4, st));
  BBF_CUDA(rb_sync(st));
  dfree(d_err, st);
  if (h_err & kErrRowPtr) { set_error("row_ptr[0] != 0 or row_ptr not non-decreasing"); return BBF_ERANGE; }
  if (h_err & kErrCol) { set_error("col index >= n_v"); return BBF_ERANGE; }
  if (h_err & kErrSign) { set_error("sign byte not in {0,1}"); return BBF_EINVAL; }
  return BBF_OK;
}

bbf_status build_graph(bbf_graph* g, const uint64_t* row_ptr, const uint32_t* col,
                       const uint8_t* sign, bool device_ptrs) {
  NvtxRange nvtx_("bbf::build_graph");
  cudaStream_t st = g->stream;
  const uint32_t n_u = g->n_u, n_v = g->n_v, n = g->n;
  uint64_t nnz = g->nnz;  // the positive-only filter may reduce it
  // device copies of the input (S1)
  const uint64_t* d_rp = row_ptr;
  const uint32_t* d_col = col;
  const uint8_t* d_sg = sign;
  uint64_t* own_rp = nullptr;
  uint32_t* own_col = nullptr;
  uint8_t* own_sg = nullptr;
  if (!device_ptrs) {
    BBF_CUDA(dmalloc(&own_rp, sizeof(uint64_t) * (n_u + 1), st));
    BBF_CUDA(cudaMemcpyAsync(own_rp, row_ptr, sizeof(uint64_t) * (n_u + 1), cudaMemcpyHostToDevice, st));
    BBF_CUDA(dmalloc(&own_col, sizeof(uint32_t) * (nnz + 1), st));
    BBF_CUDA(dmalloc(&own_sg, nnz + 1, st));
    if (nnz) {
      BBF_CUDA(cudaMemcpyAsync(own_col, col, sizeof(uint32_t) * nnz, cudaMemcpyHostToDevice, st));
      BBF_CUDA(cudaMemcpyAsync(own_sg, sign, nnz, cudaMemcpyHostToDevice, st));
    }
    d_rp = own_rp; d_col = own_col; d_sg = own_sg;
  }
  auto cleanup_input = [&]() {
    if (own_rp) dfree(own_rp, st);
    if (own_col) dfree(own_col, st);
    if (own_sg) dfree(own_sg, st);
    own_rp = nullptr; own_col = nullptr; own_sg = nullptr;
  };
  uint32_t* d_err;
  BBF_CUDA(dmalloc(&d_err, 4 * sizeof(uint32_t), st));
  BBF_CUDA(cudaMemsetAsync(d_err, 0, 4 * sizeof(uint32_t), st));
  k_validate_rows<<<grid_for(n_u + 1, 256, 1u << 30), 256, 0, st>>>(d_rp, n_u, d_err);
  if (nnz) k_validate_edges<<<grid_for(nnz, 256), 256, 0, st>>>(d_col, d_sg, nnz, n_v, d_err);
  g->launches += 2;
  uint32_t h_err = 0;
  BBF_CUDA(rb_add(&h_err, d_err, 4, st)); g->launches++;
  BBF_CUDA(rb_sync(st));
  if (h_err) {
    dfree(d_err, st);
    cleanup_input();
    cudaStreamSynchronize(st);
    if (h_err & kErrRowPtr) { set_error("row_ptr[0] != 0 or row_ptr not non-decreasing"); return BBF_ERANGE; }
    if (h_err & kErrCol) { set_error("col index >= n_v"); return BBF_ERANGE; }
    set_error("sign byte not in {0,1}");
    return BBF_EINVAL;
  }
  dfree(d_err, st);

  // BBF_POSITIVE_ONLY: restrict to the positive edges (case-study analytics) before anything else
  if (g->positive_only && nnz) {
    uint32_t *keep, *pos, *pcol;
    uint64_t* prp;
    uint8_t* psg;
    BBF_CUDA(dmalloc(&keep, 4ull * (nnz + 1), st));
    BBF_CUDA(dmalloc(&pos, 4ull * (nnz + 1), st));
    BBF_CUDA(dmalloc(&prp, 8ull * (n_u + 1), st));
    BBF_CUDA(dmalloc(&pcol, 4ull * (nnz + 1), st));
    BBF_CUDA(dmalloc(&psg, nnz + 1, st));
    k_keep_pos<<<grid_for(nnz, 256), 256, 0, st>>>(d_sg, nnz, keep);
    BBF_CUDA(cudaMemsetAsync(keep + nnz, 0, 4, st));
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, keep, pos, (int64_t)(nnz + 1), st);
    void* tmp0;
    BBF_CUDA(dmalloc(&tmp0, tb + 16, st));
    BBF_CUDA(cub::DeviceScan::ExclusiveSum(tmp0, tb, keep, pos, (int64_t)(nnz + 1), st));
    k_pos_rows<<<grid_for(n_u + 1, 256, 1u << 30), 256, 0, st>>>(d_rp, n_u, pos, prp);
    k_pos_compact<<<grid_for(nnz, 256), 256, 0, st>>>(nnz, keep, pos, d_col, d_sg, pcol, psg);
    g->launches += 5;
    uint32_t kept = 0;
    BBF_CUDA(rb_add(&kept, pos + nnz, 4, st)); g->launches++;
    BBF_CUDA(rb_sync(st));
    dfree(tmp0, st);
    dfree(keep, st);
    dfree(pos, st);
    cleanup_input();
    own_rp = prp; own_col = pcol; own_sg = psg;
    d_rp = prp; d_col = pcol; d_sg = psg;
    g->nnz = kept;
    nnz = kept;
  }

  // S2-S3: degrees and per-side priority ranks
  uint32_t *key_u, *key_v;  // per side: degrees [0, cnt), gids [cnt, 2 cnt); sorted copies likewise
  uint32_t *skd_u, *skd_v;
  uint32_t* dv;
  BBF_CUDA(dmalloc(&key_u, 8ull * (n_u + 1), st));
  BBF_CUDA(dmalloc(&key_v, 8ull * (n_v + 1), st));
  BBF_CUDA(dmalloc(&skd_u, 8ull * (n_u + 1), st));
  BBF_CUDA(dmalloc(&skd_v, 8ull * (n_v + 1), st));
  BBF_CUDA(dmalloc(&g->skey, 8ull * (n + 1), st));
  BBF_CUDA(dmalloc(&dv, 4ull * (n_v + 1), st));
  BBF_CUDA(dmalloc(&g->lr, 4ull * (n + 1), st));
  BBF_CUDA(cudaMemsetAsync(dv, 0, 4ull * (n_v + 1), st));
  if (n_u) k_keys_u<<<grid_for(n_u, 256, 1u << 30), 256, 0, st>>>(d_rp, n_u, key_u, key_u + n_u);
  if (nnz) {
    const uint64_t chunks = (nnz + kHistChunk - 1) / kHistChunk;
    if (n_v <= kHistDirectMax) {
      const int smem = 4 * (int)n_v;
      if (smem > 48 * 1024)
        BBF_CUDA(cudaFuncSetAttribute(k_hist_v_direct, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      k_hist_v_direct<<<(unsigned)std::min<uint64_t>(chunks, g->num_sms), kHistThreads, smem, st>>>(d_col, nnz,
                                                                                                  n_v, dv);
    } else {
      k_hist_v<<<(unsigned)std::min<uint64_t>(chunks, 2ull * g->num_sms), kHistThreads, 0, st>>>(d_col, nnz, dv);
    }
  }
  if (n_v) k_keys_v<<<grid_for(n_v, 256, 1u << 30), 256, 0, st>>>(dv, n_u, n_v, key_v, key_v + n_v);
  g->launches += 3;
  uint64_t* skey_u = g->skey;
  uint64_t* skey_v = g->skey + n_u;
  uint32_t* lr_u = g->lr;
  uint32_t* lr_v = g->lr + n_u;

  size_t tmp_bytes = 0, t1 = 0, t2 = 0, t4 = 0;
  const int kbits = bits_for(std::max<uint64_t>(nnz, 1));  // degree <= nnz
  cub::DeviceRadixSort::SortPairsDescending(nullptr, t1, key_u, skd_u, key_u + n_u, skd_u + n_u, (int)n_u, 0, kbits, st);
  cub::DeviceRadixSort::SortPairsDescending(nullptr, t2, key_v, skd_v, key_v + n_v, skd_v + n_v, (int)n_v, 0, kbits, st);
  cub::DeviceScan::ExclusiveSum(nullptr, t4, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)(n + 1), st);
  tmp_bytes = std::max(std::max(t1, t2), t4);
  void* tmp;
  BBF_CUDA(dmalloc(&tmp, tmp_bytes + 16, st));
  if (n_u)
    BBF_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp, t1, key_u, skd_u, key_u + n_u, skd_u + n_u, (int)n_u, 0,
                                                        kbits, st));
  if (n_v)
    BBF_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp, t2, key_v, skd_v, key_v + n_v, skd_v + n_v, (int)n_v, 0,
                                                        kbits, st));
  g->launches += (n_u ? cub_sort_kernels(kbits) : 0) + (n_v ? cub_sort_kernels(kbits) : 0);

  BBF_CUDA(dmalloc(&g->inv, 4ull * (n + 1), st));
  BBF_CUDA(dmalloc(&g->degs, 4ull * (n + 1), st));
  BBF_CUDA(dmalloc(&g->off, 4ull * (n + 1), st));
  if (n_u)
    k_rank_tables<<<grid_for(n_u, 256, 1u << 30), 256, 0, st>>>(skd_u, skd_u + n_u, n_u, 0, 0, skey_u, g->inv, g->degs, lr_u);
  if (n_v)
    k_rank_tables<<<grid_for(n_v, 256, 1u << 30), 256, 0, st>>>(skd_v, skd_v + n_v, n_v, n_u, n_u, skey_v, g->inv, g->degs,
                                                                 lr_v);
  g->launches += 2;
  // row offsets: exclusive scan of degrees in row order (rows U by rank, then V by rank)
  BBF_CUDA(cudaMemsetAsync(g->degs + n, 0, 4, st));
  BBF_CUDA(cub::DeviceScan::ExclusiveSum(tmp, t4, g->degs, g->off, (int)(n + 1), st));
  g->launches += kCubScanKernels;
  dfree(tmp, st);

  // zone boundaries per side (rank counts of degree thresholds), overflow bound
  unsigned long long* d_cnt;
  BBF_CUDA(dmalloc(&d_cnt, 16 * sizeof(unsigned long long), st));
  BBF_CUDA(cudaMemsetAsync(d_cnt, 0, 16 * sizeof(unsigned long long), st));
  k_count_ge<<<1, 32, 0, st>>>(g->degs, 0, n_u, d_cnt);
  k_count_ge<<<1, 32, 0, st>>>(g->degs, n_u, n_v, d_cnt + 6);
  k_ws<<<grid_for(n, 256, 148 * 8), 256, 0, st>>>(g->degs, n_u, n, d_cnt + 12);
  g->launches += 3;
  unsigned long long h_cnt[16];
  BBF_CUDA(rb_add(h_cnt, d_cnt, sizeof(h_cnt), st)); g->launches++;
  uint32_t h_maxdeg[2] = {0, 0};
  if (n_u) { BBF_CUDA(rb_add(&h_maxdeg[0], g->degs, 4, st)); g->launches++; }
  if (n_v) { BBF_CUDA(rb_add(&h_maxdeg[1], g->degs + n_u, 4, st)); g->launches++; }
  BBF_CUDA(rb_sync(st));
  dfree(d_cnt, st);
  g->maxdeg[0] = h_maxdeg[0];
  g->maxdeg[1] = h_maxdeg[1];
  for (int s2 = 0; s2 < 2; ++s2) {
    Zones& z = g->zones[s2];
    for (int i = 0; i < 5; ++i) z.L[i] = (uint32_t)h_cnt[6 * s2 + i];
    g->Llong[s2] = (uint32_t)h_cnt[6 * s2 + 5];
    z.WB[0] = 0;
    z.WB[1] = 2u * z.L[0];
    z.WB[2] = z.WB[1] + (z.L[1] - z.L[0]);
    z.WB[3] = z.WB[2] + (z.L[2] - z.L[1] + 1) / 2;
    z.WB[4] = z.WB[3] + (z.L[3] - z.L[2] + 3) / 4;
    z.WB[5] = z.WB[4] + (z.L[4] - z.L[3] + 7) / 8;
    g->L4[s2] = z.L[4];
  }
  // B + N = sum_{u<w} C(T_uw, 2) <= (maxT - 1)/2 * sum_{u<w} T_uw = (maxdeg_U - 1)/2 * W_S(U)
  {
    long double bu = (long double)(g->maxdeg[0] ? g->maxdeg[0] - 1 : 0) / 2.0L * (long double)h_cnt[13];
    long double bv = (long double)(g->maxdeg[1] ? g->maxdeg[1] - 1 : 0) / 2.0L * (long double)h_cnt[12];
    g->ws_bound = std::min(bu, bv);
  }

  // dense candidates: W_G without the adjacency, then the dispatch rule decides the load path
  bool dense_load = false;
  if (dense_supported(g) && !(g->load_flags & BBF_FORCE_SPARSE)) {
    uint32_t* mcnt;
    unsigned long long* d_wg;
    uint64_t* key64;  // by input id: U keys [0, n_u), V keys [n_u, n)
    BBF_CUDA(dmalloc(&key64, 8ull * (n + 1), st));
    k_keys64<<<grid_for(n, 256, 1u << 30), 256, 0, st>>>(d_rp, dv, n_u, n, key64);
    g->launches += 1;
    const uint64_t* kk_u = key64;
    const uint64_t* kk_v = key64 + n_u;
    BBF_CUDA(dmalloc(&mcnt, 4ull * (n + 1), st));
    BBF_CUDA(dmalloc(&d_wg, 8, st));
    BBF_CUDA(cudaMemsetAsync(mcnt, 0, 4ull * (n + 1), st));
    BBF_CUDA(cudaMemsetAsync(d_wg, 0, 8, st));
    if (n_u && n_v <= kHistDirectMax) {
      const int smem = 4 * (int)n_v;
      if (smem > 48 * 1024)
        BBF_CUDA(cudaFuncSetAttribute(k_wg_m_direct, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      k_wg_m_direct<<<(unsigned)std::min<uint64_t>((n_u + 31) / 32, g->num_sms), 1024, smem, st>>>(
          d_rp, d_col, n_u, n_v, kk_u, kk_v, mcnt);
    } else if (n_u) {
      k_wg_m<<<grid_for(32ull * n_u, 256), 256, 0, st>>>(d_rp, d_col, n_u, kk_u, kk_v, mcnt);
    }
    if (n) k_wg_sum<<<grid_for(n, 256, 148 * 8), 256, 0, st>>>(mcnt, kk_u, kk_v, n_u, n, d_wg);
    g->launches += 2;
    unsigned long long wg = 0;
    BBF_CUDA(rb_add(&wg, d_wg, 8, st)); g->launches++;
    BBF_CUDA(rb_sync(st));
    dfree(mcnt, st);
    dfree(d_wg, st);
    dfree(key64, st);
    g->W_G = wg;
    g->wg_valid = true;
    g->dense_cand = true;
    dense_load = (g->load_flags & BBF_FORCE_DENSE) || dense_preferred(g, true);
  }
  dfree(key_u, st);
  dfree(key_v, st);
  dfree(skd_u, st);
  dfree(skd_v, st);
  dfree(dv, st);

  if (dense_load) {
    bbf_status s = build_dense_operands(g, d_rp, d_col, d_sg);
    if (s != BBF_OK) { cleanup_input(); cudaStreamSynchronize(st); return s; }
    // keep the input CSR for a later sparse call (build_adj); device inputs are only borrowed
    if (own_rp) {
      g->in_rp = own_rp; g->in_col = own_col; g->in_sg = own_sg;
      own_rp = nullptr; own_col = nullptr; own_sg = nullptr;
    } else {
      BBF_CUDA(dmalloc(&g->in_rp, sizeof(uint64_t) * (n_u + 1), st));
      BBF_CUDA(dmalloc(&g->in_col, sizeof(uint32_t) * (nnz + 1), st));
      BBF_CUDA(dmalloc(&g->in_sg, nnz + 1, st));
      BBF_CUDA(cudaMemcpyAsync(g->in_rp, d_rp, sizeof(uint64_t) * (n_u + 1), cudaMemcpyDeviceToDevice, st));
      if (nnz) {
        BBF_CUDA(cudaMemcpyAsync(g->in_col, d_col, 4ull * nnz, cudaMemcpyDeviceToDevice, st));
        BBF_CUDA(cudaMemcpyAsync(g->in_sg, d_sg, nnz, cudaMemcpyDeviceToDevice, st));
      }
    }
    BBF_CUDA(cudaGetLastError());
    return BBF_OK;
  }
  bbf_status s = build_adj(g, d_rp, d_col, d_sg);
  cleanup_input();
  return s;
}

bbf_status ensure_adj(bbf_graph* g) {
  if (g->adj_built) return BBF_OK;
  if (!g->in_rp) { set_error("internal: adjacency requested without the input CSR"); return BBF_ECUDA; }
  BBF_TRY(build_adj(g, g->in_rp, g->in_col, g->in_sg));
  return BBF_OK;
}

// S4: rank-space adjacency of both directions (one radix sort of the 2*nnz directed entries),
// duplicate check, mid_start / end1 cuts, degree prefix, hub-kernel counter addresses and runs
bbf_status build_adj(bbf_graph* g, const uint64_t* d_rp, const uint32_t* d_col, const uint8_t* d_sg) {
  NvtxRange nvtx_("bbf::build_adj");
  cudaStream_t st = g->stream;
  const uint32_t n_u = g->n_u, n_v = g->n_v, n = g->n;
  const uint64_t nnz = g->nnz;
  const uint64_t m = 2 * nnz;
  const uint64_t* skey_u = g->skey;
  const uint64_t* skey_v = g->skey + n_u;
  const uint32_t* lr_u = g->lr;
  const uint32_t* lr_v = g->lr + n_u;
  uint32_t* d_err;
  BBF_CUDA(dmalloc(&d_err, 4 * sizeof(uint32_t), st));
  BBF_CUDA(cudaMemsetAsync(d_err, 0, 4 * sizeof(uint32_t), st));
  size_t t3 = 0, t5 = 0;
  const int bits_u = bits_for(std::max<uint32_t>(n_u, 1)), bits_v = bits_for(std::max<uint32_t>(n_v, 1));
  size_t t3b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t3, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (int)nnz, 0, std::max(bits_u, bits_v), st);
  cub::DeviceRadixSort::SortPairs(nullptr, t3b, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint64_t*)nullptr,
                                  (uint64_t*)nullptr, (int)nnz, 0, std::max(bits_u, bits_v), st);
  t3 = std::max(t3, t3b);
  cub::DeviceScan::InclusiveSum(nullptr, t5, (uint64_t*)nullptr, (uint64_t*)nullptr, (int)n, st);
  void* tmp;
  BBF_CUDA(dmalloc(&tmp, std::max(t3, t5) + 16, st));
  BBF_CUDA(dmalloc(&g->mid, 4ull * (n + 1), st));
  BBF_CUDA(dmalloc(&g->end1, 4ull * (n + 1), st));
  BBF_CUDA(dmalloc(&g->adj, 4ull * (m + 1), st));
  BBF_CUDA(dmalloc(&g->erow, 4ull * (m + 1), st));
  BBF_CUDA(dmalloc(&g->rev, 4ull * (m + 1), st));
  BBF_CUDA(dmalloc(&g->degpre, 8ull * (n + 1), st));
  if (m) {
    uint32_t *ka, *va, *kb;
    uint64_t *wa, *wb;
    BBF_CUDA(dmalloc(&ka, 4ull * nnz, st));
    BBF_CUDA(dmalloc(&va, 4ull * nnz, st));
    BBF_CUDA(dmalloc(&kb, 4ull * nnz, st));
    BBF_CUDA(dmalloc(&wa, 8ull * nnz, st));
    BBF_CUDA(dmalloc(&wb, 8ull * nnz, st));
    k_entries<<<grid_for(32ull * n_u, 256), 256, 0, st>>>(d_rp, d_col, d_sg, nnz, n_u, lr_u, lr_v, g->off, ka, va);
    BBF_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t3, ka, kb, va, g->adj + nnz, (int)nnz, 0, bits_v, st));
    k_transpose_keys<<<grid_for(nnz, 256), 256, 0, st>>>(kb, g->adj + nnz, nnz, n_u, g->erow + nnz, ka, wa);
    BBF_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t3, ka, g->erow, wa, wb, (int)nnz, 0, bits_u, st));
    k_u_adj<<<grid_for(nnz, 256), 256, 0, st>>>(wb, nnz, g->erow, g->adj, g->rev, d_err);
    g->launches += 3 + cub_sort_kernels(bits_v) + cub_sort_kernels(bits_u);  // + k_entries, k_transpose_keys, k_u_adj
    dfree(ka, st);
    dfree(va, st);
    dfree(kb, st);
    dfree(wa, st);
    dfree(wb, st);
  }
  // the duplicate-edge flag is read back with the run count below (one host round trip): the
  // steps in between are harmless on a graph that turns out to be rejected
  g->rb_err = 0;
  BBF_CUDA(rb_add(&g->rb_err, d_err, 4, st)); g->launches++;
  dfree(d_err, st);
  if (m == 0) BBF_CUDA(rb_sync(st));
  if (n) {
    k_cuts<<<grid_for(n, 256, 1u << 30), 256, 0, st>>>(g->off, g->adj, skey_u, skey_v, n_u, n_v,
                                                      g->L4[0], g->L4[1], g->mid, g->end1);
    // inclusive prefix of degrees over rows (u64), used to split hub end-ranges by expected work
    uint64_t* d64;
    BBF_CUDA(dmalloc(&d64, 8ull * n, st));
    k_u32_to_u64<<<grid_for(n, 256, 1u << 30), 256, 0, st>>>(g->degs, n, d64);
    BBF_CUDA(cub::DeviceScan::InclusiveSum(tmp, t5, d64, g->degpre, (int)n, st));
    g->launches += 2 + kCubScanKernels;
    dfree(d64, st);
  }
  dfree(tmp, st);
  // hub-kernel counter addresses and window runs (DESIGN.md §"Counter windows")
  for (int s2 = 0; s2 < 2; ++s2)
    if (g->zones[s2].WB[5] > kCWordMask) {
      set_error("too many counter words on one side for the hub kernel's 23-bit address");
      return BBF_ERANGE;
    }
  g->compact = g->zones[0].L[0] == 0 && g->zones[1].L[0] == 0 && g->zones[0].WB[5] <= kCpWordMask &&
               g->zones[1].WB[5] <= kCpWordMask && !getenv("BBF_NO_COMPACT");  // env: test hook
  const uint32_t wmask = g->compact ? kCpWordMask : kCWordMask, wshift = g->compact ? 2u : 0u;
  BBF_CUDA(dmalloc(&g->adjc, 4ull * (m + 512), st));  // padded: chunk loads and the hub kernel's
  // long-record prefetch (count_sparse.cu kAdjcPad) may read past the last entry
  BBF_CUDA(dmalloc(&g->runid, 4ull * (m + 1), st));
  g->nruns = 0;
  if (m) {
    uint32_t* flag;
    BBF_CUDA(dmalloc(&flag, 4ull * (m + 1), st));
    k_caddr<<<grid_for(m, 256), 256, 0, st>>>(g->adj, g->erow, m, nnz, g->zones[0], g->zones[1], g->compact,
                                            wshift, wmask, g->adjc, flag);
    // entry 0 always starts a run: with its flag cleared the inclusive scan is the 0-based run index
    BBF_CUDA(cudaMemsetAsync(flag, 0, 4, st));
    size_t ts = 0;
    cub::DeviceScan::InclusiveSum(nullptr, ts, flag, g->runid, (int64_t)m, st);
    void* tmp2;
    BBF_CUDA(dmalloc(&tmp2, ts + 16, st));
    BBF_CUDA(cub::DeviceScan::InclusiveSum(tmp2, ts, flag, g->runid, (int64_t)m, st));
    BBF_CUDA(rb_add(&g->nruns, g->runid + (m - 1), 4, st)); g->launches++;
    BBF_CUDA(rb_sync(st));
    if (g->rb_err & kErrDup) {
      dfree(tmp2, st);
      dfree(flag, st);
      cudaStreamSynchronize(st);
      set_error("duplicate (u,v) edge");
      return BBF_EDUP;
    }
    g->nruns += 1;
    BBF_CUDA(dmalloc(&g->runs, sizeof(uint2) * (g->nruns + 1), st));
    k_runs<<<grid_for(m, 256), 256, 0, st>>>(g->adjc, flag, m, wshift, wmask, g->runid, g->runs);
    BBF_CUDA(dmalloc(&g->rlast, 4ull * (n + 1), st));
    if (n) k_rlast<<<(n + 255) / 256, 256, 0, st>>>(g->off, g->end1, g->runid, n, g->rlast);
    g->launches += 3 + kCubScanKernels;  // k_caddr, scan, k_runs, k_rlast
    dfree(tmp2, st);
    dfree(flag, st);
  } else {
    BBF_CUDA(dmalloc(&g->runs, sizeof(uint2), st));
    BBF_CUDA(dmalloc(&g->rlast, 4ull * (n + 1), st));
    BBF_CUDA(cudaMemsetAsync(g->rlast, 0, 4ull * (n + 1), st));
  }
  BBF_CUDA(cudaGetLastError());
  g->adj_built = true;
  return BBF_OK;
}

}  // namespace bbf
