// count_sparse.cu — S6-S8 of the hot path: sparse wedge aggregation on sm_100a.
//
// For a start x and each eligible middle v (Alg. 2 line 9) and end w
// (line 10) the wedge x-v-w is symmetric iff sigma(x,v) == sigma(v,w)
// (Def. Symmetric Wedge): with the sign in bit 31 of the column words this is
// cls = (e_xv ^ e_vw) >> 31 (0 = symmetric -> a / B1, 1 = asymmetric -> d / B2, lines 11-14).
// After all middles of x: balanced += C(a,2) + C(d,2) (lines 15-18, Lemma 2),
// unbalanced += a*d.
//
// Two kernels, chosen per start by its wedge count (plan.cu):
//   * k_t1 (<= 512 wedges): one warp per start, open-addressing hash of (end, a|d) in the
//     warp's shared-memory slice; wedges enumerated load-balanced over the warp lanes.
//   * k_t3 (hubs): one 1024-thread CTA per unit (start, end-rank range).  Counters are a dense
//     window of 48K shared-memory words over the end ranks, in degree zones (bbf_internal.cuh):
//     one shared atomic per wedge, a touched-word bitmap for the epilogue, and per-middle
//     cursors so each window streams only its slice of every middle's sorted list.
// Per-vertex counts (vBBFC semantics) use the 4-role scatter (DESIGN.md §"Per-vertex"): the
// start and the end get C(a,2)+C(d,2) / a*d of their pair, a middle of a symmetric wedge gets
// (a-1, d), of an asymmetric wedge (d-1, a) — pass 2 re-streams the window's wedges.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "bbf_internal.cuh"

namespace bbf {
namespace {

constexpr int kT3Threads = 1024;
constexpr uint32_t kWin = 48 * 1024;  // counter words per CTA window (192 KB)
constexpr uint32_t kBm = kWin / 32;   // bitmap words
constexpr uint32_t kLong = 64;        // middles with longer remaining segments go warp-wide
constexpr int kT1Warps = 12;
constexpr uint32_t kT1Slots = 1024;

struct EngineArgs {
  const uint32_t* off;
  const uint32_t* adj;
  const uint32_t* mid;   // route G middle start; nullptr for route S (off used)
  const uint32_t* end1;
  const uint32_t* ub;
  const uint64_t* work;
  const uint32_t* inv;
  const uint32_t* t1;
  const Unit* units;
  uint32_t n_t1, n_units;
  uint32_t n_u, n;
  Zones z[2];
  int rank, nranks;
  unsigned long long* acc;  // [0] B [1] N [2] unit cursor [3] t1 cursor [4] cand count
  unsigned long long* pv;   // [0, n) balanced per row, [n, 2n) unbalanced per row
  uint32_t* scratch;
  uint32_t max_mid;
  // pair candidates (top-k): balanced, unbalanced, (min id << 32 | max id)
  unsigned long long* cb;
  unsigned long long* cn;
  unsigned long long* cid;
  unsigned long long cap;
};

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void emit_pair(const EngineArgs& a, uint32_t x, uint32_t wrow,
                                          unsigned long long fb, unsigned long long fn) {
  unsigned long long slot = atomicAdd(&a.acc[4], 1ull);
  if (slot < a.cap) {
    unsigned long long ix = a.inv[x], iw = a.inv[wrow];
    unsigned long long lo = ix < iw ? ix : iw, hi = ix < iw ? iw : ix;
    a.cb[slot] = fb;
    a.cn[slot] = fn;
    a.cid[slot] = (lo << 32) | hi;
  }
}

// ===================================================================================== T3
template <bool PV, bool PAIRS>
__global__ void __launch_bounds__(kT3Threads, 1) k_t3(const EngineArgs a) {
  extern __shared__ uint32_t smem[];
  uint32_t* ctr = smem;         // kWin
  uint32_t* bm = smem + kWin;   // kBm
  __shared__ uint32_t sh_unit, sh_next, sh_nlong, sh_next2;
  __shared__ unsigned long long sh_red[2][32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = kT3Threads / 32;

  for (uint32_t i = tid; i < kWin + kBm; i += kT3Threads) smem[i] = 0;
  uint32_t* Sw = a.scratch + (size_t)blockIdx.x * 4 * a.max_mid;
  uint32_t* Scur = Sw + a.max_mid;
  uint32_t* Sold = Scur + a.max_mid;
  uint32_t* Send = Sold + a.max_mid;
  unsigned long long totB = 0, totN = 0;
  __syncthreads();

  while (true) {
    if (tid == 0) sh_unit = (uint32_t)atomicAdd(&a.acc[2], 1ull);
    __syncthreads();
    const uint64_t ui = (uint64_t)sh_unit * a.nranks + a.rank;
    if (ui >= a.n_units) break;
    const Unit u = a.units[ui];
    const uint32_t x = u.x;
    const bool xu = x < a.n_u;
    const uint32_t sb = xu ? 0 : a.n_u, ob = xu ? a.n_u : 0, lx = x - sb;
    const Zones& Z = a.z[xu ? 0 : 1];
    const uint32_t m_lo = a.mid ? a.mid[x] : a.off[x];
    const uint32_t m = a.end1[x] - m_lo;
    if (tid == 0) { sh_next = 0xffffffffu; sh_nlong = 0; sh_next2 = 0xffffffffu; }
    __syncthreads();
    // ---- unit setup: middle words, cursors (first end >= u.lo), segment ends, long list
    uint32_t my_min = 0xffffffffu;
    for (uint32_t i = tid; i < m; i += kT3Threads) {
      uint32_t e = m_lo + i;
      uint32_t wv = a.adj[e];
      uint32_t rv = ob + (wv & kMask);
      uint32_t s = a.ub[e], en = a.end1[rv];
      if (u.lo > lx + 1 && s < en) {  // binary search for the unit's first end rank
        uint32_t b = s, f = en;
        while (b < f) {
          uint32_t md = b + (f - b) / 2;
          if ((a.adj[md] & kMask) < u.lo) b = md + 1; else f = md;
        }
        s = b;
      }
      Sw[i] = wv;
      Scur[i] = s;
      Send[i] = en;
      if (s < en) {
        uint32_t l0 = a.adj[s] & kMask;
        if (l0 < my_min) my_min = l0;
      }
    }
    for (int o = 16; o; o >>= 1) my_min = min(my_min, __shfl_xor_sync(0xffffffffu, my_min, o));
    if (lane == 0 && my_min != 0xffffffffu) atomicMin(&sh_next, my_min);
    __syncthreads();
    uint32_t wl_lo = sh_next;
    unsigned long long xB = 0, xN = 0;

    while (wl_lo < u.hi) {
      const uint32_t word0 = word_of_l(Z, wl_lo);
      uint32_t wl_hi = l_first_last_word_ge(Z, (uint64_t)word0 + kWin);
      if (wl_hi > u.hi) wl_hi = u.hi;
      // ---------------- pass 1: count symmetric / asymmetric wedges per end (Alg. 2 l. 9-14)
      // a warp owns a chunk of 32 middles in both passes; short remaining segments are walked
      // one lane per middle, long ones by the whole warp (coalesced 128-B reads)
      uint32_t nmin = 0xffffffffu;
      for (uint32_t c = warp; c * 32 < m; c += nw) {
        const uint32_t i = c * 32 + lane;
        uint32_t cur = 0, en = 0, wv = 0;
        bool has = false, lng = false;
        if (i < m) {
          cur = Scur[i]; en = Send[i]; wv = Sw[i];
          has = cur < en;
          lng = has && (en - cur > kLong);
        }
        const uint32_t old = cur;
        if (has && !lng) {
          uint32_t l = 0xffffffffu;
          while (cur < en) {
            uint32_t ev = a.adj[cur];
            l = ev & kMask;
            if (l >= wl_hi) break;
            uint32_t base, word, inc;
            field_of(Z, l, (ev ^ wv) >> 31, base, word, inc);
            uint32_t prev = atomicAdd(&ctr[word - word0], inc);
            if (prev == 0) atomicOr(&bm[(base - word0) >> 5], 1u << ((base - word0) & 31));
            ++cur;
          }
          if (cur < en) nmin = min(nmin, l);
        }
        uint32_t lmask = __ballot_sync(0xffffffffu, lng);
        while (lmask) {
          const int j = __ffs(lmask) - 1;
          lmask &= lmask - 1;
          uint32_t jc = __shfl_sync(0xffffffffu, cur, j);
          const uint32_t je = __shfl_sync(0xffffffffu, en, j);
          const uint32_t jw = __shfl_sync(0xffffffffu, wv, j);
          while (true) {
            uint32_t idx = jc + lane;
            uint32_t ev = idx < je ? a.adj[idx] : 0xffffffffu;
            uint32_t l = ev & kMask;
            bool in = idx < je && l < wl_hi;
            if (in) {
              uint32_t base, word, inc;
              field_of(Z, l, (ev ^ jw) >> 31, base, word, inc);
              uint32_t prev = atomicAdd(&ctr[word - word0], inc);
              if (prev == 0) atomicOr(&bm[(base - word0) >> 5], 1u << ((base - word0) & 31));
            }
            uint32_t cnt = __popc(__ballot_sync(0xffffffffu, in));
            uint32_t lnext = __shfl_sync(0xffffffffu, l, cnt & 31);
            jc += cnt;
            if (cnt < 32) {
              if (jc < je) nmin = min(nmin, lnext);
              break;
            }
          }
          if (lane == j) cur = jc;
        }
        if (i < m) { Sold[i] = old; Scur[i] = cur; }
      }
      for (int o = 16; o; o >>= 1) nmin = min(nmin, __shfl_xor_sync(0xffffffffu, nmin, o));
      if (lane == 0 && nmin != 0xffffffffu) atomicMin(&sh_next2, nmin);
      __syncthreads();
      const uint32_t next_lo = sh_next2;
      __syncthreads();
      if (tid == 0) sh_next2 = 0xffffffffu;

      // ---------------- pass 2: middles' per-vertex shares from the final (a, d) of each end
      if (PV) {
        for (uint32_t c = warp; c * 32 < m; c += nw) {
          const uint32_t i = c * 32 + lane;
          uint32_t old = 0, cur = 0, wv = 0;
          if (i < m) { old = Sold[i]; cur = Scur[i]; wv = Sw[i]; }
          const bool lng = cur - old > kLong;
          if (!lng && cur > old) {
            unsigned long long cb = 0, cn = 0;
            for (uint32_t p = old; p < cur; ++p) {
              uint32_t ev = a.adj[p];
              uint32_t ad, dd;
              field_read(Z, ctr, word0, ev & kMask, ad, dd);
              if (((ev ^ wv) >> 31) == 0) { cb += ad - 1; cn += dd; }
              else { cb += dd - 1; cn += ad; }
            }
            if (cb | cn) {
              uint32_t vr = ob + (wv & kMask);
              atomicAdd(&a.pv[vr], cb);
              atomicAdd(&a.pv[a.n + vr], cn);
            }
          }
          uint32_t lmask = __ballot_sync(0xffffffffu, lng);
          while (lmask) {
            const int j = __ffs(lmask) - 1;
            lmask &= lmask - 1;
            const uint32_t jo = __shfl_sync(0xffffffffu, old, j);
            const uint32_t jc = __shfl_sync(0xffffffffu, cur, j);
            const uint32_t jw = __shfl_sync(0xffffffffu, wv, j);
            unsigned long long b2 = 0, n2 = 0;
            for (uint32_t p = jo + lane; p < jc; p += 32) {
              uint32_t ev = a.adj[p];
              uint32_t ad, dd;
              field_read(Z, ctr, word0, ev & kMask, ad, dd);
              if (((ev ^ jw) >> 31) == 0) { b2 += ad - 1; n2 += dd; }
              else { b2 += dd - 1; n2 += ad; }
            }
            b2 = warp_sum(b2);
            n2 = warp_sum(n2);
            if (lane == 0 && (b2 | n2)) {
              uint32_t vr = ob + (jw & kMask);
              atomicAdd(&a.pv[vr], b2);
              atomicAdd(&a.pv[a.n + vr], n2);
            }
          }
        }
        __syncthreads();
      }

      // ---------------- epilogue: Lemma 2 per touched end, clear the window
      for (uint32_t bw = tid; bw < kBm; bw += kT3Threads) {
        uint32_t bits = bm[bw];
        if (!bits) continue;
        bm[bw] = 0;
        while (bits) {
          uint32_t j = __ffs(bits) - 1;
          bits &= bits - 1;
          uint32_t wi = bw * 32 + j;
          uint32_t gw = word0 + wi;
          uint32_t v = ctr[wi];
          ctr[wi] = 0;
          uint32_t nf, fbits, lbase;
          uint32_t av[8], dv[8];
          if (gw < Z.WB[1]) {  // zone 0: (a word, d word)
            av[0] = v;
            dv[0] = ctr[wi + 1];
            ctr[wi + 1] = 0;
            nf = 1; fbits = 64; lbase = gw >> 1;
          } else if (gw < Z.WB[2]) {
            av[0] = v & 0xffffu; dv[0] = v >> 16; nf = 1; fbits = 32; lbase = Z.L[0] + (gw - Z.WB[1]);
          } else if (gw < Z.WB[3]) {
            nf = 2; fbits = 16; lbase = Z.L[1] + 2 * (gw - Z.WB[2]);
            for (int f = 0; f < 2; ++f) { uint32_t q = (v >> (16 * f)) & 0xffffu; av[f] = q & 0xffu; dv[f] = q >> 8; }
          } else if (gw < Z.WB[4]) {
            nf = 4; fbits = 8; lbase = Z.L[2] + 4 * (gw - Z.WB[3]);
            for (int f = 0; f < 4; ++f) { uint32_t q = (v >> (8 * f)) & 0xffu; av[f] = q & 0xfu; dv[f] = q >> 4; }
          } else {
            nf = 8; fbits = 4; lbase = Z.L[3] + 8 * (gw - Z.WB[4]);
            for (int f = 0; f < 8; ++f) { uint32_t q = (v >> (4 * f)) & 0xfu; av[f] = q & 3u; dv[f] = q >> 2; }
          }
          (void)fbits;
          for (uint32_t f = 0; f < nf; ++f) {
            unsigned long long A = av[f], D = dv[f];
            if (!(A | D)) continue;
            unsigned long long fb = comb2(A) + comb2(D), fn = A * D;
            if (!(fb | fn)) continue;
            xB += fb;
            xN += fn;
            uint32_t wrow = sb + lbase + f;
            if (PV) {
              atomicAdd(&a.pv[wrow], fb);
              atomicAdd(&a.pv[a.n + wrow], fn);
            }
            if (PAIRS && fb) emit_pair(a, x, wrow, fb, fn);
          }
        }
      }
      __syncthreads();
      wl_lo = next_lo;
    }
    // unit totals -> start vertex
    totB += xB;
    totN += xN;
    if (PV) {
      unsigned long long b = warp_sum(xB), nn = warp_sum(xN);
      if (lane == 0) { sh_red[0][warp] = b; sh_red[1][warp] = nn; }
      __syncthreads();
      if (warp == 0) {
        b = sh_red[0][lane];
        nn = sh_red[1][lane];
        b = warp_sum(b);
        nn = warp_sum(nn);
        if (lane == 0 && (b | nn)) {
          atomicAdd(&a.pv[x], b);
          atomicAdd(&a.pv[a.n + x], nn);
        }
      }
    }
    __syncthreads();
  }
  totB = warp_sum(totB);
  totN = warp_sum(totN);
  if (lane == 0 && (totB | totN)) {
    atomicAdd(&a.acc[0], totB);
    atomicAdd(&a.acc[1], totN);
  }
}

// ===================================================================================== T1
__device__ __forceinline__ uint32_t hslot(uint32_t l, uint32_t mask) {
  return (l * 0x9E3779B1u) >> 16 & mask;
}

template <bool PV, bool PAIRS>
__global__ void __launch_bounds__(kT1Warps * 32) k_t1(const EngineArgs a) {
  extern __shared__ uint32_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  volatile uint32_t* keys = smem + warp * (2 * kT1Slots + 3 * 32 + 64);
  uint32_t* vals = (uint32_t*)keys + kT1Slots;
  uint32_t* sh_incl = vals + kT1Slots;
  uint32_t* sh_s = sh_incl + 32;
  uint32_t* sh_wv = sh_s + 32;
  uint32_t* sh_mb = sh_wv + 32;  // 32 balanced partials (u32)
  uint32_t* sh_mn = sh_mb + 32;  // 32 unbalanced partials (u32)
  for (uint32_t i = lane; i < 2 * kT1Slots; i += 32) ((uint32_t*)keys)[i] = 0;
  if (lane < 32) { sh_mb[lane] = 0; sh_mn[lane] = 0; }
  __syncwarp();
  unsigned long long totB = 0, totN = 0;
  while (true) {
    unsigned long long q = 0;
    if (lane == 0) q = atomicAdd(&a.acc[3], 1ull);
    q = __shfl_sync(0xffffffffu, q, 0);
    const uint64_t ti = q * a.nranks + a.rank;
    if (ti >= a.n_t1) break;
    const uint32_t x = a.t1[ti];
    const bool xu = x < a.n_u;
    const uint32_t sb = xu ? 0 : a.n_u, ob = xu ? a.n_u : 0;
    const uint32_t m_lo = a.mid ? a.mid[x] : a.off[x];
    const uint32_t m = a.end1[x] - m_lo;
    const uint32_t W = (uint32_t)a.work[x];
    uint32_t S = 32;
    while (S < 2 * W && S < kT1Slots) S <<= 1;
    const uint32_t mask = S - 1;
    // ---- pass 1: enumerate wedges middle-chunk by middle-chunk, load-balanced over lanes
    for (int pass = 0; pass < (PV ? 2 : 1); ++pass) {
      for (uint32_t cb = 0; cb < m; cb += 32) {
        uint32_t i = cb + lane;
        uint32_t wv = 0, s = 0, len = 0;
        if (i < m) {
          wv = a.adj[m_lo + i];
          s = a.ub[m_lo + i];
          uint32_t en = a.end1[ob + (wv & kMask)];
          len = en > s ? en - s : 0;
        }
        uint32_t incl = len;
        for (int o = 1; o < 32; o <<= 1) {
          uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
        if (tot == 0) continue;
        sh_incl[lane] = incl;
        sh_s[lane] = s;
        sh_wv[lane] = wv;
        __syncwarp();
        for (uint32_t t = lane; t < tot + 31 - (tot + 31) % 32; t += 32) {
          bool act = t < tot;
          if (act) {
            uint32_t lo = 0, hi = 31;  // first j with incl[j] > t
            while (lo < hi) {
              uint32_t md = (lo + hi) >> 1;
              if (sh_incl[md] > t) hi = md; else lo = md + 1;
            }
            uint32_t j = lo;
            uint32_t excl = j ? sh_incl[j - 1] : 0;
            uint32_t ev = a.adj[sh_s[j] + (t - excl)];
            uint32_t l = ev & kMask;
            uint32_t cls = (ev ^ sh_wv[j]) >> 31;
            uint32_t key = l + 1;
            uint32_t h = hslot(l, mask);
            if (pass == 0) {
              while (true) {
                uint32_t k = keys[h];
                if (k == key) break;
                if (k == 0) {
                  k = atomicCAS((uint32_t*)&keys[h], 0u, key);
                  if (k == 0 || k == key) break;
                }
                h = (h + 1) & mask;
              }
              atomicAdd(&vals[h], cls ? 65536u : 1u);
            } else {
              while (keys[h] != key) h = (h + 1) & mask;
              uint32_t v = vals[h];
              uint32_t ad = v & 0xffffu, dd = v >> 16;
              uint32_t b2 = cls ? dd - 1 : ad - 1, n2 = cls ? ad : dd;
              if (b2) atomicAdd(&sh_mb[j], b2);
              if (n2) atomicAdd(&sh_mn[j], n2);
            }
          }
        }
        __syncwarp();
        if (pass == 1) {
          uint32_t b2 = sh_mb[lane], n2 = sh_mn[lane];
          if (b2 | n2) {
            uint32_t vr = ob + (wv & kMask);
            atomicAdd(&a.pv[vr], (unsigned long long)b2);
            atomicAdd(&a.pv[a.n + vr], (unsigned long long)n2);
          }
          sh_mb[lane] = 0;
          sh_mn[lane] = 0;
        }
        __syncwarp();
      }
    }
    // ---- epilogue: Lemma 2 per end, clear
    unsigned long long xB = 0, xN = 0;
    for (uint32_t k = lane; k < S; k += 32) {
      uint32_t key = keys[k];
      if (!key) continue;
      uint32_t v = vals[k];
      keys[k] = 0;
      vals[k] = 0;
      unsigned long long A = v & 0xffffu, D = v >> 16;
      unsigned long long fb = comb2(A) + comb2(D), fn = A * D;
      if (!(fb | fn)) continue;
      xB += fb;
      xN += fn;
      uint32_t wrow = sb + key - 1;
      if (PV) {
        atomicAdd(&a.pv[wrow], fb);
        atomicAdd(&a.pv[a.n + wrow], fn);
      }
      if (PAIRS && fb) emit_pair(a, x, wrow, fb, fn);
    }
    __syncwarp();
    totB += xB;
    totN += xN;
    if (PV) {
      xB = warp_sum(xB);
      xN = warp_sum(xN);
      if (lane == 0 && (xB | xN)) {
        atomicAdd(&a.pv[x], xB);
        atomicAdd(&a.pv[a.n + x], xN);
      }
    }
  }
  totB = warp_sum(totB);
  totN = warp_sum(totN);
  if (lane == 0 && (totB | totN)) {
    atomicAdd(&a.acc[0], totB);
    atomicAdd(&a.acc[1], totN);
  }
}

template <bool PV, bool PAIRS>
cudaError_t launch_engine(bbf_graph* g, const EngineArgs& ea, cudaStream_t st, Plan* p,
                          cudaEvent_t e0, cudaEvent_t e1, cudaEvent_t e2) {
  const size_t smem3 = sizeof(uint32_t) * (kWin + kBm);
  const size_t smem1 = sizeof(uint32_t) * kT1Warps * (2 * kT1Slots + 3 * 32 + 64);
  cudaError_t err;
  err = cudaFuncSetAttribute(k_t3<PV, PAIRS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3);
  if (err != cudaSuccess) return err;
  err = cudaFuncSetAttribute(k_t1<PV, PAIRS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
  if (err != cudaSuccess) return err;
  cudaEventRecord(e0, st);
  if (p->n_units) {
    k_t3<PV, PAIRS><<<g->num_sms, kT3Threads, smem3, st>>>(ea);
    g->launches++;
  }
  cudaEventRecord(e1, st);
  if (p->n_t1) {
    k_t1<PV, PAIRS><<<g->num_sms * 2, kT1Warps * 32, smem1, st>>>(ea);
    g->launches++;
  }
  cudaEventRecord(e2, st);
  return cudaGetLastError();
}

}  // namespace

bbf_status run_sparse_impl(bbf_graph* g, Plan* p, bool per_vertex, bool pairs, int rank,
                           int nranks, unsigned long long* host_BN, unsigned long long* cb,
                           unsigned long long* cn, unsigned long long* cid,
                           unsigned long long cap, unsigned long long* n_cand) {
  cudaStream_t st = g->stream;
  // scratch for the hub kernel's middle arrays
  size_t need = (size_t)g->num_sms * 4 * std::max<uint32_t>(p->max_mid, 1);
  if (need > g->scratch_words) {
    if (g->scratch) cudaFree(g->scratch);
    g->scratch = nullptr;
    BBF_CUDA(cudaMalloc(&g->scratch, need * sizeof(uint32_t)));
    g->scratch_words = need;
  }
  BBF_CUDA(cudaMemsetAsync(g->d_acc, 0, 16 * sizeof(unsigned long long), st));
  EngineArgs ea{};
  ea.off = g->off; ea.adj = g->adj; ea.mid = p->route == 0 ? g->mid : nullptr; ea.end1 = g->end1;
  ea.ub = p->ub; ea.work = p->work; ea.inv = g->inv; ea.t1 = p->t1; ea.units = p->units;
  ea.n_t1 = p->n_t1; ea.n_units = p->n_units; ea.n_u = g->n_u; ea.n = g->n;
  ea.z[0] = g->zones[0]; ea.z[1] = g->zones[1];
  ea.rank = rank; ea.nranks = nranks;
  ea.acc = g->d_acc; ea.pv = (unsigned long long*)g->pv; ea.scratch = g->scratch;
  ea.max_mid = std::max<uint32_t>(p->max_mid, 1);
  ea.cb = cb; ea.cn = cn; ea.cid = cid; ea.cap = cap;
  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
  cudaError_t err;
  if (pairs) err = launch_engine<false, true>(g, ea, st, p, e0, e1, e2);
  else if (per_vertex) err = launch_engine<true, false>(g, ea, st, p, e0, e1, e2);
  else err = launch_engine<false, false>(g, ea, st, p, e0, e1, e2);
  if (err != cudaSuccess) {
    cudaEventDestroy(e0); cudaEventDestroy(e1); cudaEventDestroy(e2);
    return cuda_status(err, "sparse engine launch");
  }
  unsigned long long h[8];
  BBF_CUDA(cudaMemcpyAsync(h, g->d_acc, sizeof(h), cudaMemcpyDeviceToHost, st));
  BBF_CUDA(cudaStreamSynchronize(st));
  float ms1 = 0, ms2 = 0;
  cudaEventElapsedTime(&ms1, e0, e1);
  cudaEventElapsedTime(&ms2, e1, e2);
  cudaEventDestroy(e0); cudaEventDestroy(e1); cudaEventDestroy(e2);
  g->ms_main = ms1;
  host_BN[0] = h[0];
  host_BN[1] = h[1];
  if (n_cand) *n_cand = h[4];
  // algorithmic bytes of the hub kernel k_t3: 4 B column word per
  // visited wedge per pass (pass 2 re-reads it for per-vertex counts) + 16 B per eligible
  // middle of its starts (column word, ub, end1 of the middle's row, 4 B id-side output)
  g->algo_bytes = 4ull * p->W_t3 * (per_vertex ? 2 : 1) + 16ull * p->M_t3;
  return BBF_OK;
}

bbf_status run_sparse(bbf_graph* g, Plan* p, bool per_vertex, int rank, int nranks,
                      unsigned long long* host_BN) {
  return run_sparse_impl(g, p, per_vertex, false, rank, nranks, host_BN, nullptr, nullptr, nullptr,
                         0, nullptr);
}

}  // namespace bbf

namespace bbf {
namespace {
__global__ void k_iota(uint32_t* a, unsigned long long n) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    a[i] = (uint32_t)i;
}
__global__ void k_gather_u64(const unsigned long long* __restrict__ src, const uint32_t* __restrict__ idx,
                             unsigned long long n, unsigned long long* __restrict__ dst) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}
}  // namespace

// S11: top-k same-side pairs by balanced count (route S on `side`, every unordered pair once).
// Order: balanced desc, then smaller input id asc, then larger input id asc (reading R11) —
// two stable radix sorts (ids ascending, then balanced descending).  Every rank computes the
// full candidate set (top-k is requested only on small graphs).
bbf_status run_pairs_topk(bbf_graph* g, int side, uint32_t k, bbf_pair* out, uint32_t* n_out) {
  cudaStream_t st = g->stream;
  Plan* p = &g->plan_s[side];
  if (!p->valid) BBF_TRY(make_plan(g, 1 + side, p));
  unsigned long long cap = std::min<unsigned long long>(p->W_pruned + 1024, 1ull << 24);
  unsigned long long ncand = 0;
  unsigned long long *cb = nullptr, *cn = nullptr, *cid = nullptr;
  for (int attempt = 0; attempt < 2; ++attempt) {
    BBF_CUDA(cudaMallocAsync(&cb, 8 * cap, st));
    BBF_CUDA(cudaMallocAsync(&cn, 8 * cap, st));
    BBF_CUDA(cudaMallocAsync(&cid, 8 * cap, st));
    unsigned long long BN[2];
    BBF_TRY(run_sparse_impl(g, p, false, true, 0, 1, BN, cb, cn, cid, cap, &ncand));
    if (ncand <= cap) break;
    cudaFreeAsync(cb, st); cudaFreeAsync(cn, st); cudaFreeAsync(cid, st);
    cap = ncand + 1024;
    if (attempt == 1) { set_error("top-k candidate buffer overflow"); return BBF_ENOMEM; }
  }
  uint32_t take = (uint32_t)std::min<unsigned long long>(k, ncand);
  *n_out = take;
  if (take == 0) {
    cudaFreeAsync(cb, st); cudaFreeAsync(cn, st); cudaFreeAsync(cid, st);
    BBF_CUDA(cudaStreamSynchronize(st));
    return BBF_OK;
  }
  const int nc = (int)ncand;
  uint32_t *idx0, *idx1, *idx2;
  unsigned long long *kid, *kb, *kb2;
  BBF_CUDA(cudaMallocAsync(&idx0, 4ull * nc, st));
  BBF_CUDA(cudaMallocAsync(&idx1, 4ull * nc, st));
  BBF_CUDA(cudaMallocAsync(&idx2, 4ull * nc, st));
  BBF_CUDA(cudaMallocAsync(&kid, 8ull * nc, st));
  BBF_CUDA(cudaMallocAsync(&kb, 8ull * nc, st));
  BBF_CUDA(cudaMallocAsync(&kb2, 8ull * nc, st));
  k_iota<<<256, 256, 0, st>>>(idx0, ncand);
  size_t t1 = 0, t2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t1, cid, kid, idx0, idx1, nc, 0, 64, st);
  cub::DeviceRadixSort::SortPairsDescending(nullptr, t2, kb, kb2, idx1, idx2, nc, 0, 64, st);
  void* tmp;
  BBF_CUDA(cudaMallocAsync(&tmp, std::max(t1, t2) + 16, st));
  BBF_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t1, cid, kid, idx0, idx1, nc, 0, 64, st));
  k_gather_u64<<<256, 256, 0, st>>>(cb, idx1, ncand, kb);
  BBF_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp, t2, kb, kb2, idx1, idx2, nc, 0, 64, st));
  g->launches += 6;
  // gather the first `take`
  k_gather_u64<<<64, 256, 0, st>>>(cid, idx2, take, kid);
  k_gather_u64<<<64, 256, 0, st>>>(cn, idx2, take, kb);
  std::vector<unsigned long long> hb(take), hn(take), hid(take);
  BBF_CUDA(cudaMemcpyAsync(hb.data(), kb2, 8ull * take, cudaMemcpyDeviceToHost, st));
  BBF_CUDA(cudaMemcpyAsync(hid.data(), kid, 8ull * take, cudaMemcpyDeviceToHost, st));
  BBF_CUDA(cudaMemcpyAsync(hn.data(), kb, 8ull * take, cudaMemcpyDeviceToHost, st));
  BBF_CUDA(cudaStreamSynchronize(st));
  for (uint32_t i = 0; i < take; ++i) {
    out[i].a = (uint32_t)(hid[i] >> 32);
    out[i].b = (uint32_t)(hid[i] & 0xffffffffu);
    out[i].balanced = hb[i];
    out[i].unbalanced = hn[i];
  }
  void* fr[] = {cb, cn, cid, idx0, idx1, idx2, kid, kb, kb2, tmp};
  for (void* q : fr) cudaFreeAsync(q, st);
  BBF_CUDA(cudaStreamSynchronize(st));
  return BBF_OK;
}

}  // namespace bbf
