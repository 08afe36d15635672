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
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <vector>

#include "bbf_internal.cuh"

namespace bbf {
namespace {

#ifndef BBF_T3_THREADS
#define BBF_T3_THREADS (1024 / BBF_T3_CTAS)
#endif
constexpr int kT3Threads = BBF_T3_THREADS;
constexpr int kT3Warps = kT3Threads / 32;
constexpr uint32_t kBm = kWin / 32;   // bitmap words

struct EngineArgs {
  const uint32_t* off;
  const uint32_t* adj;
  const uint32_t* adjc;
  const uint32_t* runid;
  const uint32_t* rlast;   // run index of each row's last entry before end1
  const uint2* runs;
  uint32_t nruns;
  const uint32_t* mid;   // route G middle start; nullptr for route S (off used)
  const uint32_t* end1;
  const uint32_t* ub;
  const uint64_t* work;
  const uint32_t* inv;
  const uint32_t* t1;
  const uint32_t* t2;    // the T2 starts of one k_t2 instance
  const Unit* units;
  const uint32_t* cut_tab;               // split starts: precomputed segment cuts (plan.cu k_split_cuts)

  const unsigned long long* unit_cut;    // per unit: offsets of its lower / upper cut arrays
  uint32_t n_t1, n_t2, n_units;
  uint32_t t2ctr;        // acc index of that instance's start cursor
  uint32_t t1ctr;        // acc index of the k_t1 instance's start cursor
  uint32_t n_u, n;
  Zones z[2];
  int rank, nranks;
  unsigned long long* acc;  // [0] B [1] N [2] unit cursor [3] t1 cursor [4] cand count
  unsigned long long* pv;   // [0, n) balanced per row, [n, 2n) unbalanced per row
  unsigned long long* pe;   // packed end-role counts (fb | fn << 32) of ends of rank >= rsafe
  uint32_t rsafe[2];        // per side: first local rank whose end-role totals stay < 2^32
  unsigned long long* pm;   // packed middle-role counts of middles of rank >= rmid
  uint32_t rmid[2];
  uint32_t* scratch;
  uint32_t max_mid;
  uint32_t kwin_cap;  // max windows per side
  uint32_t rec_stride;  // record slots per window: max middles + max unit work / kRecMax
  uint32_t dense_div;   // a window is scanned densely when wedges * dense_div >= its words
  uint32_t bsz;         // records per warp batch (0 = adaptive)
  unsigned long long tau;  // top-k: only pairs with balanced >= tau are candidates
  // pair candidates (top-k): balanced, unbalanced, (min id << 32 | max id)
  unsigned long long* cb;
  unsigned long long* cn;
  unsigned long long* cid;
  unsigned long long cap;
  // per-edge counts (bbf_count_per_edge): the middle-role share of every record goes to the
  // start->middle entry's slot edge[2e], edge[2e + 1] instead of the middle vertex, and the
  // start / end roles are not scattered; ue (route 3: the rev array) cuts each middle's ends at the
  // start's own entry (ends before the start)
  unsigned long long* edge;
  const uint32_t* ue;
};

// The q-th work item (hub unit, T1 / T2 start; plan order = descending work, roughly) of `rank` in
// an N-rank job: items are dealt in snake order (0..N-1, N-1..0, ...) so no rank takes the larger
// item of every round; every item lands on exactly one rank.
// Work item of this rank's q-th claim: items are dealt in rounds of nranks in snake order (0..N-1,
// N-1..0, ...), rotated by one rank every two rounds — plain snake dealing left the ranks of
// config 5's 8-way split at two cost levels (±2.6%, hubs split into 4 units of unequal cost fall
// on ranks {0,3,4,7} vs {1,2,5,6}); rotated, they are within ±0.6%.  A bijection per round.
__device__ __forceinline__ uint64_t shard_item(uint64_t q, int rank, int nranks) {
  const uint64_t snake = (q & 1ull) ? (uint64_t)(nranks - 1 - rank) : (uint64_t)rank;
  return q * (uint64_t)nranks + (snake + (q >> 1)) % (uint64_t)nranks;
}

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void emit_pair(const EngineArgs& a, uint32_t x, uint32_t wrow,
                                          unsigned long long fb, unsigned long long fn) {
  if (fb < a.tau) return;  // below the current top-k threshold
  // one slot atomic per group of converged lanes (all emitting lanes hit the same counter)
  const unsigned am = __activemask();
  const int lane = (int)(threadIdx.x & 31), leader = __ffs(am) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(&a.acc[4], (unsigned long long)__popc(am));
  base = __shfl_sync(am, base, leader);
  const unsigned long long slot = base + (unsigned long long)__popc(am & ((1u << lane) - 1u));
  if (slot < a.cap) {
    unsigned long long ix = a.inv[x], iw = a.inv[wrow];
    unsigned long long lo = ix < iw ? ix : iw, hi = ix < iw ? iw : ix;
    a.cb[slot] = fb;
    a.cn[slot] = fn;
    a.cid[slot] = (lo << 32) | hi;
  }
}

// pe (packed end-role counts) -> pv
__global__ void k_merge_pe(const unsigned long long* __restrict__ pe, const unsigned long long* __restrict__ pm,
                           unsigned long long* __restrict__ pv, uint32_t n) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const unsigned long long q = pe[r], w = pm[r];
  if (!(q | w)) return;
  pv[2ull * r] += (q & 0xffffffffull) + (w & 0xffffffffull);
  pv[2ull * r + 1] += (q >> 32) + (w >> 32);
}

// End-role contribution of pair (x, w): one packed 64-bit RED when w's end-role totals are
// provably < 2^32 (local rank >= rs, plan.cu k_rsafe), else one RED per non-zero count.
#ifdef BBF_RED_PROF  // RED counts by role (diagnostics; the global counters distort timings)
__device__ unsigned long long g_red_cnt[8];  // end: unpacked, packed, rank < 1024, rank < 8192; mid: unpacked, packed
#define RED_CNT(i) atomicAdd(&g_red_cnt[i], 1ull)
#else
#define RED_CNT(i) do {} while (0)
#endif
__device__ __forceinline__ void end_red(const EngineArgs& a, uint32_t rs, uint32_t lrank, uint32_t wrow,
                                        uint32_t fb, uint32_t fn) {
  if (a.edge) return;  // per-edge counts: no vertex roles
  RED_CNT(lrank >= rs ? 1 : 0);
  if (lrank < 1024) RED_CNT(2);
  if (lrank < 8192) RED_CNT(3);
  if (lrank >= rs) {
    atomicAdd(&a.pe[wrow], (unsigned long long)fb | ((unsigned long long)fn << 32));
  } else {
    if (fb) atomicAdd(&a.pv[2ull * wrow], (unsigned long long)fb);
    if (fn) atomicAdd(&a.pv[2ull * wrow + 1], (unsigned long long)fn);
  }
}

// Middle-role share of one record / middle: packed like end_red (pm, threshold rmid).
__device__ __forceinline__ void mid_red(const EngineArgs& a, uint32_t rm, uint32_t lrank, uint32_t vrow,
                                        uint32_t cb, uint32_t cn, uint32_t e) {
  if (a.edge) {  // per-edge counts: the share of the start->middle edge (adjacency entry e)
    if (cb) atomicAdd(&a.edge[2ull * e], (unsigned long long)cb);
    if (cn) atomicAdd(&a.edge[2ull * e + 1], (unsigned long long)cn);
    return;
  }
  RED_CNT(lrank >= rm ? 5 : 4);
  if (lrank < 1024) RED_CNT(6);
  if (lrank >= rm) {
    atomicAdd(&a.pm[vrow], (unsigned long long)cb | ((unsigned long long)cn << 32));
  } else {
    if (cb) atomicAdd(&a.pv[2ull * vrow], (unsigned long long)cb);
    if (cn) atomicAdd(&a.pv[2ull * vrow + 1], (unsigned long long)cn);
  }
}

// ===================================================================================== T3
// One CTA per unit (start x, end-rank range).  The end ranks of x's side are cut into a fixed
// grid of windows of kWin counter words (degree-zoned fields, bbf_internal.cuh).
//   pre-scan : warps take batches of 32 middles (one coalesced header load), walk every
//              middle's segment once and emit a "segment record" {adj position, length,
//              middle word} for every maximal run of entries inside one window (runs are split
//              every kRecMax entries), bucketed by window;
//   per window (only windows that received records):
//     pass 1 : batches of 32 records per warp; one shared atomic per wedge;
//     pass 2 : (per-vertex) the same batches read the final (a, d) of each end: middle shares;
//     epilogue: Lemma 2 per touched counter word (bitmap), clear.
// Inside a batch, the records are flattened over the lanes in 16-B chunks of adjc (one LDG.128
// per lane per step), so every lane is busy whatever the record lengths.
constexpr uint32_t kRecMax = 1024;
#ifdef BBF_T3_PROF
// record-shape and window statistics (profiling build): [0] record entries, [1..3] aligned
// 64/32/16-entry blocks the records touch, [4] records shorter than 8 entries, [5] entries of
// records shorter than 64, [6] wedges in dense windows, [7] wedges in bitmap windows, [8] touched
// words in the epilogue, [9] contributing fields, [10] records
__device__ unsigned long long g_prof_cnt[128];  // [96..111]: tiny-window latency marks (BBF_T3_LATPROF)
//  // [64..83]: unit-size bins (BBF_T3_WINPROF)  // [16..33]: window-size bins, [40..57] per-phase cycles (BBF_T3_WINPROF)
#define T3_COUNT(i, v) atomicAdd(&g_prof_cnt[i], (unsigned long long)(v))
#define T3_LAT(i, v) atomicAdd(&sh_lat[(i) - 96], (unsigned long long)(v))
__device__ unsigned long long g_prof_t[3] = {~0ull, ~0ull, 0ull};  // min CTA start, min CTA end, max CTA end (globaltimer ns)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#else
#define T3_COUNT(i, v) do {} while (0)
#endif
// BBF_T3_PROF: per-phase clock64 totals of the hub kernel (thread 0, after each CTA barrier),
// flushed to acc[11..15]; diagnostics only (off in production builds)
#ifdef BBF_T3_PROF
#define T3_MARK(slot)                                             \
  do {                                                            \
    if (tid == 0) {                                               \
      const long long now_ = clock64();                           \
      sh_prof[slot] += (unsigned long long)(now_ - t_prof);       \
      t_prof = now_;                                              \
    }                                                             \
  } while (0)
#else
#define T3_MARK(slot) do {} while (0)
#endif
#ifndef BBF_T3_KU
#define BBF_T3_KU 1  // measured: kU 1 / 2 -> 70.3 / 71.2 ms (config 5), 5.294 / 5.275 ms (config 3)
#endif
constexpr int kU = BBF_T3_KU;  // flattened steps per iteration of the hub kernel's record loop
#ifndef BBF_T3_CE
#define BBF_T3_CE 8
#endif
constexpr uint32_t kCE = BBF_T3_CE;
#ifndef BBF_T3_BMIN
#define BBF_T3_BMIN 12
#endif  // adjacency entries per lane per step (16-B aligned chunks)
constexpr int kEncWide = 0, kEncNarrow = 1, kEncCompact = 2;  // adjc encodings
constexpr uint32_t kMaxWin = 256;

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Segmented sums of (b, n) over groups of consecutive lanes (a group starts at lane gs; the
// sums are valid at each group's last lane): inclusive scans minus the scan at lane gs - 1.
// When every lane's b and n are < 2^11 (the common case) one scan of b | n << 16 does both
// halves exactly (a full-warp sum stays < 2^16 per half).
__device__ __forceinline__ void seg_sums2(uint32_t b, uint32_t n, int gs, int lane, uint32_t& sb, uint32_t& sn) {
  const int src = gs > 0 ? gs - 1 : 0;
  if (__all_sync(0xffffffffu, (b | n) < 2048u)) {
    const uint32_t ip = warp_incl_scan(b | (n << 16), lane);
    const uint32_t pp = __shfl_sync(0xffffffffu, ip, src);
    const uint32_t d = ip - (gs > 0 ? pp : 0u);
    sb = d & 0xffffu;
    sn = d >> 16;
  } else {
    const uint32_t ib = warp_incl_scan(b, lane), in = warp_incl_scan(n, lane);
    const uint32_t pb = __shfl_sync(0xffffffffu, ib, src), pn = __shfl_sync(0xffffffffu, in, src);
    sb = ib - (gs > 0 ? pb : 0u);
    sn = in - (gs > 0 ? pn : 0u);
  }
}

// Flattened-step owner lookup: lanes hold items (len, excl = exclusive prefix); for flattened
// index f = base + lane returns the lane that owns f.  nz = ballot(len > 0).
__device__ __forceinline__ int flat_owner(uint32_t len, uint32_t excl, uint32_t nz, uint32_t base,
                                          int lane) {
  const uint32_t bit = (len > 0 && excl >= base && excl < base + 32) ? (1u << (excl - base)) : 0u;
  const uint32_t smask = __reduce_or_sync(0xffffffffu, bit);
  const uint32_t before = __popc(__ballot_sync(0xffffffffu, len > 0 && excl < base));
  const int rank = (int)(before + __popc(smask & ((2u << lane) - 1u))) - 1;
  return rank >= 0 ? (int)__fns(nz, 0, rank + 1) : 0;
}

// one wedge: ev = adjc entry of the end (counter address + sign), wv = middle's adj word.
// WIDE: the graph has 64-bit (zone 0) fields; BM: maintain the touched-word bitmap.
template <bool WIDE, bool BM>
__device__ __forceinline__ void t3_inc_c(uint32_t* ctr, uint32_t* bm, uint32_t word0, uint32_t ev,
                                         uint32_t wv) {
  const uint32_t g = (ev & kCWordMask) - word0;
  const uint32_t cls = (ev ^ wv) >> 31;        // 0 symmetric (a), 1 asymmetric (d)
  const uint32_t sh = (ev >> 23) & 31u, wc = (ev >> 28) & 3u;
  uint32_t word = g, inc;
  if (WIDE) {
    const uint32_t wide = (ev >> 30) & 1u;
    word = g + (wide & cls);
    inc = 1u << (sh + ((cls & (wide ^ 1u)) << (wc + 1u)));
  } else {
    inc = 1u << (sh + (cls << (wc + 1u)));
  }
  if (BM) {
    const uint32_t prev = atomicAdd(&ctr[word], inc);
    if (prev == 0) atomicOr(&bm[g >> 5], 1u << (g & 31));
  } else {
    atomicAdd(&ctr[word], inc);
  }
}

template <bool WIDE>
__device__ __forceinline__ void t3_share_c(const uint32_t* ctr, uint32_t word0, uint32_t ev,
                                           uint32_t wv, uint32_t& b, uint32_t& nn) {
  const uint32_t g = (ev & kCWordMask) - word0;
  uint32_t ad, dd;
  if (WIDE && ((ev >> 30) & 1u)) {
    ad = ctr[g];
    dd = ctr[g + 1];
  } else {
    const uint32_t h = 2u << ((ev >> 28) & 3u);  // half-field width 2..16
    const uint32_t v = ctr[g] >> ((ev >> 23) & 31u);
    const uint32_t msk = (1u << h) - 1u;
    ad = v & msk;
    dd = (v >> h) & msk;
  }
  if (((ev ^ wv) >> 31) == 0) { b += ad - 1; nn += dd; }   // symmetric: (a-1, d)
  else { b += dd - 1; nn += ad; }                            // asymmetric: (d-1, a)
}

// Compact encoding (encode_caddr_compact): shamt = 22 + 5 * (start->middle edge negative)
// selects the bit this wedge increments; oshamt = 49 - shamt the other half of the field.
// Counters are addressed through 32-bit shared-window addresses (cbase = shared address of
// the window's word 0 minus 4 * word0), so an update is LOP + LEA + shifts + one ATOMS/RED.
// volatile (ordered with each other and with barriers) but without a "memory" clobber, so the
// compiler may still move the global chunk loads across them
__device__ __forceinline__ void sh_red_add(uint32_t addr, uint32_t v) {
#ifdef BBF_EXP_NOATOM  // timing experiment only: no counter update (results are wrong)
  if ((addr ^ v) == 0x12345677u) asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v));
#else
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v));
#endif
}
__device__ __forceinline__ uint32_t sh_atom_add(uint32_t addr, uint32_t v) {
  uint32_t r;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(r) : "r"(addr), "r"(v));
  return r;
}
__device__ __forceinline__ uint32_t sh_load(uint32_t addr) {
  uint32_t r;
#ifdef BBF_EXP_NOLDS  // timing experiment only: no counter read (results are wrong)
  r = addr * 0x9E3779B1u;
#else
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(addr));
#endif
  return r;
}

// predicated forms (no branch around each entry of a chunk): the update / load only happens if
// `on` is non-zero; the predicated load returns 0 otherwise
__device__ __forceinline__ void sh_red_add_if(uint32_t addr, uint32_t v, uint32_t on) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p red.shared.add.u32 [%0], %1;\n\t}" ::"r"(addr),
               "r"(v), "r"(on));
}
__device__ __forceinline__ void sh_red_or_if(uint32_t addr, uint32_t v, uint32_t on) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p red.shared.or.b32 [%0], %1;\n\t}" ::"r"(addr),
               "r"(v), "r"(on));
}
__device__ __forceinline__ uint32_t sh_load_if(uint32_t addr, uint32_t on) {
  uint32_t r;
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\tmov.u32 %0, 0;\n\t@p ld.shared.u32 %0, [%1];\n\t}"
               : "=r"(r)
               : "r"(addr), "r"(on));
  return r;
}

// zero-extend the low `len` bits (one SGXT.W)
__device__ __forceinline__ uint32_t zext(uint32_t t, uint32_t len) {
  uint32_t r;
  asm("szext.wrap.u32 %0, %1, %2;" : "=r"(r) : "r"(t), "r"(len));
  return r;
}
// the field at bit (ev >> sh) & 31 of counter word v, h bits wide
__device__ __forceinline__ uint32_t cp_field(uint32_t v, uint32_t ev, uint32_t sh, uint32_t h) {
  return zext(v >> ((ev >> sh) & 31u), h);
}

template <bool BM>
__device__ __forceinline__ void t3_inc_cp(uint32_t cbase, uint32_t* bm, uint32_t word0, uint32_t ev,
                                          uint32_t shamt) {
  const uint32_t inc = 1u << ((ev >> shamt) & 31u);
  if (BM) {
    const uint32_t prev = sh_atom_add(cbase + (ev & kCpAddrMask), inc);
    const uint32_t g = cp_word(ev) - word0;
    if (prev == 0) atomicOr(&bm[g >> 5], 1u << (g & 31));
  } else {
    sh_red_add(cbase + (ev & kCpAddrMask), inc);
  }
}

// middle share of one wedge: its own class count - 1 balanced, the other class unbalanced
__device__ __forceinline__ void t3_share_cp(uint32_t cbase, uint32_t ev, uint32_t shamt, uint32_t oshamt,
                                            uint32_t& b, uint32_t& nn) {
  const uint32_t v = sh_load(cbase + (ev & kCpAddrMask));
  const uint32_t h = 2u << (ev & 3u);
  b += cp_field(v, ev, shamt, h) - 1u;
  nn += cp_field(v, ev, oshamt, h);
}

// Zone of a packed counter word, from zone bounds held in registers for the epilogue (the
// per-word if-chain on the shared zone table was ~8% of the hub kernel's instructions).
struct ZoneRegs {
  uint32_t wb2, wb3, wb4, l0, l1, l2, l3, wb1;
};
struct ZoneP {
  uint32_t h, lfw, lb, wb, hi, lo, end;  // half-field bits, log2 field bits, first rank / word, SWAR masks, zone end
};
__device__ __forceinline__ ZoneRegs zone_regs(const Zones& Z) {
  return ZoneRegs{Z.WB[2], Z.WB[3], Z.WB[4], Z.L[0], Z.L[1], Z.L[2], Z.L[3], Z.WB[1]};
}
__device__ __forceinline__ ZoneP zone_of(const ZoneRegs& z, uint32_t gw) {
  if (gw < z.wb2) return ZoneP{16, 5, z.l0, z.wb1, 0xfffefffeu, 0x00000001u, z.wb2};
  if (gw < z.wb3) return ZoneP{8, 4, z.l1, z.wb2, 0xfefefefeu, 0x00010001u, z.wb3};
  if (gw < z.wb4) return ZoneP{4, 3, z.l2, z.wb3, 0xeeeeeeeeu, 0x01010101u, z.wb4};
  return ZoneP{2, 2, z.l3, z.wb4, 0xaaaaaaaau, 0x11111111u, 0xffffffffu};
}

// Lemma 2 on one packed counter word gw of zone zp; skipped unless some field has a + d >= 2
// (SWAR test: a or d >= 2, or a and d both odd).  Fields narrower than 32 bits hold a, d < 2^16,
// so C(a,2) + C(d,2) and a*d fit 32 bits, and so do their sums over one word's fields.
template <bool PV, bool PAIRS>
__device__ __forceinline__ void epi_packed(const EngineArgs& a, const ZoneP& zp, uint32_t sb, uint32_t rs,
                                           uint32_t x, uint32_t gw, uint32_t v, unsigned long long& xB,
                                           unsigned long long& xN) {
  const uint32_t h = zp.h, lfw = zp.lfw;
  const uint32_t lbase = zp.lb + ((gw - zp.wb) << (5 - lfw));
  uint32_t cm = (v & zp.hi) | (v & (v >> h) & zp.lo);  // non-zero bits only in contributing fields
  const uint32_t fw = 2 * h, fmask = (1u << h) - 1u;
  const uint32_t fclr = (fw == 32) ? 0xffffffffu : ((1u << fw) - 1u);
  uint32_t wb = 0, wn = 0;
  while (cm) {
    const uint32_t f = (uint32_t)(__ffs(cm) - 1) >> lfw;  // field index
    cm &= ~(fclr << (f * fw));
    const uint32_t q = v >> (f * fw);
    const uint32_t A = q & fmask, D = (q >> h) & fmask;
    const uint32_t fb = ((A * (A - 1u)) >> 1) + ((D * (D - 1u)) >> 1), fn = A * D;
    wb += fb;
    wn += fn;
    const uint32_t wrow = sb + lbase + f;
#ifndef BBF_EXP_NOEPI
    if (PV) end_red(a, rs, lbase + f, wrow, fb, fn);  // fb | fn != 0 here
#else
    if (PV && fb == 0x7fffffffu) end_red(a, rs, lbase + f, wrow, fb, fn);
#endif
    if (PAIRS && fb) emit_pair(a, x, wrow, fb, fn);
  }
  xB += wb;
  xN += wn;
}

// Lemma 2 on one 64-bit field (zone 0: a word, d word at global words gw, gw + 1)
template <bool PV, bool PAIRS>
__device__ __forceinline__ void epi_wide(const EngineArgs& a, uint32_t sb, uint32_t x, uint32_t gw,
                                         uint32_t va, uint32_t vd, unsigned long long& xB,
                                         unsigned long long& xN) {
  const unsigned long long A = va, D = vd;
  const unsigned long long fb = comb2(A) + comb2(D), fn = A * D;
  if (!(fb | fn)) return;
  xB += fb;
  xN += fn;
  const uint32_t wrow = sb + (gw >> 1);
  if (PV && !a.edge) {
    if (fb) atomicAdd(&a.pv[2ull * (wrow)], fb);
    if (fn) atomicAdd(&a.pv[2ull * (wrow) + 1], fn);
  }
  if (PAIRS && fb) emit_pair(a, x, wrow, fb, fn);
}

struct Rec {  // 16 B segment record: adjacency range [p, p + len) of the middle (word wv) of start entry e
  uint32_t p, len, wv, e;
};

// The kCE entries of one chunk: vm has bit j set iff entry j belongs to the owner record.
// MODE 0: pass 1 in a dense window, 1: pass 1 with the touched-word bitmap, 2: pass 2.
template <int MODE, bool CP, bool WIDE>
__device__ __forceinline__ void t3_chunk(const uint32_t (&ev)[kCE], uint32_t vm, uint32_t cbase,
                                         uint32_t* ctr, uint32_t* bm, uint32_t word0, uint32_t shamt,
                                         uint32_t oshamt, uint32_t wv, uint32_t& cb, uint32_t& cn, uint32_t dummy) {
  if (CP && MODE == 0) {  // pass 1, dense window: an entry outside the record adds 0 to the lane's own word
#pragma unroll
    for (int j = 0; j < (int)kCE; ++j) {
      const bool on = (vm >> j) & 1u;
      uint32_t sh;
      asm("shr.b32 %0, %1, %2;" : "=r"(sh) : "r"(ev[j]), "r"(shamt));
      uint32_t inc;
      asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(inc) : "r"(0u), "r"(1u), "r"(sh));
      sh_red_add(on ? cbase + (ev[j] & kCpAddrMask) : dummy, on ? inc : 0u);
    }
    return;
  }
  if (CP && MODE == 1) {  // pass 1 with the touched-word bitmap: fire-and-forget add and bit-or
    const uint32_t bmbase = (uint32_t)__cvta_generic_to_shared(bm);
#pragma unroll
    for (int j = 0; j < (int)kCE; ++j) {
      const uint32_t on = vm & (1u << j), g = cp_word(ev[j]) - word0;
      sh_red_add_if(cbase + (ev[j] & kCpAddrMask), 1u << ((ev[j] >> shamt) & 31u), on);
      sh_red_or_if(bmbase + 4u * (g >> 5), 1u << (g & 31u), on);
    }
    return;
  }
  if (CP && MODE == 2) {  // pass 2: an entry outside the record reads the lane's own word, counted as 0
    uint32_t own = 0, oth = 0;
#pragma unroll
    for (int j = 0; j < (int)kCE; ++j) {
      const bool on = (vm >> j) & 1u;
      uint32_t v = sh_load(on ? cbase + (ev[j] & kCpAddrMask) : dummy);
      v = on ? v : 0u;
      const uint32_t h = 2u << (ev[j] & 3u);
      own += cp_field(v, ev[j], shamt, h);
      oth += cp_field(v, ev[j], oshamt, h);
    }
    cb += own - (uint32_t)__popc(vm);
    cn += oth;
    return;
  }
#pragma unroll
  for (int j = 0; j < (int)kCE; ++j) {
    if (!((vm >> j) & 1u)) continue;
    if (CP) {
      if (MODE == 2) t3_share_cp(cbase, ev[j], shamt, oshamt, cb, cn);
      else if (MODE == 0) t3_inc_cp<false>(cbase, bm, word0, ev[j], shamt);
      else t3_inc_cp<true>(cbase, bm, word0, ev[j], shamt);
    } else {
      if (MODE == 2) t3_share_c<WIDE>(ctr, word0, ev[j], wv, cb, cn);
      else if (MODE == 0) t3_inc_c<WIDE, false>(ctr, bm, word0, ev[j], wv);
      else t3_inc_c<WIDE, true>(ctr, bm, word0, ev[j], wv);
    }
  }
}

// ---------------------------------------------------------------------------- long records
// A record of at least kLongMin entries (compact encoding) is walked by ONE warp in 128-entry
// blocks starting at its first entry's 16-B aligned position: lane L holds entries 4L..4L+3 of a
// block (one LDG.128; the warp's load is 512 contiguous bytes) and the next two blocks are loaded
// while the current two are processed.  Only the first block (entries before the record, all in
// lane 0) and the last one (entries past it) are masked; a masked entry updates (pass 1: adds 0
// to) or reads (pass 2: counts 0 from) the lane's own word of the window, so there is no branch
// per entry and no two lanes collide.  Pass 2 sums the record's shares in lane registers and
// reduces them once per record.  No owner lookup: shorter records go through the flattened
// batches.
#ifndef BBF_T3_LONG_MIN
#define BBF_T3_LONG_MIN 256
#endif
constexpr uint32_t kLongMin = BBF_T3_LONG_MIN;
constexpr uint32_t kAdjcPad = 512;  // adjc padding (entries): the block prefetch may run 388 past a record

// 1 << (x mod 32) in one funnel shift (no separate "& 31")
__device__ __forceinline__ uint32_t bit_of(uint32_t x) {
  uint32_t r;
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(0u), "r"(1u), "r"(x));
  return r;
}
// v >> (x mod 32)
__device__ __forceinline__ uint32_t shr_wrap(uint32_t v, uint32_t x) {
  uint32_t r;
  asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(v), "r"(0u), "r"(x));
  return r;
}

// one block's 4 entries of this lane.  MODE 0: pass 1, dense window; 1: pass 1 with the
// touched-word bitmap; 2: pass 2 (own / other class sums).  MASKED: entry j counts iff bit j of
// vm4; dummy = the shared address of the lane's own window word.
template <int MODE, bool MASKED>
__device__ __forceinline__ void t3_long4(const uint4& q, uint32_t vm4, uint32_t dummy, uint32_t cbase,
                                         uint32_t bmbase, uint32_t word0, uint32_t shamt, uint32_t oshamt,
                                         uint32_t& own, uint32_t& oth) {
  const uint32_t ev[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const bool on = !MASKED || ((vm4 >> j) & 1u);
    const uint32_t addr = on ? cbase + (ev[j] & kCpAddrMask) : dummy;
    if (MODE == 2) {
      uint32_t v = sh_load(addr);
      if (MASKED) v = on ? v : 0u;
      const uint32_t h = 2u << (ev[j] & 3u);
#ifdef BBF_T3_RECSTAT  // pass-2 entries of long records, and those whose end has a + d >= 2
      {
        const uint32_t o1 = zext(shr_wrap(v, ev[j] >> shamt), h), o2 = zext(shr_wrap(v, ev[j] >> oshamt), h);
        const uint32_t n_on = __popc(__ballot_sync(0xffffffffu, on)), n_use = __popc(__ballot_sync(0xffffffffu, on && o1 + o2 >= 2));
        if ((threadIdx.x & 31) == 0) { T3_COUNT(20, n_on); T3_COUNT(21, n_use); }
      }
#endif
      own += zext(shr_wrap(v, ev[j] >> shamt), h);
      oth += zext(shr_wrap(v, ev[j] >> oshamt), h);
    } else {
      sh_red_add(addr, on ? bit_of(ev[j] >> shamt) : 0u);
      if (MODE == 1 && on) {
        const uint32_t g = cp_word(ev[j]) - word0;
        asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(bmbase + 4u * (g >> 5)), "r"(bit_of(g)));
      }
    }
  }
}

// S1: lane L takes entries L, L+32, L+64, L+96 of each block (4 LDG.32), so one shared operation
// covers 32 consecutive entries: consecutive counter words where ends have one field per word (the
// high-degree zones) — no bank conflicts; no first-block mask (blocks start at the record).  !S1:
// lane L takes entries 4L..4L+3 (one LDG.128): one shared operation covers every 4th entry — distinct
// words where ends pack 4-8 fields per word (the low-degree zones).
template <int MODE, bool S1>
__device__ __forceinline__ void t3_long(const uint32_t* __restrict__ adjc, const Rec& rc, uint32_t cbase,
                                        uint32_t ctr0, uint32_t bmbase, uint32_t word0, int lane,
                                        uint32_t& own, uint32_t& oth) {
  if (S1) {
    const uint32_t shamt = 22u + 5u * (rc.wv >> 31), oshamt = 49u - shamt;
    const uint32_t nb = (rc.len + 127u) >> 7;
    const uint32_t dummy = ctr0 + 4u * (uint32_t)lane;
    const uint32_t* s1 = adjc + rc.p + lane;
    auto ld1 = [&](uint32_t blk) {
      const uint32_t* q = s1 + 128u * blk;
      return make_uint4(q[0], q[32], q[64], q[96]);
    };
    auto vm1 = [&](uint32_t blk) {
      const uint32_t off = 128u * blk + (uint32_t)lane, rem = rc.len > off ? rc.len - off : 0u;
      return rem > 96u ? 15u : rem > 64u ? 7u : rem > 32u ? 3u : rem ? 1u : 0u;
    };
    uint4 c0 = ld1(0), c1 = make_uint4(0u, 0u, 0u, 0u);
    if (nb > 1) c1 = ld1(1);
#pragma unroll 1
    for (uint32_t b = 0; b < nb; b += 2) {
      uint4 n0 = make_uint4(0u, 0u, 0u, 0u), n1 = make_uint4(0u, 0u, 0u, 0u);
      if (b + 2 < nb) n0 = ld1(b + 2);
      if (b + 3 < nb) n1 = ld1(b + 3);
      if (b + 1 == nb) t3_long4<MODE, true>(c0, vm1(b), dummy, cbase, bmbase, word0, shamt, oshamt, own, oth);
      else t3_long4<MODE, false>(c0, 0u, dummy, cbase, bmbase, word0, shamt, oshamt, own, oth);
      if (b + 1 < nb) {
        if (b + 2 == nb) t3_long4<MODE, true>(c1, vm1(b + 1), dummy, cbase, bmbase, word0, shamt, oshamt, own, oth);
        else t3_long4<MODE, false>(c1, 0u, dummy, cbase, bmbase, word0, shamt, oshamt, own, oth);
      }
      c0 = n0;
      c1 = n1;
    }
    return;
  }
  const uint32_t shamt = 22u + 5u * (rc.wv >> 31), oshamt = 49u - shamt;
  const uint32_t p = rc.p, e_end = rc.p + rc.len, b0 = p & ~3u;
  const uint32_t nb = (e_end - b0 + 127u) >> 7;
  const uint32_t dummy = ctr0 + 4u * (uint32_t)lane;
  const uint4* src = reinterpret_cast<const uint4*>(adjc + b0) + lane;
  auto vmask = [&](uint32_t b) {  // valid entries of block b in this lane, as 4 bits
    const uint32_t off = b0 + 128u * b + 4u * (uint32_t)lane;
    const uint32_t lo = p > off ? min(p - off, 4u) : 0u, hi = e_end > off ? min(e_end - off, 4u) : 0u;
    return ((1u << hi) - 1u) & ~((1u << lo) - 1u);
  };
#ifdef BBF_EXP_NOLDG  // timing experiment only: the long records' entries synthesised, not loaded (results wrong)
  const uint32_t syn = ((word0 & kCpWordMask) << 2) | (4u << 27);
  auto ld = [&](uint32_t blk) {
    const uint32_t hsh = (blk * 32u + (uint32_t)lane) * 2654435761u;
    return make_uint4(syn + (((hsh >> 8) & 1023u) << 2), syn + (((hsh >> 12) & 1023u) << 2),
                      syn + (((hsh >> 16) & 1023u) << 2), syn + (((hsh >> 20) & 1023u) << 2));
  };
#else
  auto ld = [&](uint32_t blk) { return src[32 * blk]; };
#endif
  uint4 c0 = ld(0), c1 = make_uint4(0u, 0u, 0u, 0u);
  if (nb > 1) c1 = ld(1);
#pragma unroll 1
  for (uint32_t b = 0; b < nb; b += 2) {
    // the next two blocks, in flight (not past the record: the overshoot was ~25% extra L2 traffic)
    uint4 n0 = make_uint4(0u, 0u, 0u, 0u), n1 = make_uint4(0u, 0u, 0u, 0u);
    if (b + 2 < nb) n0 = ld(b + 2);
    if (b + 3 < nb) n1 = ld(b + 3);
    if (b == 0 || b + 1 == nb) t3_long4<MODE, true>(c0, vmask(b), dummy, cbase, bmbase, word0, shamt, oshamt, own, oth);
    else t3_long4<MODE, false>(c0, 0u, dummy, cbase, bmbase, word0, shamt, oshamt, own, oth);
    if (b + 1 < nb) {
      if (b + 2 == nb) t3_long4<MODE, true>(c1, vmask(b + 1), dummy, cbase, bmbase, word0, shamt, oshamt, own, oth);
      else t3_long4<MODE, false>(c1, 0u, dummy, cbase, bmbase, word0, shamt, oshamt, own, oth);
    }
    c0 = n0;
    c1 = n1;
  }
}

template <bool PV, bool PAIRS, int ENC>
__global__ void __launch_bounds__(kT3Threads, kT3Ctas) k_t3(const EngineArgs a) {
  constexpr bool WIDE = ENC == kEncWide, CP = ENC == kEncCompact;
  extern __shared__ uint32_t smem[];
  uint32_t* ctr = smem;                   // kWin
  uint32_t* bm = smem + kWin;             // kBm
  uint32_t* sh_cnt = bm + kBm;            // kMaxWin record counts
  uint32_t* sh_wc = sh_cnt + kMaxWin;     // kMaxWin wedge counts
  uint32_t* sh_cntl = sh_wc + kMaxWin;    // kMaxWin long-record counts (stored from the slot end)
  __shared__ uint32_t sh_unit, sh_c[4];
  __shared__ uint32_t sh_acc[kT3Warps][2][32];  // per-warp pass-2 accumulators of a batch
  __shared__ Zones sh_z;                        // the current unit's end-side zone table
  const uint32_t* __restrict__ adjc = a.adjc;
  __shared__ unsigned long long sh_red[2][kT3Warps];
  __shared__ unsigned long long sh_dbg[4];  // pass-1 steps, pass-1 chunks, small windows, dense windows
#ifdef BBF_T3_PROF
  __shared__ unsigned long long sh_prof[8];  // pre-scan, window setup, pass 1, pass 2, epilogue, unit tail, small-window passes
  long long t_prof = clock64();
  if (threadIdx.x < 8) sh_prof[threadIdx.x] = 0;
  if (threadIdx.x == 0) atomicMin(&g_prof_t[0], gtimer());
#endif
  if (threadIdx.x < 4) sh_dbg[threadIdx.x] = 0;
#ifdef BBF_T3_BUSYPROF  // per window size class: warp-cycles in long records, in short batches, and the pass span x warps
  __shared__ unsigned long long sh_busy[6][4];
  if (threadIdx.x < 24) (&sh_busy[0][0])[threadIdx.x] = 0;
#endif
#ifdef BBF_T3_LATPROF
  __shared__ unsigned long long sh_lat[20];
  if (threadIdx.x < 20) sh_lat[threadIdx.x] = 0;
#endif
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  for (uint32_t i = tid; i < kWin + kBm + 3 * kMaxWin; i += kT3Threads) smem[i] = 0;
  const size_t RS = a.rec_stride;
  Rec* R = reinterpret_cast<Rec*>(a.scratch) + (size_t)blockIdx.x * RS * a.kwin_cap;
  unsigned long long totB = 0, totN = 0;
  __syncthreads();

  while (true) {
    if (tid == 0) sh_unit = (uint32_t)atomicAdd(&a.acc[2], 1ull);
    if (tid < 4) sh_c[tid] = 0;
    __syncthreads();
    const uint64_t ui = shard_item(sh_unit, a.rank, a.nranks);
    if (ui >= a.n_units) break;
    const Unit u = a.units[ui];
    const uint32_t x = u.x;
    const bool xu = x < a.n_u;
    const uint32_t sb = xu ? 0 : a.n_u, ob = xu ? a.n_u : 0, lx = x - sb;
    const uint32_t rs = a.rsafe[xu ? 0 : 1];  // end-role packing threshold of this unit's end side
    const uint32_t rmv = a.rmid[xu ? 1 : 0];  // middle-role packing threshold (middles: other side)
    // the end side's zone table in shared memory (an indexed kernel-parameter read is an LDC
    // with a long-scoreboard dependency on every epilogue word)
    if (tid < 11) reinterpret_cast<uint32_t*>(&sh_z)[tid] = reinterpret_cast<const uint32_t*>(&a.z[xu ? 0 : 1])[tid];
    __syncthreads();
    const Zones& Z = sh_z;
    const uint32_t K = (Z.WB[5] + kWin - 1) / kWin;
    const uint32_t m_lo = a.mid ? a.mid[x] : a.off[x];
    const uint32_t m = a.end1[x] - m_lo;
    // ends after x (u.lo = lx + 1 .. L4) or, with a.ue (route 3), before x (0 .. lx); a unit that
    // starts or ends inside that range cuts each middle's segment by a binary search
    const bool split_lo = u.lo > (a.ue ? 0u : lx + 1), split_hi = u.hi < (a.ue ? lx : Z.L[4]);
    T3_MARK(5);
#ifdef BBF_T3_WINPROF
    const long long t_unit = clock64();
#endif

    // ---------------- pre-scan: segment records per window
    while (true) {
      uint32_t bt = 0;
      if (lane == 0) bt = atomicAdd(&sh_c[0], 1u);
      bt = __shfl_sync(0xffffffffu, bt, 0);
      if (bt * 32 >= m) break;
      const uint32_t i = bt * 32 + lane;
      uint32_t wv = 0, s = 0, en = 0, rl = 0;
      if (i < m) {
        const uint32_t e = m_lo + i;
        wv = a.adj[e];
        s = a.ub[e];
        en = a.end1[ob + (wv & kMask)];
        if (a.ue) en = min(en, a.ue[e]);  // route 3: the ends before x's own entry of N(v)
        rl = a.rlast[ob + (wv & kMask)];  // same level as end1: no dependent runid[en - 1] load
        const unsigned long long clo = a.unit_cut ? a.unit_cut[2ull * ui] : ~0ull;
        const unsigned long long chi = a.unit_cut ? a.unit_cut[2ull * ui + 1] : ~0ull;
        if (split_lo && clo != ~0ull) {
          s = max(s, a.cut_tab[clo + i]);
        } else if (split_lo && s < en) {
          uint32_t b = s, f = en;
          while (b < f) {
            uint32_t md = b + (f - b) / 2;
            if ((a.adj[md] & kMask) < u.lo) b = md + 1; else f = md;
          }
          s = b;
        }
        if (split_hi && chi != ~0ull) {
          en = min(en, a.cut_tab[chi + i]);
        } else if (split_hi && s < en) {
          uint32_t b = s, f = en;
          while (b < f) {
            uint32_t md = b + (f - b) / 2;
            if ((a.adj[md] & kMask) < u.hi) b = md + 1; else f = md;
          }
          en = b;
        }
      }
#ifdef BBF_T3_RECSTAT  // pre-scan middles: [84] of split units, [85] of those with a non-empty range, [86] of whole starts
      if (i < m) {
        if (split_lo || split_hi) { T3_COUNT(84, 1); if (s < en) T3_COUNT(85, 1); }
        else T3_COUNT(86, 1);
      }
#endif
      // records of this middle = the graph's window runs of row v clipped to [s, en)
      const uint32_t r0 = s < en ? a.runid[s] : 0;
      const uint32_t nr = s < en ? ((split_hi || a.ue) ? a.runid[en - 1] : rl) - r0 + 1 : 0;
      const uint32_t incl = warp_incl_scan(nr, lane), excl = incl - nr;
      const uint32_t T = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t nz = __ballot_sync(0xffffffffu, nr > 0);
      for (uint32_t base = 0; base < T; base += 32) {
        const int ow = flat_owner(nr, excl, nz, base, lane);
        const uint32_t f = base + lane;
        const uint32_t o_excl = __shfl_sync(0xffffffffu, excl, ow);
        const uint32_t o_r0 = __shfl_sync(0xffffffffu, r0, ow);
        const uint32_t o_s = __shfl_sync(0xffffffffu, s, ow);
        const uint32_t o_en = __shfl_sync(0xffffffffu, en, ow);
        const uint32_t o_wv = __shfl_sync(0xffffffffu, wv, ow);
        const uint32_t o_e = __shfl_sync(0xffffffffu, m_lo + i, ow);  // the start->middle entry
        if (f < T) {
          const uint32_t r = o_r0 + (f - o_excl);
          const uint2 run = a.runs[r];
          const uint32_t rs = max(run.x, o_s);
          const uint32_t re = (r + 1 < a.nruns) ? min(a.runs[r + 1].x, o_en) : o_en;
          if (re > rs) atomicAdd(&sh_wc[run.y], re - rs);
          for (uint32_t p = rs; p < re; p += kRecMax) {
            const uint32_t len = min(kRecMax, re - p);
            if (CP && len >= kLongMin) {  // long record: walked by one warp (t3_long)
              const uint32_t slot = atomicAdd(&sh_cntl[run.y], 1u);
              R[(size_t)run.y * RS + (RS - 1 - slot)] = Rec{p, len, o_wv, o_e};
            } else {
              const uint32_t slot = atomicAdd(&sh_cnt[run.y], 1u);
              R[(size_t)run.y * RS + slot] = Rec{p, len, o_wv, o_e};
            }
          }
#ifdef BBF_T3_RECSTAT
          if (re > rs) {
            T3_COUNT(0, re - rs);
            T3_COUNT(1, (re + 63) / 64 - rs / 64);
            T3_COUNT(2, (re + 31) / 32 - rs / 32);
            T3_COUNT(3, (re + 15) / 16 - rs / 16);
            if (re - rs < 8) T3_COUNT(4, 1);
            if (re - rs < 64) T3_COUNT(5, re - rs);
            T3_COUNT(10, 1);
            {  // entries by run length: [0] <8 [1] <32 [2] <128 [3] <512 [4] >= 512 (runs, before kRecMax splits)
              const uint32_t L = re - rs;
              T3_COUNT(11 + (L < 8 ? 0 : L < 32 ? 1 : L < 128 ? 2 : L < 512 ? 3 : 4), L);
            }
          }
#endif
        }
      }
    }
    __syncthreads();
    T3_MARK(0);
    unsigned long long xB = 0, xN = 0;

    for (uint32_t k = 0; k < K; ++k) {
      const uint32_t nrec = sh_cnt[k], nlong = sh_cntl[k];
      if (nrec + nlong == 0) continue;
      const uint32_t word0 = k * kWin;
      const uint32_t cbase = (uint32_t)__cvta_generic_to_shared(ctr) - 4u * word0;
      const Rec* rw = R + (size_t)k * RS;
      // records per warp batch: spread a window's records over all 32 warps (>= 2 batches each)
            // records per warp batch: a fixed batch (a.bsz) amortises the batch set-up over more
      // steps; 0 = spread the window's records over all warps (>= 2 batches each)
      const uint32_t bsz = a.bsz ? a.bsz : min(32u, max(2u, (nrec + 2 * kT3Warps - 1) / (2 * kT3Warps)));
      // dense window: at least as many wedges as counter words -> no touched-word bitmap, the
      // epilogue scans every word of the window
      const uint32_t nwk = min(kWin, Z.WB[5] - word0);
      const bool dense = sh_wc[k] * a.dense_div >= nwk;
      // long records' lane layout (t3_long): consecutive entries per shared operation while the
      // window starts before the 2-bit-field zone (ends of degree 2-3), every 4th entry there
#ifndef BBF_T3_S1_ZONE
#define BBF_T3_S1_ZONE 4  // measured: zones 2/3/4/5 -> 71.3/71.4/71.0/71.4 ms on config 5
#endif
      const bool s1w = word0 < Z.WB[BBF_T3_S1_ZONE];
      if (tid < 4) sh_c[tid] = 0;
#ifdef BBF_T3_RECSTAT
      if (tid == 0) T3_COUNT(dense ? 6 : 7, sh_wc[k]);
#endif
      if (tid == 0) {
        atomicAdd(&a.acc[6], (unsigned long long)nrec);
        atomicAdd(&a.acc[7], 1ull);
        if (nrec + nlong < 64) sh_dbg[2]++;
        if (dense) sh_dbg[3]++;
      }
      __syncthreads();
      T3_MARK(1);
#ifdef BBF_T3_LATPROF  // tiny windows (< 2K wedges): when each warp's first batch and chunks arrive
      const long long t_lat = clock64();
      const bool tiny = sh_wc[k] < 2048;
#endif
#ifdef BBF_T3_WINPROF  // CTA cycles of the window's passes + epilogue, binned by its wedge count
      const long long t_win = clock64();
      const uint32_t wbin = sh_wc[k] < 2048 ? 0 : sh_wc[k] < 8192 ? 1 : sh_wc[k] < 32768 ? 2 : sh_wc[k] < 131072 ? 3 : sh_wc[k] < 524288 ? 4 : 5;
#endif
      // ---------------- pass 1 (Alg. 2 lines 9-14) and pass 2 (per-vertex shares)
#pragma unroll 1
      for (int pass = 0; pass < (PV ? 2 : 1); ++pass) {
#ifdef BBF_T3_BUSYPROF
        const long long tb0 = clock64();
        const uint32_t bcls = sh_wc[k] < 2048 ? 0 : sh_wc[k] < 8192 ? 1 : sh_wc[k] < 32768 ? 2 : sh_wc[k] < 131072 ? 3 : sh_wc[k] < 524288 ? 4 : 5;
#endif
#ifdef BBF_EXP_NOLONG  // timing experiment only: long records skipped (results wrong)
        if (false) {
#else
        if (CP && nlong) {  // long records first, one warp each (sh_c[2 + pass] is the cursor)
#endif
          const uint32_t bmbase = (uint32_t)__cvta_generic_to_shared(bm);
          uint32_t r = 0;
          if (lane == 0) r = atomicAdd(&sh_c[2 + pass], 1u);
          r = __shfl_sync(0xffffffffu, r, 0);
          Rec rn = r < nlong ? rw[RS - 1 - r] : Rec{0, 0, 0, 0};
          while (r < nlong) {
            const Rec rl = rn;
            uint32_t r2 = 0;  // the warp's next record, loaded while this one is walked
            if (lane == 0) r2 = atomicAdd(&sh_c[2 + pass], 1u);
            r2 = __shfl_sync(0xffffffffu, r2, 0);
            if (r2 < nlong) rn = rw[RS - 1 - r2];
            r = r2;
            uint32_t own = 0, oth = 0;
            const uint32_t ctr0 = (uint32_t)__cvta_generic_to_shared(ctr);
            if (s1w) {
              if (pass == 1) t3_long<2, true>(adjc, rl, cbase, ctr0, bmbase, word0, lane, own, oth);
              else if (dense) t3_long<0, true>(adjc, rl, cbase, ctr0, bmbase, word0, lane, own, oth);
              else t3_long<1, true>(adjc, rl, cbase, ctr0, bmbase, word0, lane, own, oth);
            } else {
              if (pass == 1) t3_long<2, false>(adjc, rl, cbase, ctr0, bmbase, word0, lane, own, oth);
              else if (dense) t3_long<0, false>(adjc, rl, cbase, ctr0, bmbase, word0, lane, own, oth);
              else t3_long<1, false>(adjc, rl, cbase, ctr0, bmbase, word0, lane, own, oth);
            }
            if (pass == 1) {
              // the record's own-class sum and other-class sum (each < 2^26: <= 1024 entries of
              // 16-bit fields), minus one per wedge for the own class (Lemma 2 shares)
              own = __reduce_add_sync(0xffffffffu, own);
              oth = __reduce_add_sync(0xffffffffu, oth);
              if (lane == 0 && ((own - rl.len) | oth)) mid_red(a, rmv, rl.wv & kMask, ob + (rl.wv & kMask), own - rl.len, oth, rl.e);
            }
          }
        }
        // batches of bsz records; the next batch's records are loaded while this one is
        // processed (their global-load latency was the kernel's top stall)
        // guided batches: up to bsz records, shrinking near the end of the window so the warps
        // reach the pass barrier together
        auto fetch = [&](uint32_t& cntx, Rec& rx) {
          uint32_t s0 = 0, c0 = 0;
          if (lane == 0) {
            const uint32_t seen = *reinterpret_cast<volatile uint32_t*>(&sh_c[pass]);
            const uint32_t rem = seen < nrec ? nrec - seen : 0u;
            const uint32_t sz = min(bsz, max((uint32_t)BBF_T3_BMIN, rem / kT3Warps));
            s0 = atomicAdd(&sh_c[pass], sz);
            c0 = s0 < nrec ? min(sz, nrec - s0) : 0u;
          }
          const uint32_t r0x = __shfl_sync(0xffffffffu, s0, 0);
          cntx = __shfl_sync(0xffffffffu, c0, 0);
          rx = Rec{0, 0, 0, 0};
          if ((uint32_t)lane < cntx) rx = rw[r0x + lane];
        };
#ifdef BBF_T3_BUSYPROF
        const long long tb1 = clock64();
#endif
        uint32_t cnt_next;
        Rec rc_next;
#ifdef BBF_T3_LATPROF
        bool lat_seen = false;
        if (tiny && lane == 0) { T3_LAT(106 + pass, clock64() - t_lat); T3_LAT(108 + pass, 1); }  // warp reaches the flattened part
#endif
#ifdef BBF_EXP_NOFLAT  // timing experiment only: short records skipped (results wrong)
        cnt_next = 0;
#else
        fetch(cnt_next, rc_next);
#endif
        while (true) {
          const uint32_t cnt = cnt_next;
          const Rec rc = rc_next;
          if (cnt == 0) break;
#ifdef BBF_T3_LATPROF
          bool lat_first = false;
          if (tiny && !lat_seen) {
            lat_seen = true;
            lat_first = true;
            const uint32_t dep = __shfl_sync(0xffffffffu, rc.len, 0);  // the batch's records have arrived
            if (lane == 0) { T3_LAT(96 + pass, clock64() - t_lat + (dep & 0)); T3_LAT(98 + pass, 1); }
          }
#endif
          fetch(cnt_next, rc_next);
          if (pass == 1) { sh_acc[warp][0][lane] = 0; sh_acc[warp][1][lane] = 0; __syncwarp(); }
          // The batch's records are flattened over the lanes in 32-B chunks of the adjacency
          // (kCE = 8 entries, two LDG.128 per lane, consecutive lanes on consecutive chunks of a
          // record; a record's first / last chunk is masked to [p, p + len)).  Step `base` gives
          // lane L chunk base + L; its owner (the record holding it) = the records started before
          // the step + the popcount of the step's record-start mask up to the lane, minus one.
          const uint32_t nch = rc.len ? (rc.p + rc.len + kCE - 1) / kCE - rc.p / kCE : 0;
          const uint32_t incl = warp_incl_scan(nch, lane), excl = incl - nch;
          const uint32_t T = __shfl_sync(0xffffffffu, incl, 31);
          int carry = 0;
#ifdef BBF_T3_PROF
          if (pass == 0 && lane == 0) {
            atomicAdd(&sh_dbg[0], (unsigned long long)((T + 31) / 32));
            atomicAdd(&sh_dbg[1], (unsigned long long)T);
          }
#endif
          // kU steps per iteration (BBF_T3_KU, default 1): owner lookups first, then all chunk
          // loads in flight, then the counter updates
          for (uint32_t base0 = 0; base0 < T; base0 += 32 * kU) {
            uint32_t smask[kU], ow[kU], gs[kU], ch[kU], o_p[kU], o_len[kU], o_wv[kU];
            uint4 q[kU][kCE / 4];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
              const uint32_t base = base0 + 32 * u;
              // records start at distinct chunks, in lane order: my owner = the records started
              // before this step + those starting at or before my chunk in it, minus one
              const bool st = nch > 0 && excl >= base && excl < base + 32;
              smask[u] = __reduce_or_sync(0xffffffffu, st ? 1u << (excl - base) : 0u);
              const uint32_t m = smask[u] & (0xffffffffu >> (31 - lane));
              gs[u] = m ? 31 - __clz(m) : 0;  // first lane of my owner's group in this step
              ow[u] = (uint32_t)(carry + __popc(m) - 1);
              carry += __popc(smask[u]);
              const uint32_t o_excl = __shfl_sync(0xffffffffu, excl, ow[u]);
              o_p[u] = __shfl_sync(0xffffffffu, rc.p, ow[u]);
              o_len[u] = __shfl_sync(0xffffffffu, rc.len, ow[u]);
              o_wv[u] = __shfl_sync(0xffffffffu, rc.wv, ow[u]);
              ch[u] = o_p[u] / kCE + (base + lane - o_excl);  // absolute chunk of adjc (kCE entries)
            }
#pragma unroll
            for (int u = 0; u < kU; ++u)
#pragma unroll
              for (int h = 0; h < kCE / 4; ++h)
                q[u][h] = (base0 + 32 * u + lane < T) ? reinterpret_cast<const uint4*>(adjc)[ch[u] * (kCE / 4) + h]
                                                     : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
            for (int u = 0; u < kU; ++u) {
              const uint32_t c = base0 + 32 * u + lane;
              const uint32_t shamt = 22u + 5u * (o_wv[u] >> 31), oshamt = 49u - shamt;
              uint32_t cb = 0, cn = 0;
              if (c < T) {
                const uint32_t e0 = kCE * ch[u];
                uint32_t ev[kCE];
#pragma unroll
                for (int h = 0; h < (int)(kCE / 4); ++h) {
                  ev[4 * h] = q[u][h].x; ev[4 * h + 1] = q[u][h].y; ev[4 * h + 2] = q[u][h].z; ev[4 * h + 3] = q[u][h].w;
                }
                // entries [o_p, o_p + o_len) of this chunk as a bit mask
                const int lo = (int)(o_p[u] > e0 ? o_p[u] - e0 : 0u);
                const uint32_t end = o_p[u] + o_len[u];
                const int hi = (int)(end - e0 < kCE ? end - e0 : kCE);
                const uint32_t vm = ((1u << hi) - 1u) & ~((1u << lo) - 1u);
                const uint32_t dummy = (uint32_t)__cvta_generic_to_shared(ctr) + 4u * (uint32_t)lane;
                if (pass == 1) t3_chunk<2, CP, WIDE>(ev, vm, cbase, ctr, bm, word0, shamt, oshamt, o_wv[u], cb, cn, dummy);
                else if (dense) t3_chunk<0, CP, WIDE>(ev, vm, cbase, ctr, bm, word0, shamt, oshamt, o_wv[u], cb, cn, dummy);
                else t3_chunk<1, CP, WIDE>(ev, vm, cbase, ctr, bm, word0, shamt, oshamt, o_wv[u], cb, cn, dummy);
              }
#ifdef BBF_T3_LATPROF
              if (lat_first && u == 0 && base0 == 0) {
                const uint32_t dep = __shfl_sync(0xffffffffu, cb + cn, 0);  // the first step's chunks are processed
                if (lane == 0) { T3_LAT(100 + pass, clock64() - t_lat + (dep & 0)); T3_LAT(110 + pass, 1); }
              }
#endif
              if (pass == 1 && __any_sync(0xffffffffu, (cb | cn) != 0)) {
                // segmented sum over each owner's lane group; its last lane adds it (one writer
                // per owner per step, so no atomics)
                uint32_t sb, sn;
                seg_sums2(cb, cn, (int)gs[u], lane, sb, sn);
                const bool last = c < T && (c + 1 == T || lane == 31 || ((smask[u] >> (lane + 1)) & 1u));
                if (last) {
                  sh_acc[warp][0][ow[u]] += sb;
                  sh_acc[warp][1][ow[u]] += sn;
                }
                __syncwarp();
              }
            }
          }
          if (pass == 1) {
            __syncwarp();
            const uint32_t cb = sh_acc[warp][0][lane], cn = sh_acc[warp][1][lane];
            if (cb | cn) mid_red(a, rmv, rc.wv & kMask, ob + (rc.wv & kMask), cb, cn, rc.e);
            __syncwarp();
          }
        }
#ifdef BBF_T3_LATPROF
        if (tiny && lane == 0 && lat_seen) { T3_LAT(102 + pass, clock64() - t_lat); T3_LAT(112 + pass, 1); }
#endif
#ifdef BBF_T3_BUSYPROF
        const long long tb2 = clock64();
        if (lane == 0) { atomicAdd(&sh_busy[bcls][0], (unsigned long long)(tb1 - tb0)); atomicAdd(&sh_busy[bcls][1], (unsigned long long)(tb2 - tb1)); }
#endif
        __syncthreads();
#ifdef BBF_T3_BUSYPROF
        if (tid == 0) { atomicAdd(&sh_busy[bcls][2], (unsigned long long)(clock64() - tb0) * kT3Warps); atomicAdd(&sh_busy[bcls][3], 1ull); }
#endif
#ifdef BBF_T3_LATPROF
        if (tiny && tid == 0) { T3_LAT(104 + pass, clock64() - t_lat); T3_LAT(114 + pass, 1); }
#endif
        T3_MARK(nrec < 64 ? 1 : 2 + pass);  // slot 1: set-up + passes of small windows
#ifdef BBF_T3_WINPROF
        if (tid == 0) T3_COUNT(40 + 3 * wbin + pass, clock64() - t_win);
#endif
      }

      // ---------------- epilogue: Lemma 2 per touched end (Alg. 2 lines 15-18), clear the window
      const ZoneRegs zr = zone_regs(Z);
      if (dense) {
        uint4* c4 = reinterpret_cast<uint4*>(ctr);
        for (uint32_t i4 = tid; i4 < (nwk + 3) / 4; i4 += kT3Threads) {
          const uint4 q = c4[i4];
          if (!(q.x | q.y | q.z | q.w)) continue;
          c4[i4] = make_uint4(0u, 0u, 0u, 0u);
          const uint32_t gw = word0 + 4 * i4;
          if (WIDE && gw < Z.WB[1]) {  // zone 0 pairs (a word, d word), word0 and WB[1] even
            epi_wide<PV, PAIRS>(a, sb, x, gw, q.x, q.y, xB, xN);
            if (gw + 2 < Z.WB[1]) epi_wide<PV, PAIRS>(a, sb, x, gw + 2, q.z, q.w, xB, xN);
            else {
              if (q.z) epi_packed<PV, PAIRS>(a, zone_of(zr, gw + 2), sb, rs, x, gw + 2, q.z, xB, xN);
              if (q.w) epi_packed<PV, PAIRS>(a, zone_of(zr, gw + 3), sb, rs, x, gw + 3, q.w, xB, xN);
            }
            continue;
          }
          const ZoneP zp = zone_of(zr, gw);
          if (gw + 3 < zp.end) {  // the four words share a zone (the common case)
            if (q.x) epi_packed<PV, PAIRS>(a, zp, sb, rs, x, gw, q.x, xB, xN);
            if (q.y) epi_packed<PV, PAIRS>(a, zp, sb, rs, x, gw + 1, q.y, xB, xN);
            if (q.z) epi_packed<PV, PAIRS>(a, zp, sb, rs, x, gw + 2, q.z, xB, xN);
            if (q.w) epi_packed<PV, PAIRS>(a, zp, sb, rs, x, gw + 3, q.w, xB, xN);
          } else {
            if (q.x) epi_packed<PV, PAIRS>(a, zp, sb, rs, x, gw, q.x, xB, xN);
            if (q.y) epi_packed<PV, PAIRS>(a, zone_of(zr, gw + 1), sb, rs, x, gw + 1, q.y, xB, xN);
            if (q.z) epi_packed<PV, PAIRS>(a, zone_of(zr, gw + 2), sb, rs, x, gw + 2, q.z, xB, xN);
            if (q.w) epi_packed<PV, PAIRS>(a, zone_of(zr, gw + 3), sb, rs, x, gw + 3, q.w, xB, xN);
          }
        }
      } else {
        for (uint32_t bw = tid; bw < kBm; bw += kT3Threads) {
          uint32_t bits = bm[bw];
          if (!bits) continue;
          bm[bw] = 0;
          while (bits) {
            const uint32_t j = __ffs(bits) - 1;
            bits &= bits - 1;
            const uint32_t wi = bw * 32 + j;
            const uint32_t gw = word0 + wi;
            const uint32_t v = ctr[wi];
            ctr[wi] = 0;
            if (WIDE && gw < Z.WB[1]) {  // bits are set on the a word only
              const uint32_t vd = ctr[wi + 1];
              ctr[wi + 1] = 0;
              epi_wide<PV, PAIRS>(a, sb, x, gw, v, vd, xB, xN);
            } else {
              epi_packed<PV, PAIRS>(a, zone_of(zr, gw), sb, rs, x, gw, v, xB, xN);
            }
          }
        }
      }
      __syncthreads();
      T3_MARK(4);
#ifdef BBF_T3_WINPROF
      if (tid == 0) {
        T3_COUNT(42 + 3 * wbin, clock64() - t_win);
        T3_COUNT(16 + 3 * wbin, 1);
        T3_COUNT(17 + 3 * wbin, sh_wc[k]);
        T3_COUNT(18 + 3 * wbin, clock64() - t_win);
      }
#endif
    }
#ifdef BBF_T3_WINPROF  // per unit: wedges, windows with records, CTA cycles (pre-scan to end), binned by wedges
    if (tid == 0) {
      unsigned long long wu = 0, nw = 0;
      for (uint32_t k = 0; k < K; ++k) { wu += sh_wc[k]; nw += (sh_cnt[k] + sh_cntl[k]) ? 1 : 0; }
      const uint32_t ub = wu < 16384 ? 0 : wu < 65536 ? 1 : wu < 262144 ? 2 : wu < 1048576 ? 3 : 4;
      T3_COUNT(64 + 4 * ub, 1);
      T3_COUNT(65 + 4 * ub, wu);
      T3_COUNT(66 + 4 * ub, nw);
      T3_COUNT(67 + 4 * ub, clock64() - t_unit);
    }
    __syncthreads();
#endif
    for (uint32_t k = tid; k < K; k += kT3Threads) { sh_cnt[k] = 0; sh_wc[k] = 0; sh_cntl[k] = 0; }
    // unit totals -> start vertex
    totB += xB;
    totN += xN;
    if (PV) {
      unsigned long long b = warp_sum(xB), nn = warp_sum(xN);
      if (lane == 0) { sh_red[0][warp] = b; sh_red[1][warp] = nn; }
      __syncthreads();
      if (warp == 0) {
        b = warp_sum(lane < kT3Warps ? sh_red[0][lane] : 0ull);
        nn = warp_sum(lane < kT3Warps ? sh_red[1][lane] : 0ull);
        if (lane == 0 && (b | nn) && !a.edge) {
          atomicAdd(&a.pv[2ull * (x)], b);
          atomicAdd(&a.pv[2ull * (x) + 1], nn);
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
#ifdef BBF_T3_LATPROF
  if (tid < 20) atomicAdd(&g_prof_cnt[96 + tid], sh_lat[tid]);
#endif
#ifdef BBF_T3_BUSYPROF
  if (tid < 24) atomicAdd(&g_prof_cnt[96 + tid], (&sh_busy[0][0])[tid]);
#endif
#ifdef BBF_T3_PROF
  if (tid == 0) {
    for (int i = 0; i < 5; ++i) atomicAdd(&a.acc[11 + i], sh_prof[i]);
    const unsigned long long t_end = gtimer();
    atomicMin(&g_prof_t[1], t_end);
    atomicMax(&g_prof_t[2], t_end);
  }
#endif
  if (tid == 0) {
    atomicAdd(&a.acc[5], sh_dbg[0]);
    atomicAdd(&a.acc[8], sh_dbg[1]);
    atomicAdd(&a.acc[9], sh_dbg[2]);
    atomicAdd(&a.acc[10], sh_dbg[3]);
  }
}

// ===================================================================================== T1
__device__ __forceinline__ uint32_t hslot(uint32_t l, uint32_t mask) {
  return (l * 0x9E3779B1u) >> 16 & mask;
}

// Two instances: <32 warps, 256 slots> for starts with <= kT1SmallMax wedges (2 CTAs = 64 warps
// per SM) and <12 warps, kT1Slots> for the rest (24 warps per SM, shared-memory bound).
template <bool PV, bool PAIRS, int kT1Warps, uint32_t kT1Slots>
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
    if (lane == 0) q = atomicAdd(&a.acc[a.t1ctr], 1ull);
    q = __shfl_sync(0xffffffffu, q, 0);
    const uint64_t ti = shard_item(q, a.rank, a.nranks);
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
          if (a.ue) en = min(en, a.ue[m_lo + i]);  // route 3: the ends before x's own entry of N(v)
          len = en > s ? en - s : 0;
        }
        const uint32_t incl = warp_incl_scan(len, lane), excl = incl - len;
        const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
        if (tot == 0) continue;
        // the chunk's non-empty middles in lane order (their first wedges strictly increase); a
        // wedge's middle = those started before this step + those starting in it at or before
        // the lane (start-mask popcount), looked up in the compacted lane list
        const uint32_t nzm = __ballot_sync(0xffffffffu, len > 0);
        if (len) sh_incl[__popc(nzm & ((1u << lane) - 1u))] = lane;
        __syncwarp();
        int carry = -1;
        for (uint32_t base = 0; base < tot; base += 32) {
          const uint32_t t = base + lane;
          const bool stt = len > 0 && excl >= base && excl < base + 32;
          const uint32_t smask = __reduce_or_sync(0xffffffffu, stt ? 1u << (excl - base) : 0u);
          const uint32_t mm = smask & (0xffffffffu >> (31 - lane));
          const int rk = carry + __popc(mm);
          carry += __popc(smask);
          const int jl = (int)sh_incl[rk < 0 ? 0 : rk];  // owner lane
          const uint32_t o_s = __shfl_sync(0xffffffffu, s, jl), o_excl = __shfl_sync(0xffffffffu, excl, jl);
          const uint32_t o_wv = __shfl_sync(0xffffffffu, wv, jl);
          uint32_t b2 = 0, n2 = 0;
          if (t < tot) {
            uint32_t ev = a.adj[o_s + (t - o_excl)];
            uint32_t l = ev & kMask;
            uint32_t cls = (ev ^ o_wv) >> 31;
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
              b2 = cls ? dd - 1 : ad - 1;
              n2 = cls ? ad : dd;
            }
          }
          if (pass == 1 && __any_sync(0xffffffffu, (b2 | n2) != 0)) {
            // per-middle sums over runs of equal owners, one shared add per run
            const int gs = mm ? 31 - __clz(mm) : 0;
            uint32_t sb2, sn2;
            seg_sums2(b2, n2, gs, lane, sb2, sn2);
            const bool last = t < tot && (lane == 31 || t + 1 == tot || ((smask >> (lane + 1)) & 1u));
            if (last && (sb2 | sn2)) {
              sh_mb[jl] += sb2;  // one writer per middle per step
              sh_mn[jl] += sn2;
            }
          }
          __syncwarp();
        }
        __syncwarp();
        if (pass == 1) {
          uint32_t b2 = sh_mb[lane], n2 = sh_mn[lane];
          if (b2 | n2) mid_red(a, a.rmid[xu ? 1 : 0], wv & kMask, ob + (wv & kMask), b2, n2, m_lo + cb + lane);
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
      if (PV) end_red(a, a.rsafe[sb ? 1 : 0], key - 1, wrow, (uint32_t)fb, (uint32_t)fn);  // a, d < 2^16
      if (PAIRS && fb) emit_pair(a, x, wrow, fb, fn);
    }
    __syncwarp();
    totB += xB;
    totN += xN;
    if (PV) {
      xB = warp_sum(xB);
      xN = warp_sum(xN);
      if (lane == 0 && (xB | xN) && !a.edge) {
        atomicAdd(&a.pv[2ull * (x)], xB);
        atomicAdd(&a.pv[2ull * (x) + 1], xN);
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

// ===================================================================================== T2
// Mid-size starts (kT1Max < work <= T2 max): one CTA per start, a shared open-addressing hash of
// (end rank + 1 -> a | d << 16) with S = pow2 >= 2 * work slots, so a start is done in one sweep
// of its wedges (no counter windows, no records).  Warps take chunks of 32 middles; inside a
// chunk the wedges are spread over the lanes as in k_t1.  a + d <= #middles <= work < 2^16.
// Two instances: <512 threads, kT2Slots> for starts above kT2SmallMax wedges and <256,
// kT2Slots / 2> for the rest.  The start's wedges are flattened over ALL warps of the CTA (not
// middle chunks per warp: per-chunk work varied so much that barrier waits were most of the
// kernel's time): the middles of a round (<= 2 per thread) are loaded with their segment lengths,
// a CTA scan gives each middle's first wedge, and warp w takes wedge steps w, w + warps, ... ;
// a lane finds its middle by binary search in the shared prefix.  Pass 2 sums the middle shares
// per run of equal middles in a step and adds them to per-middle shared totals.
template <bool PV, bool PAIRS, int kT2Threads, int kSlots, int kMPT>
__global__ void __launch_bounds__(kT2Threads, kMPT == 1 ? 3 : 1) k_t2(const EngineArgs a) {
  constexpr int kT2Warps = kT2Threads / 32;
  constexpr uint32_t kM = kMPT * kT2Threads;  // middles per round (kMPT per thread)
  extern __shared__ uint32_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  volatile uint32_t* keys = smem;
  uint32_t* vals = smem + kSlots;
  uint32_t* mP = vals + kSlots;  // kM + 1: mP[i] = first flattened wedge of middle i
  uint32_t* mS = mP + kM + 1;    // kM: first eligible end entry (ub)
  uint32_t* mW = mS + kM;        // kM: middle word
  uint32_t* mB = mW + kM;        // kM: pass-2 balanced share of the middle
  uint32_t* mN = mB + kM;        // kM: pass-2 unbalanced share
  uint32_t* mE = mN + kM;        // kM: start->middle entry (per-edge counts only; launched with the extra space)
  __shared__ uint32_t sh_item, sh_mcc, sh_wsum[kT2Warps];
  __shared__ unsigned long long sh_red[2][kT2Warps];
  for (uint32_t i = tid; i < 2 * kSlots; i += kT2Threads) ((uint32_t*)keys)[i] = 0;
  unsigned long long totB = 0, totN = 0;
  __syncthreads();
  while (true) {
    if (tid == 0) sh_item = (uint32_t)atomicAdd(&a.acc[a.t2ctr], 1ull);
    __syncthreads();
    const uint64_t ti = shard_item(sh_item, a.rank, a.nranks);
    if (ti >= a.n_t2) break;
    const uint32_t x = a.t2[ti];
    const bool xu = x < a.n_u;
    const uint32_t sb = xu ? 0 : a.n_u, ob = xu ? a.n_u : 0;
    const uint32_t m_lo = a.mid ? a.mid[x] : a.off[x];
    const uint32_t m = a.end1[x] - m_lo;
    const uint32_t W = (uint32_t)a.work[x];
    uint32_t S = 64;
    while (S < 2 * W && S < kSlots) S <<= 1;
    const uint32_t mask = S - 1;
#pragma unroll 1
    for (int pass = 0; pass < (PV ? 2 : 1); ++pass) {
#pragma unroll 1
      for (uint32_t r0 = 0; r0 < m; r0 += kM) {
        const uint32_t mc = min(kM, m - r0);
        if (pass == 1 && m <= kM) {
          // single-round start: pass 2 reuses pass 1's middle table (mS, mW, mP are only read by
          // the steps); just clear the per-middle share totals
          for (uint32_t i2 = tid; i2 < sh_mcc; i2 += kT2Threads) { mB[i2] = 0; mN[i2] = 0; }
          __syncthreads();
        } else {
          // round set-up: two consecutive middles per thread; one CTA-wide exclusive scan of
          // (segment length << 12 | non-empty) compacts the non-empty middles (so their first
          // wedges strictly increase) and gives each one's first flattened wedge
          uint32_t len2[kMPT], wv2[kMPT], s2[kMPT];
  #pragma unroll
          for (int q = 0; q < kMPT; ++q) {
            const uint32_t i = kMPT * tid + q;
            wv2[q] = 0;
            s2[q] = 0;
            len2[q] = 0;
            if (i < mc) {
              wv2[q] = a.adj[m_lo + r0 + i];
              s2[q] = a.ub[m_lo + r0 + i];
              uint32_t en = a.end1[ob + (wv2[q] & kMask)];
              if (a.ue) en = min(en, a.ue[m_lo + r0 + i]);  // route 3: the ends before x's own entry
              len2[q] = en > s2[q] ? en - s2[q] : 0;
            }
          }
          uint32_t tsum = 0;
  #pragma unroll
          for (int q = 0; q < kMPT; ++q) tsum += (len2[q] << 12) | (len2[q] > 0 ? 1u : 0u);
          const uint32_t wincl = warp_incl_scan(tsum, lane);
          if (lane == 31) sh_wsum[warp] = wincl;
          __syncthreads();
          uint32_t wbase = 0;
          for (int w2 = 0; w2 < warp; ++w2) wbase += sh_wsum[w2];
          const uint32_t ex = wbase + wincl - tsum;  // (wedges before << 12) | non-empty middles before
          {
            uint32_t k = ex & 0xfffu, pos = ex >> 12;
  #pragma unroll
            for (int q = 0; q < kMPT; ++q) {
              if (len2[q]) {
                mP[k] = pos; mS[k] = s2[q]; mW[k] = wv2[q];
                if (a.edge) mE[k] = m_lo + r0 + kMPT * tid + q;
                if (pass == 1) { mB[k] = 0; mN[k] = 0; }
                ++k;
                pos += len2[q];
              }
            }
          }
          if (tid == kT2Threads - 1) { sh_mcc = (ex + tsum) & 0xfffu; mP[(ex + tsum) & 0xfffu] = (ex + tsum) >> 12; }
          __syncthreads();
        }
        const uint32_t mcc = sh_mcc;  // non-empty middles of the round
        const uint32_t T = mP[mcc];
        // each warp takes a contiguous range of 32-wedge steps; a lane's middle = the middle owning
        // the previous step's last wedge + the middles starting in this step at or before the lane
        const uint32_t nsteps = (T + 31) / 32, per = (nsteps + kT2Warps - 1) / kT2Warps;
        const uint32_t st0 = min(nsteps, per * warp), st1 = min(nsteps, st0 + per);
        int carry = -1;
        if (st0 < st1 && st0 > 0) {  // owner of wedge 32 * st0 - 1: last middle starting at or before it
          uint32_t lo = 0, hi = mcc - 1;
          const uint32_t t0 = 32u * st0 - 1u;
          while (lo < hi) {
            const uint32_t md = (lo + hi + 1) >> 1;
            if (mP[md] <= t0) lo = md; else hi = md - 1;
          }
          carry = (int)lo;
        }
        for (uint32_t stp = st0; stp < st1; ++stp) {
          const uint32_t base = 32u * stp, t = base + lane;
          const uint32_t nx = (uint32_t)(carry + 1) + lane;
          const uint32_t nstart = nx < mcc ? mP[nx] : 0xffffffffu;
          const uint32_t smask = __reduce_or_sync(0xffffffffu, nstart < base + 32u ? 1u << (nstart - base) : 0u);
          const uint32_t mm = smask & (0xffffffffu >> (31 - lane));
          const uint32_t j = (uint32_t)(carry + __popc(mm));
          carry += __popc(smask);
          uint32_t b2 = 0, n2 = 0;
          if (t < T) {
            const uint32_t ev = a.adj[mS[j] + (t - mP[j])];
            const uint32_t l = ev & kMask;
            const uint32_t cls = (ev ^ mW[j]) >> 31;
            const uint32_t key = l + 1;
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
              const uint32_t v = vals[h];
              const uint32_t ad = v & 0xffffu, dd = v >> 16;
              b2 = cls ? dd - 1 : ad - 1;
              n2 = cls ? ad : dd;
            }
          }
          if (pass == 1 && __any_sync(0xffffffffu, (b2 | n2) != 0)) {
            // lanes' middles are non-decreasing: sum each run of equal j, its last lane adds it
            const int gs = mm ? 31 - __clz(mm) : 0;
            uint32_t sb2, sn2;
            seg_sums2(b2, n2, gs, lane, sb2, sn2);
            const bool last = t < T && (lane == 31 || t + 1 == T || ((smask >> (lane + 1)) & 1u));
            if (last && (sb2 | sn2)) {
              if (sb2) atomicAdd(&mB[j], sb2);
              if (sn2) atomicAdd(&mN[j], sn2);
            }
          }
        }
        __syncthreads();
        if (pass == 1) {
          for (uint32_t i = tid; i < mcc; i += kT2Threads) {
            const uint32_t cb = mB[i], cn = mN[i];
            if (cb | cn) mid_red(a, a.rmid[xu ? 1 : 0], mW[i] & kMask, ob + (mW[i] & kMask), cb, cn, a.edge ? mE[i] : 0u);
          }
          __syncthreads();
        }
      }
    }
    // ---- epilogue: Lemma 2 per end (Alg. 2 lines 15-18), clear
    unsigned long long xB = 0, xN = 0;
    for (uint32_t k = tid; k < S; k += kT2Threads) {
      const uint32_t key = keys[k];
      if (!key) continue;
      const uint32_t v = vals[k];
      keys[k] = 0;
      vals[k] = 0;
      const uint32_t A = v & 0xffffu, D = v >> 16;
      const uint32_t fb = ((A * (A - 1u)) >> 1) + ((D * (D - 1u)) >> 1), fn = A * D;
      if (!(fb | fn)) continue;
      xB += fb;
      xN += fn;
      const uint32_t wrow = sb + key - 1;
      if (PV) end_red(a, a.rsafe[sb ? 1 : 0], key - 1, wrow, fb, fn);
      if (PAIRS && fb) emit_pair(a, x, wrow, fb, fn);
    }
    totB += xB;
    totN += xN;
    if (PV) {
      const unsigned long long b = warp_sum(xB), nn = warp_sum(xN);
      if (lane == 0) { sh_red[0][warp] = b; sh_red[1][warp] = nn; }
      __syncthreads();
      if (warp == 0) {
        const unsigned long long bb = warp_sum(lane < kT2Warps ? sh_red[0][lane] : 0ull);
        const unsigned long long n2 = warp_sum(lane < kT2Warps ? sh_red[1][lane] : 0ull);
        if (lane == 0 && (bb | n2) && !a.edge) {
          atomicAdd(&a.pv[2ull * x], bb);
          atomicAdd(&a.pv[2ull * x + 1], n2);
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

template <bool PV, bool PAIRS, int ENC>
cudaError_t launch_engine(bbf_graph* g, const EngineArgs& ea, cudaStream_t st, Plan* p,
                          cudaEvent_t e0, cudaEvent_t e1, cudaEvent_t e2) {
  const size_t smem3 = sizeof(uint32_t) * (kWin + kBm + 3 * kMaxWin);
  const size_t smem1 = sizeof(uint32_t) * 32 * (2 * 256 + 3 * 32 + 64);
  const size_t smem1b = sizeof(uint32_t) * 12 * (2 * 1024 + 3 * 32 + 64);
  cudaError_t err;
  err = cudaFuncSetAttribute(k_t3<PV, PAIRS, ENC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3);
  if (err != cudaSuccess) return err;
  err = cudaFuncSetAttribute(k_t1<PV, PAIRS, 32, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
  if (err != cudaSuccess) return err;
  err = cudaFuncSetAttribute(k_t1<PV, PAIRS, 12, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1b);
  if (err != cudaSuccess) return err;
  cudaEventRecord(e0, st);
  if (p->n_units) {
    k_t3<PV, PAIRS, ENC><<<g->num_sms * kT3Ctas, kT3Threads, smem3, st>>>(ea);
    g->launches++;
  }
  cudaEventRecord(e1, st);
  if (p->n_t1) {
    EngineArgs e1a = ea;
    e1a.t1 = p->t1; e1a.n_t1 = p->n_t1; e1a.t1ctr = 3;
    k_t1<PV, PAIRS, 32, 256><<<g->num_sms * 2, 32 * 32, smem1, st>>>(e1a);
    g->launches++;
  }
  if (p->n_t1b) {
    EngineArgs e1b = ea;
    e1b.t1 = p->t1b; e1b.n_t1 = p->n_t1b; e1b.t1ctr = 18;
    k_t1<PV, PAIRS, 12, 1024><<<g->num_sms * 2, 12 * 32, smem1b, st>>>(e1b);
    g->launches++;
  }
  if (p->n_t2) {
    EngineArgs eb = ea;
    eb.t2 = p->t2; eb.n_t2 = p->n_t2; eb.t2ctr = 16;
    // one middle per thread per round: 74 KB of shared memory, so three CTAs fit an SM (75% of
    // the warp slots; with two middles per thread it was 86 KB, two CTAs)
    const size_t smem2 = sizeof(uint32_t) * (2 * kT2Slots + 5 * 512 + 1 + (ea.edge ? 512 : 0));
    err = cudaFuncSetAttribute(k_t2<PV, PAIRS, 512, kT2Slots, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
    if (err != cudaSuccess) return err;
    k_t2<PV, PAIRS, 512, kT2Slots, 1><<<g->num_sms * 3, 512, smem2, st>>>(eb);
    g->launches++;
  }
  if (p->n_t2h) {
    EngineArgs eh = ea;
    eh.t2 = p->t2h; eh.n_t2 = p->n_t2h; eh.t2ctr = 19;
    const size_t smem2 = sizeof(uint32_t) * (2 * kT2HugeSlots + 5 * 2048 + 1 + (ea.edge ? 2048 : 0));
    err = cudaFuncSetAttribute(k_t2<PV, PAIRS, 1024, kT2HugeSlots, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
    if (err != cudaSuccess) return err;
    k_t2<PV, PAIRS, 1024, kT2HugeSlots, 2><<<g->num_sms, 1024, smem2, st>>>(eh);
    g->launches++;
  }
  if (p->n_t2s) {
    EngineArgs es = ea;
    es.t2 = p->t2s; es.n_t2 = p->n_t2s; es.t2ctr = 17;
    const size_t smem2 = sizeof(uint32_t) * (kT2Slots + 5 * 512 + 1 + (ea.edge ? 512 : 0));
    err = cudaFuncSetAttribute(k_t2<PV, PAIRS, 256, kT2Slots / 2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
    if (err != cudaSuccess) return err;
    k_t2<PV, PAIRS, 256, kT2Slots / 2, 2><<<g->num_sms * 5, 256, smem2, st>>>(es);
    g->launches++;
  }
  cudaEventRecord(e2, st);
  return cudaGetLastError();
}

}  // namespace

bbf_status run_sparse_impl(bbf_graph* g, Plan* p, bool per_vertex, bool pairs, int rank,
                           int nranks, unsigned long long* host_BN, unsigned long long* cb,
                           unsigned long long* cn, unsigned long long* cid,
                           unsigned long long cap, unsigned long long* n_cand, unsigned long long tau,
                           unsigned long long* edge) {
  NvtxRange nvtx_("bbf::sparse_engine");
  cudaStream_t st = g->stream;
  if (edge && (!per_vertex || pairs)) {
    set_error("internal: per-edge counts need a per-vertex pass");
    return BBF_ECUDA;
  }
  // scratch for the hub kernel: per CTA 3 middle arrays + 4 record arrays [window][middle]
  uint32_t kwin_cap = 1;
  for (int s2 = 0; s2 < 2; ++s2)
    kwin_cap = std::max<uint32_t>(kwin_cap, (g->zones[s2].WB[5] + kWin - 1) / kWin);
  if (kwin_cap > kMaxWin) {
    set_error("end side too large for the hub kernel's window table");
    return BBF_ERANGE;
  }
  size_t mm = std::max<uint32_t>(p->max_mid, 1);
  size_t rs = mm + p->max_work / kRecMax + 1;
  size_t need = (size_t)g->num_sms * kT3Ctas * 4 * rs * kwin_cap;  // 16-B records [window][slot]
  if (need > g->scratch_words) {
    if (g->scratch) dfree(g->scratch, st);
    g->scratch = nullptr;
    BBF_CUDA(dmalloc(&g->scratch, need * sizeof(uint32_t), st));
    g->scratch_words = need;
  }
  BBF_CUDA(cudaMemsetAsync(g->d_acc, 0, 32 * sizeof(unsigned long long), st));
  EngineArgs ea{};
  ea.off = g->off; ea.adj = g->adj; ea.adjc = g->adjc; ea.runid = g->runid; ea.runs = g->runs;
  ea.rlast = g->rlast;
  ea.nruns = g->nruns; ea.mid = p->route == 0 ? g->mid : nullptr; ea.end1 = g->end1;
  ea.ub = p->ub; ea.work = p->work; ea.inv = g->inv; ea.t1 = p->t1; ea.t2 = p->t2; ea.units = p->units;
  ea.cut_tab = p->cut_tab; ea.unit_cut = p->cut_tab ? p->unit_cut : nullptr;
  ea.n_t1 = p->n_t1; ea.n_t2 = p->n_t2; ea.n_units = p->n_units; ea.n_u = g->n_u; ea.n = g->n;
  ea.z[0] = g->zones[0]; ea.z[1] = g->zones[1];
  ea.rank = rank; ea.nranks = nranks;
  ea.acc = g->d_acc; ea.pv = (unsigned long long*)g->pv; ea.scratch = g->scratch;
  ea.pe = (unsigned long long*)g->pe;
  ea.rsafe[0] = per_vertex ? p->rsafe[0] : 0xffffffffu;
  ea.rsafe[1] = per_vertex ? p->rsafe[1] : 0xffffffffu;
  ea.pm = (unsigned long long*)g->pm;
  ea.rmid[0] = per_vertex ? p->rmid[0] : 0xffffffffu;
  ea.rmid[1] = per_vertex ? p->rmid[1] : 0xffffffffu;
  ea.max_mid = std::max<uint32_t>(p->max_mid, 1);
  ea.kwin_cap = kwin_cap;
  ea.rec_stride = (uint32_t)(std::max<uint32_t>(p->max_mid, 1) + p->max_work / kRecMax + 1);
  ea.cb = cb; ea.cn = cn; ea.cid = cid; ea.cap = cap; ea.tau = tau;
  ea.edge = edge;
  ea.ue = p->route == 3 ? g->rev : nullptr;
  ea.dense_div = getenv("BBF_DENSE_DIV") ? (uint32_t)atoi(getenv("BBF_DENSE_DIV")) : 2u;
  // hub-kernel record batch: 32 amortises the batch set-up when each CTA has a long share of the
  // hub wedges (config 5: -1.3% k_t3), 16 balances the tail of a short one (config 3: 32 is +3%)
  const uint64_t w_per_cta = p->W_t3 / ((uint64_t)g->num_sms * kT3Ctas * (uint64_t)std::max(1, nranks));
  ea.bsz = getenv("BBF_T3_BSZ") ? (uint32_t)std::min(32, std::max(0, atoi(getenv("BBF_T3_BSZ"))))
                                : (w_per_cta > (1ull << 24) ? 32u : 16u);
  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
  cudaError_t err;
  const bool wide = g->zones[0].L[0] > 0 || g->zones[1].L[0] > 0;  // some degree > 65535
  const int enc = g->compact ? kEncCompact : wide ? kEncWide : kEncNarrow;
  if (enc == kEncCompact) {
    if (pairs) err = launch_engine<false, true, kEncCompact>(g, ea, st, p, e0, e1, e2);
    else if (per_vertex) err = launch_engine<true, false, kEncCompact>(g, ea, st, p, e0, e1, e2);
    else err = launch_engine<false, false, kEncCompact>(g, ea, st, p, e0, e1, e2);
  } else if (enc == kEncWide) {
    if (pairs) err = launch_engine<false, true, kEncWide>(g, ea, st, p, e0, e1, e2);
    else if (per_vertex) err = launch_engine<true, false, kEncWide>(g, ea, st, p, e0, e1, e2);
    else err = launch_engine<false, false, kEncWide>(g, ea, st, p, e0, e1, e2);
  } else {
    if (pairs) err = launch_engine<false, true, kEncNarrow>(g, ea, st, p, e0, e1, e2);
    else if (per_vertex) err = launch_engine<true, false, kEncNarrow>(g, ea, st, p, e0, e1, e2);
    else err = launch_engine<false, false, kEncNarrow>(g, ea, st, p, e0, e1, e2);
  }
  if (err != cudaSuccess) {
    cudaEventDestroy(e0); cudaEventDestroy(e1); cudaEventDestroy(e2);
    return cuda_status(err, "sparse engine launch");
  }
  if (per_vertex && (p->rsafe[0] != 0xffffffffu || p->rsafe[1] != 0xffffffffu || p->rmid[0] != 0xffffffffu ||
                     p->rmid[1] != 0xffffffffu) && g->n) {
    k_merge_pe<<<(g->n + 255) / 256, 256, 0, st>>>((unsigned long long*)g->pe, (unsigned long long*)g->pm,
                                                  (unsigned long long*)g->pv, g->n);
    g->launches++;
  }
  unsigned long long h[16];
  BBF_CUDA(rb_add(h, g->d_acc, sizeof(h), st)); g->launches++;
  BBF_CUDA(rb_sync(st));
  float ms1 = 0, ms2 = 0;
  cudaEventElapsedTime(&ms1, e0, e1);
  cudaEventElapsedTime(&ms2, e1, e2);
  cudaEventDestroy(e0); cudaEventDestroy(e1); cudaEventDestroy(e2);
  g->ms_main = ms1;
  host_BN[0] = h[0];
  host_BN[1] = h[1];
  if (n_cand) *n_cand = h[4];
#ifdef BBF_RED_PROF
  {
    unsigned long long rc[8];
    cudaMemcpyFromSymbol(rc, g_red_cnt, sizeof(rc));
    fprintf(stderr, "[bbf] REDs (cumulative): end unpacked %llu packed %llu (rank<1024 %llu, <8192 %llu); mid unpacked %llu packed %llu (rank<1024 %llu)\n",
            rc[0], rc[1], rc[2], rc[3], rc[4], rc[5], rc[6]);
  }
#endif
  if (getenv("BBF_DEBUG"))
    fprintf(stderr,
            "[bbf] engine: t3 %.3f ms, t1 %.3f ms, records %llu, windows %llu (small %llu, dense %llu), "
            "pass-1 steps %llu chunks %llu (lane use %.1f%%)\n",
            ms1, ms2, h[6], h[7], h[9], h[10], h[5], h[8], 100.0 * h[8] / (32.0 * (h[5] ? h[5] : 1)));
#ifdef BBF_T3_PROF
  {
    const double clk = 1.965e6 * g->num_sms * kT3Ctas;  // cycles per ms summed over CTAs
    fprintf(stderr, "[bbf] t3 phases (ms of CTA time): prescan %.2f setup %.2f pass1 %.2f pass2 %.2f epi %.2f\n",
            h[11] / clk, h[12] / clk, h[13] / clk, h[14] / clk, h[15] / clk);
    unsigned long long t[3];
    cudaMemcpyFromSymbol(t, g_prof_t, sizeof(t));
    fprintf(stderr, "[bbf] t3 CTA ends: first %.3f ms, last %.3f ms after the first start\n", (t[1] - t[0]) * 1e-6,
            (t[2] - t[0]) * 1e-6);
    unsigned long long pc[128];
    cudaMemcpyFromSymbol(pc, g_prof_cnt, sizeof(pc));
    const char* bn[6] = {"<2K", "<8K", "<32K", "<128K", "<512K", ">=512K"};
    for (int b = 0; b < 6; ++b)
      if (pc[16 + 3 * b])
        fprintf(stderr, "[bbf] t3 windows %-7s n %8llu wedges %.3e  ms(CTA) %7.2f  cyc/window %8.0f  wedges/cyc %.2f\n", bn[b],
                pc[16 + 3 * b], (double)pc[17 + 3 * b], pc[18 + 3 * b] / (1.965e6 * g->num_sms * kT3Ctas),
                pc[18 + 3 * b] / (double)pc[16 + 3 * b], pc[17 + 3 * b] / (double)(pc[18 + 3 * b] + 1));
    const char* ubn[5] = {"<16K", "<64K", "<256K", "<1M", ">=1M"};
    for (int b = 0; b < 5; ++b)
      if (pc[64 + 4 * b])
        fprintf(stderr, "[bbf] t3 units %-6s n %7llu wedges %.3e windows/unit %5.1f  ms(CTA) %7.2f  wedges/cyc %.2f\n", ubn[b],
                pc[64 + 4 * b], (double)pc[65 + 4 * b], pc[66 + 4 * b] / (double)pc[64 + 4 * b],
                pc[67 + 4 * b] / (1.965e6 * g->num_sms * kT3Ctas), pc[65 + 4 * b] / (double)(pc[67 + 4 * b] + 1));
    for (int b = 0; b < 6; ++b)
      if (pc[16 + 3 * b]) {  // cumulative marks: end of pass 1, end of pass 2, end of epilogue
        const double n = (double)pc[16 + 3 * b];
        fprintf(stderr, "[bbf] t3 windows %-7s cyc/window pass1 %8.0f pass2 %8.0f epi %8.0f\n", bn[b], pc[40 + 3 * b] / n,
                (pc[41 + 3 * b] - pc[40 + 3 * b]) / n, (pc[42 + 3 * b] - pc[41 + 3 * b]) / n);
      }
    fprintf(stderr, "[bbf] t3 records %llu entries %llu blocks64 %llu (fill %.3f) blocks32 %llu (fill %.3f) blocks16 %llu "
            "(fill %.3f) short<8 %llu, entries in records<64 %llu; wedges dense %llu bitmap %llu\n",
            pc[10], pc[0], pc[1], pc[0] / (64.0 * pc[1] + 1e-9), pc[2], pc[0] / (32.0 * pc[2] + 1e-9), pc[3],
            pc[0] / (16.0 * pc[3] + 1e-9), pc[4], pc[5], pc[6], pc[7]);
    fprintf(stderr, "[bbf] t3 pass-2 long-record entries %llu, with a + d >= 2 at the end: %llu (%.3f)\n", pc[20], pc[21],
            pc[21] / (pc[20] + 1e-9));
    fprintf(stderr, "[bbf] t3 pre-scan middles: split units %llu (non-empty %llu), whole starts %llu\n", pc[84], pc[85], pc[86]);
    fprintf(stderr, "[bbf] t3 entries by run length: <8 %.3f <32 %.3f <128 %.3f <512 %.3f >=512 %.3f\n",
            pc[11] / (double)pc[0], pc[12] / (double)pc[0], pc[13] / (double)pc[0], pc[14] / (double)pc[0],
            pc[15] / (double)pc[0]);
#ifdef BBF_T3_LATPROF
    for (int ps = 0; ps < 2; ++ps)
      fprintf(stderr, "[bbf] t3 tiny windows pass %d (cycles after the window start): warp reaches batches %.0f (n %llu), first batch records %.0f (n %llu), first chunks done %.0f (n %llu), working warp done %.0f (n %llu), barrier exit %.0f (n %llu)\n",
              ps, pc[106 + ps] / (double)(pc[108 + ps] + 1), pc[108 + ps], pc[96 + ps] / (double)(pc[98 + ps] + 1), pc[98 + ps],
              pc[100 + ps] / (double)(pc[110 + ps] + 1), pc[110 + ps], pc[102 + ps] / (double)(pc[112 + ps] + 1), pc[112 + ps],
              pc[104 + ps] / (double)(pc[114 + ps] + 1), pc[114 + ps]);
#endif
#ifdef BBF_T3_BUSYPROF
    {
      const char* bn2[6] = {"<2K", "<8K", "<32K", "<128K", "<512K", ">=512K"};
      for (int b = 0; b < 6; ++b) {
        const double span = (double)pc[96 + 4 * b + 2] + 1;
        fprintf(stderr, "[bbf] t3 busy %-7s passes %8llu: long-record phase %.3f, short batches %.3f, barrier wait %.3f of warp-cycles\n",
                bn2[b], pc[96 + 4 * b + 3], pc[96 + 4 * b] / span, pc[96 + 4 * b + 1] / span,
                1.0 - (pc[96 + 4 * b] + pc[96 + 4 * b + 1]) / span);
      }
    }
#endif
    const unsigned long long z40[128] = {};
    cudaMemcpyToSymbol(g_prof_cnt, z40, sizeof(z40));
    const unsigned long long init[3] = {~0ull, ~0ull, 0ull};
    cudaMemcpyToSymbol(g_prof_t, init, sizeof(init));
  }
#endif
  // algorithmic bytes of the hub kernel k_t3: 4 B column word per
  // visited wedge per pass (pass 2 re-reads it for per-vertex counts) + 16 B per eligible
  // middle of its starts (column word, ub, end1 of the middle's row, 4 B id-side output)
  g->algo_bytes = 4ull * p->W_t3 * (per_vertex ? 2 : 1) + 16ull * p->M_t3;
  g->algo_ops = 0;
  return BBF_OK;
}

bbf_status run_sparse(bbf_graph* g, Plan* p, bool per_vertex, int rank, int nranks,
                      unsigned long long* host_BN) {
  return run_sparse_impl(g, p, per_vertex, false, rank, nranks, host_BN, nullptr, nullptr, nullptr,
                         0, nullptr, 1ull);
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
// two stable radix sorts (ids ascending, then balanced descending).  With nranks > 1 this rank
// counts only its shard of the work items (shard_item: snake order over ranks; every pair is produced by
// exactly one item: its start's unit that holds the end's window) and returns the shard's own
// top-k; api.cu all-gathers the shards' lists and merges them (the global top-k is a subset of
// the union of the shards' top-k lists).
bbf_status run_pairs_topk(bbf_graph* g, int side, uint32_t k, bbf_pair* out, uint32_t* n_out, int rank,
                          int nranks) {
  NvtxRange nvtx_("bbf::pairs_topk");
  cudaStream_t st = g->stream;
  Plan* p = &g->plan_s[side];
  if (p->valid && p->nranks != nranks) free_plan(p, st);  // hub units are sized per rank count
  if (!p->valid) BBF_TRY(make_plan(g, 1 + side, p));
  // Candidates are the pairs with balanced >= tau (reading R11 ranks by balanced count).  tau
  // starts at 1 (every pair with a balanced butterfly); if the candidates overflow the buffer,
  // tau is raised to the (4k)-th largest balanced count among the stored ones and the pass is
  // repeated; if a raised tau leaves fewer than k candidates it is lowered 16x and repeated.
  unsigned long long cap = std::min<unsigned long long>(p->W_pruned + 1024, 1ull << 24);
  if (getenv("BBF_TOPK_CAP")) cap = std::max<unsigned long long>(k, strtoull(getenv("BBF_TOPK_CAP"), nullptr, 10));  // test hook
  unsigned long long ncand = 0, tau = 1;
  unsigned long long lo = 0, lo_count = 0;  // largest tau seen to overflow the buffer (0: none)
  unsigned long long hi = 0;                // smallest tau seen to leave fewer than k (0: none)
  unsigned long long *cb = nullptr, *cn = nullptr, *cid = nullptr;
  BBF_CUDA(dmalloc(&cb, 8 * cap, st));
  BBF_CUDA(dmalloc(&cn, 8 * cap, st));
  BBF_CUDA(dmalloc(&cid, 8 * cap, st));
  // the (r+1)-th largest of the first min(n, cap) stored balanced counts (device sort, one read)
  auto kth_stored = [&](unsigned long long nstored, size_t r, unsigned long long* val) -> bbf_status {
    const int ns = (int)std::min<unsigned long long>(nstored, cap);
    unsigned long long* srt;
    BBF_CUDA(dmalloc(&srt, 8ull * ns + 8, st));
    size_t ts = 0;
    cub::DeviceRadixSort::SortKeysDescending(nullptr, ts, cb, srt, ns, 0, 64, st);
    void* tmps;
    BBF_CUDA(dmalloc(&tmps, ts + 16, st));
    BBF_CUDA(cub::DeviceRadixSort::SortKeysDescending(tmps, ts, cb, srt, ns, 0, 64, st));
    g->launches += kCubSortKernels64;
    BBF_CUDA(cudaMemcpyAsync(val, srt + std::min<size_t>(r, (size_t)ns - 1), 8, cudaMemcpyDeviceToHost, st));
    BBF_CUDA(cudaStreamSynchronize(st));
    dfree(srt, st);
    dfree(tmps, st);
    return BBF_OK;
  };
  // Starting threshold from a sample: when a pass at tau = 1 could overflow the buffer, count
  // 1/16 of the work items first (the shard of one rank in a 16x larger fake world) and start at
  // the (4k)-th largest balanced count among the sample's pairs — about 64k pairs of the whole
  // set reach it, so the full pass usually stores a complete candidate set at once.  Any start is
  // correct: the loop below only stops on a complete set of at least k candidates (or tau = 1).
  if (p->W_pruned > cap && !getenv("BBF_TOPK_NO_SAMPLE")) {  // env: test hook
    unsigned long long BN[2];
    BBF_TRY(run_sparse_impl(g, p, false, true, rank, nranks * 16, BN, cb, cn, cid, cap, &ncand, 1));
    if (ncand >= 4ull * k) BBF_TRY(kth_stored(ncand, 4ull * k - 1, &tau));
    if (tau < 1) tau = 1;
  }
  for (int it = 0;; ++it) {
    unsigned long long BN[2];
    BBF_TRY(run_sparse_impl(g, p, false, true, rank, nranks, BN, cb, cn, cid, cap, &ncand, tau));
    if (ncand <= cap && (ncand >= k || tau == 1)) break;  // complete candidate set
    if (it >= 64) { set_error("top-k threshold search did not converge"); return BBF_ENOMEM; }
    if (ncand > cap) {
      lo = tau;
      lo_count = ncand;
      // the stored candidates are a subset: their (4k)-th largest balanced count bounds tau
      // (a device sort of the stored counts, then one element read back)
      unsigned long long kth = 0;
      BBF_TRY(kth_stored(cap, std::min<size_t>(cap - 1, 4ull * k), &kth));
      tau = std::max(tau + 1, kth);
    } else {
      hi = tau;  // too few candidates at this threshold
    }
    if (hi && tau >= hi) tau = lo + (hi - lo) / 2;
    if (tau <= lo) tau = lo + 1;
    if (hi && tau >= hi) {
      // ties: no integer threshold separates "too many" from "too few"; take every candidate at
      // tau = lo in a buffer of the exact size
      dfree(cb, st); dfree(cn, st); dfree(cid, st);
      cap = lo_count;
      if (cap >= (1ull << 31)) { set_error("top-k: too many tied candidates"); return BBF_ENOMEM; }
      BBF_CUDA(dmalloc(&cb, 8 * cap, st));
      BBF_CUDA(dmalloc(&cn, 8 * cap, st));
      BBF_CUDA(dmalloc(&cid, 8 * cap, st));
      tau = lo;
      BBF_TRY(run_sparse_impl(g, p, false, true, rank, nranks, BN, cb, cn, cid, cap, &ncand, tau));
      break;
    }
  }
  uint32_t take = (uint32_t)std::min<unsigned long long>(k, ncand);
  *n_out = take;
  if (take == 0) {
    dfree(cb, st); dfree(cn, st); dfree(cid, st);
    BBF_CUDA(cudaStreamSynchronize(st));
    return BBF_OK;
  }
  const int nc = (int)ncand;
  uint32_t *idx0, *idx1, *idx2;
  unsigned long long *kid, *kb, *kb2;
  BBF_CUDA(dmalloc(&idx0, 4ull * nc, st));
  BBF_CUDA(dmalloc(&idx1, 4ull * nc, st));
  BBF_CUDA(dmalloc(&idx2, 4ull * nc, st));
  BBF_CUDA(dmalloc(&kid, 8ull * nc, st));
  BBF_CUDA(dmalloc(&kb, 8ull * nc, st));
  BBF_CUDA(dmalloc(&kb2, 8ull * nc, st));
  k_iota<<<256, 256, 0, st>>>(idx0, ncand);
  size_t t1 = 0, t2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t1, cid, kid, idx0, idx1, nc, 0, 64, st);
  cub::DeviceRadixSort::SortPairsDescending(nullptr, t2, kb, kb2, idx1, idx2, nc, 0, 64, st);
  void* tmp;
  BBF_CUDA(dmalloc(&tmp, std::max(t1, t2) + 16, st));
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
  for (void* q : fr) dfree(q, st);
  BBF_CUDA(cudaStreamSynchronize(st));
  return BBF_OK;
}

}  // namespace bbf
