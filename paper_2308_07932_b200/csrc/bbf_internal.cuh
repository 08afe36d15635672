// bbf_internal.cuh — device representation and shared helpers of libbbf.so (sm_100a).
//
// Rank space (DESIGN.md §"Data layout in HBM"):
//   * every vertex gets a local rank l on its own side: position in descending priority order
//     (degree desc, then global id desc) — Def. Vertex Priority.  Same-side
//     priority comparisons are comparisons of l; cross-side comparisons happen once per edge
//     at build time (mid_start).
//   * rows: U rows 0..n_u-1 (row = l), V rows n_u..n-1 (row = n_u + l).
//   * adj[2*nnz]: column word = l(y) | neg << 31, rows sorted ascending by l(y), i.e. by
//     descending priority (Alg. 2 line 3, "Rearrange Γ(u) ... in ascending order", PAPER.md:747,
//     with our rank running opposite to p).  Every compare masks bit 31.
//   * mid_start[x]: first entry whose neighbour has lower priority than x (p(v) < p(u),
//     PAPER.md:753): the eligible middles are the suffix [mid_start[x], end1[x]).
//   * end1[x]: first entry whose neighbour has degree <= 1.  Such a vertex lies on no 4-cycle,
//     so wedges ending (or centred) there contribute to no count (DESIGN.md §"Pruning").
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <string>

#include "../../include/bbf.h"

// NVTX range over a host-side phase (build, plan, engine, collective): header-only NVTX3, a no-op
// unless a profiler (nsys, ncu --nvtx) is attached
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

namespace bbf {

constexpr uint32_t kMask = 0x7fffffffu;
constexpr uint32_t kNegBit = 0x80000000u;

// ---------------------------------------------------------------------------- counter zones
// Per end side, the end-vertex rank space [0, L4) is cut into zones by degree; a same-side
// pair (x, w) has a + d <= deg(w) (each wedge x-v-w uses a distinct middle v in N(w)), so the
// packed (a, d) field of w needs only bits for deg(w):
//   zone 0: deg > 65535    64-bit field (a word, d word)
//   zone 1: 256..65535     32-bit field (a:16 | d:16)
//   zone 2: 16..255        16-bit field (a:8  | d:8 )
//   zone 3: 4..15           8-bit field (a:4  | d:4 )
//   zone 4: 2..3            4-bit field (a:2  | d:2 )
//   deg <= 1: no counter (never on a butterfly).
struct Zones {
  uint32_t L[5];   // L[z] = first rank past zone z (cumulative): L[0]=#deg>65535 ... L[4]=#deg>=2
  uint32_t WB[6];  // word base of each zone; WB[5] = total words
};

__host__ __device__ inline uint32_t zone_of_l(const Zones& z, uint32_t l) {
  return (l < z.L[0]) ? 0 : (l < z.L[1]) ? 1 : (l < z.L[2]) ? 2 : (l < z.L[3]) ? 3 : 4;
}

// global word of field l (base word for zone 0), shift within word, and increment for class
__device__ __forceinline__ void field_of(const Zones& z, uint32_t l, uint32_t cls, uint32_t& base,
                                         uint32_t& word, uint32_t& inc) {
  if (l < z.L[0]) {
    base = 2u * l;
    word = base + cls;
    inc = 1u;
  } else if (l < z.L[1]) {
    base = word = z.WB[1] + (l - z.L[0]);
    inc = 1u << (16u * cls);
  } else if (l < z.L[2]) {
    uint32_t i = l - z.L[1];
    base = word = z.WB[2] + (i >> 1);
    inc = 1u << (((i & 1u) << 4) + 8u * cls);
  } else if (l < z.L[3]) {
    uint32_t i = l - z.L[2];
    base = word = z.WB[3] + (i >> 2);
    inc = 1u << (((i & 3u) << 3) + 4u * cls);
  } else {
    uint32_t i = l - z.L[3];
    base = word = z.WB[4] + (i >> 3);
    inc = 1u << (((i & 7u) << 2) + 2u * cls);
  }
}

// read (a, d) of field l from a window whose first global word is word0
__device__ __forceinline__ void field_read(const Zones& z, const uint32_t* ctr, uint32_t word0,
                                           uint32_t l, uint32_t& a, uint32_t& d) {
  if (l < z.L[0]) {
    uint32_t w = 2u * l - word0;
    a = ctr[w];
    d = ctr[w + 1];
  } else if (l < z.L[1]) {
    uint32_t v = ctr[z.WB[1] + (l - z.L[0]) - word0];
    a = v & 0xffffu;
    d = v >> 16;
  } else if (l < z.L[2]) {
    uint32_t i = l - z.L[1];
    uint32_t v = (ctr[z.WB[2] + (i >> 1) - word0] >> ((i & 1u) << 4)) & 0xffffu;
    a = v & 0xffu;
    d = v >> 8;
  } else if (l < z.L[3]) {
    uint32_t i = l - z.L[2];
    uint32_t v = (ctr[z.WB[3] + (i >> 2) - word0] >> ((i & 3u) << 3)) & 0xffu;
    a = v & 0xfu;
    d = v >> 4;
  } else {
    uint32_t i = l - z.L[3];
    uint32_t v = (ctr[z.WB[4] + (i >> 3) - word0] >> ((i & 7u) << 2)) & 0xfu;
    a = v & 3u;
    d = v >> 2;
  }
}

// first l whose field's last word is >= g (so every l below it fits in words < g)
__host__ __device__ inline uint32_t l_first_last_word_ge(const Zones& z, uint64_t g) {
  if (g >= z.WB[5]) return z.L[4];
  if (g < z.WB[1]) {  // zone 0: last word 2l+1 >= g
    uint64_t l = (g == 0) ? 0 : (g) / 2;  // smallest l with 2l+1 >= g
    return (uint32_t)l;
  }
  if (g < z.WB[2]) return z.L[0] + (uint32_t)(g - z.WB[1]);
  if (g < z.WB[3]) return z.L[1] + (uint32_t)(2ull * (g - z.WB[2]));
  if (g < z.WB[4]) return z.L[2] + (uint32_t)(4ull * (g - z.WB[3]));
  return z.L[3] + (uint32_t)(8ull * (g - z.WB[4]));
}

__host__ __device__ inline uint32_t word_of_l(const Zones& z, uint32_t l) {
  if (l < z.L[0]) return 2u * l;
  if (l < z.L[1]) return z.WB[1] + (l - z.L[0]);
  if (l < z.L[2]) return z.WB[2] + ((l - z.L[1]) >> 1);
  if (l < z.L[3]) return z.WB[3] + ((l - z.L[2]) >> 2);
  return z.WB[4] + ((l - z.L[3]) >> 3);
}

// ---------------------------------------------------------------------------- counter address
// adjc[e] encodes, for the end vertex y of adjacency entry e, where its (a, d) field lives in
// the zoned counter layout of y's side, so the hub kernel never evaluates the zone chain per
// wedge:  bits 0-22 base word g, 23-27 bit shift, 28-29 width code (field 4/8/16/32 bits),
// 30 wide (zone 0: a in word g, d in word g+1), 31 negative sign (as in adj).
constexpr uint32_t kCWordBits = 23;
constexpr uint32_t kCWordMask = (1u << kCWordBits) - 1u;
#ifndef BBF_T3_CTAS
#define BBF_T3_CTAS 1
#endif
constexpr uint32_t kT3Ctas = BBF_T3_CTAS;           // hub-kernel CTAs per SM
constexpr uint32_t kWin = 51 * 1024 / kT3Ctas;      // counter words per hub-kernel window (204 KB)

__host__ __device__ inline uint32_t encode_caddr(const Zones& z, uint32_t l) {
  uint32_t g, sh = 0, wc = 0, wide = 0;
  if (l < z.L[0]) { g = 2u * l; wide = 1; }
  else if (l < z.L[1]) { g = z.WB[1] + (l - z.L[0]); wc = 3; }
  else if (l < z.L[2]) { uint32_t i = l - z.L[1]; g = z.WB[2] + (i >> 1); sh = (i & 1u) << 4; wc = 2; }
  else if (l < z.L[3]) { uint32_t i = l - z.L[2]; g = z.WB[3] + (i >> 2); sh = (i & 3u) << 3; wc = 1; }
  else if (l < z.L[4]) { uint32_t i = l - z.L[3]; g = z.WB[4] + (i >> 3); sh = (i & 7u) << 2; wc = 0; }
  else { g = 0; }  // degree <= 1: never counted
  return (g & kCWordMask) | (sh << 23) | (wc << 28) | (wide << 30);
}

// Compact encoding (graphs without 64-bit fields and at most 2^20 counter words per side):
// bits 0-1 width code wc (half-field h = 2 << wc), 2-21 word g (so ev & kCpAddrMask is the
// word's byte offset 4g), 22-26 P0, 27-31 P1, where P0 / P1 is the bit of the field to
// increment when the start->middle edge is positive / negative: the wedge is symmetric (a, at
// bit sh) iff both edges have the same sign, asymmetric (d, at bit sh + h) otherwise, so the
// middle->end sign is folded into the two positions.
constexpr uint32_t kCpWordBits = 20;
constexpr uint32_t kCpWordMask = (1u << kCpWordBits) - 1u;
constexpr uint32_t kCpAddrMask = kCpWordMask << 2;
__host__ __device__ inline uint32_t cp_word(uint32_t ev) { return (ev >> 2) & kCpWordMask; }

__host__ __device__ inline uint32_t encode_caddr_compact(const Zones& z, uint32_t l, uint32_t neg) {
  uint32_t g = 0, sh = 0, wc = 0;
  if (l < z.L[1]) { g = z.WB[1] + (l - z.L[0]); wc = 3; }
  else if (l < z.L[2]) { uint32_t i = l - z.L[1]; g = z.WB[2] + (i >> 1); sh = (i & 1u) << 4; wc = 2; }
  else if (l < z.L[3]) { uint32_t i = l - z.L[2]; g = z.WB[3] + (i >> 2); sh = (i & 3u) << 3; wc = 1; }
  else if (l < z.L[4]) { uint32_t i = l - z.L[3]; g = z.WB[4] + (i >> 3); sh = (i & 7u) << 2; wc = 0; }
  const uint32_t pa = sh, pd = sh + (2u << wc);
  const uint32_t p0 = neg ? pd : pa, p1 = neg ? pa : pd;
  return ((g & kCpWordMask) << 2) | wc | (p0 << 22) | (p1 << 27);
}

__host__ __device__ inline unsigned long long comb2(unsigned long long x) {
  return x ? x * (x - 1ull) / 2ull : 0ull;
}

// ---------------------------------------------------------------------------- plan
// A "route" is one wedge enumeration the engine runs:
//   route G: Alg. 2, starts = all rows, middles = [mid_start, end1),
//            ends = N(v) ∩ {l(w) > l(x)} ∩ {deg(w) >= 2}.
//   route S(side): same-side pairs with full common neighbourhoods (vBBFC semantics,
//            PAPER.md:875 "we drop the rank comparison"), starts = rows of `side`, middles =
//            [off, end1), ends = l(w) > l(x) (each unordered pair once).
constexpr uint32_t kT2Slots = 8192;               // k_t2 shared hash slots (64 KB)
constexpr uint32_t kT2HugeSlots = 2 * kT2Slots;    // k_t2 1024-thread instance (128 KB hash)
constexpr uint64_t kT2MaxDefault = 10240;  // T2 tier: at most this many wedges per start (swept: 6144..12288)
constexpr uint64_t kT2SmallMax = kT2Slots / 4;   // T2 starts with at most this many wedges use the small k_t2
constexpr uint64_t kT1SmallMax = 128;             // T1 starts with at most this many wedges use the small k_t1
struct Unit {  // one T3 work unit: start row x, end-rank range [lo, hi)
  uint32_t x, lo, hi, pad;
};

struct Plan {
  int route;           // 0 = G, 1 = S(U), 2 = S(V), 3 = S(U) with the ends before the start
  uint32_t* ub;        // per middle entry: first eligible end (absolute adj index)
  uint64_t* work;      // per row: pruned wedge count
  uint32_t* t1;        // rows with 0 < work <= kT1SmallMax (k_t1, 256-slot warp hash)
  uint32_t* t1b;       // rows with kT1SmallMax < work <= kT1Max (k_t1, 1024-slot warp hash)
  uint32_t* t2;        // rows with kT2SmallMax < work <= kT2Slots * 3/4 (k_t2, CTA shared hash)
  uint32_t* t2s;       // rows with kT1Max < work <= kT2SmallMax (k_t2, half-size CTA)
  uint32_t* t2h;       // rows with kT2Slots * 3/4 < work <= T2 max (k_t2, 1024 threads, kT2HugeSlots)
  Unit* units;         // T3 units
  // split hubs: for every boundary between two units of one start, the cut position of each of its
  // middles' end segments (the first entry with rank >= the boundary), computed once in parallel
  // (k_split_cuts) instead of two binary searches per middle in every unit's pre-scan;
  // unit_cut[2i], unit_cut[2i + 1] = offsets of unit i's lower / upper cut array (~0 = none)
  uint32_t* cut_tab;
  unsigned long long* unit_cut;

  uint32_t n_t1, n_t1b, n_t2, n_t2s, n_t2h, n_units;
  uint32_t max_mid;    // max middles of a T3 start
  unsigned long long max_work;  // max wedges of a T3 start
  unsigned long long W_full;    // un-pruned wedge count (route G: W_G of the paper)
  unsigned long long W_pruned;  // wedges the kernels actually visit
  unsigned long long W_t1, W_t2, W_t3;
  unsigned long long M_t3;     // eligible middles of T3 starts
  // end-role packing (route G): ends of local rank >= rsafe[side] have provably < 2^32 end-role
  // balanced and unbalanced totals, so both go in ONE 64-bit RED (fb | fn << 32) into g->pe
  uint32_t rsafe[2];
  // middle-role packing: middles of local rank >= rmid[side] (C(deg,2) * max degree of the
  // other side < 2^32) put (B | N << 32) of a record in ONE 64-bit RED into g->pm
  uint32_t rmid[2];
  int nranks;          // ranks the hub units were sized for
  // hybrid dense-core plan (hybrid.cu): core = side-local ranks < nc[side]; the
  // core wedges (core start, core middle, core end) are skipped (their ub moved past the middle's
  // core ends); {0, 0} = the plain route
  uint32_t nc[2];
  bool valid;
};

// hybrid dense-core state of a graph (hybrid.cu): built once per core size
struct Hybrid {
  uint32_t nc[2];          // core sizes the buffers below were built for ({0,0}: none)
  uint32_t* ccnt;          // n: per row, # entries whose neighbour is in the other side's core
  uint32_t cmaxdeg[2];     // max core degree (entries inside the core) of each side's core rows
  uint32_t nwords[2];      // 32-bit bitmap words per core row of side s (over the other side's core)
  uint32_t* bmA[2];        // core-row bitmaps: neighbour present
  uint32_t* bmN[2];        //                    neighbour present with a negative edge
  uint8_t* A[2];           // u8 dense operands of the core G[C] (rows_pad x k), zero padded
  uint8_t* S[2];
  uint64_t rows_pad[2], k[2];
  uint8_t* A4[2];          // FP4 packed copies (dense_core_side)
  uint8_t* S4[2];
  uint32_t* R[2];          // nc[s] x nc[s] pair words: (a_r | d_r << 16), then (a_c | d_c << 16)
  // fp16 copies for the tensor-core (cuBLAS) form of the mixed-pair terms: A, S and A', S' (the
  // rows masked to each start's eligible core middles), rows_pad x k
  uint16_t* Ah[2];
  uint16_t* Sh[2];
  uint16_t* Aeh[2];
  uint16_t* Seh[2];
  uint8_t* Ae[2];          // u8 A', S' and their FP4 copies (the fused cross-term kernel's I operand)
  uint8_t* Se[2];
  uint8_t* Ae4[2];
  uint8_t* Se4[2];
  bool built;
};

}  // namespace bbf

// ---------------------------------------------------------------------------- graph handle
struct bbf_comm {
  void* nccl;  // ncclComm_t
  int nranks, rank, device;
};

struct bbf_graph {
  int device;
  cudaStream_t stream;
  bool own_stream;
  bbf_comm* comm;
  uint32_t load_flags;  // BBF_FORCE_SPARSE / BBF_FORCE_DENSE given at load: default dispatch
  bool positive_only;   // BBF_POSITIVE_ONLY: negative edges dropped after validation
  uint32_t n_u, n_v, n;
  uint64_t nnz;
  // rank-space CSR
  uint32_t* off;      // n+1
  uint32_t* adj;      // 2*nnz
  uint32_t* erow;     // 2*nnz: row of each entry (plan kernels; no binary search over off)
  uint32_t* rev;      // 2*nnz: position of the same edge's entry in the other side's row
  uint32_t* mid;      // n   (mid_start)
  uint32_t* end1;     // n
  uint32_t* inv;      // n   : row -> input id on its side
  uint32_t* degs;     // n   : degree by row (rank order, per side non-increasing)
  uint64_t* degpre;   // n+2 : per side inclusive prefix of degrees over rows (side-local, see plan)
  bbf::Zones zones[2];
  uint32_t* adjc;     // 2*nnz counter addresses of the end vertex (+ sign bit), see encode_caddr
  uint32_t* runid;    // 2*nnz: index of the window run containing the entry
  uint32_t* rlast;    // n: run index of each row's last entry before end1 (hub pre-scan)
  uint2* runs;        // nruns: {first entry, window id} of every maximal same-window run of a row
  uint32_t nruns;
  bool compact;       // adjc uses encode_caddr_compact (else encode_caddr + sign bit)
  // build state: core arrays always; adjacency (adj, mid, end1, degpre, adjc, runid, runs) built
  // at load for the sparse path, lazily (from the kept input CSR) after a dense load
  uint64_t* skey;     // n   : priority keys deg << 32 | gid sorted descending, U then V
  uint32_t* lr;       // n   : local rank by input id, U ids then V ids
  uint64_t* in_rp;    // device copy of the input CSR, kept only after a dense load
  uint32_t* in_col;
  uint8_t* in_sg;
  bool adj_built;
  bool wg_valid;
  bool dense_cand;    // loaded as a dense-path candidate (W_G computed at load, dense checked first)
  unsigned long long W_G;  // paper wedge count (O(nnz) formula), valid if wg_valid
  // dense operands (dense_i8.cu): per side A (u8 0/1) and S (s8 +-1/0), rows_pad x k_pad
  uint8_t* dA[2];
  uint8_t* dS[2];
  uint64_t drows[2], dk[2];
  uint8_t* dA4[2];           // fp4 (e2m1) packed copies of dA / dS for the block-scaled MMA path
  uint8_t* dS4[2];
  uint64_t dk4[2];            // bytes per fp4 row (K padded to 256 elements, / 2)
  bool dense_built;
  uint32_t rb_err;       // small readback target that outlives one host round trip (build flags)
  bool dense_v_u8;     // the V side's u8 operands are written (else only its FP4 copies)
  uint32_t L4[2];     // #vertices with degree >= 2 per side
  uint32_t Llong[2];  // #vertices with degree > 32 per side ("long" middles of the hub kernel)
  uint32_t maxdeg[2];
  long double ws_bound;  // overflow bound on B + N
  bbf::Plan plan_g;
  bbf::Plan plan_h;     // route G with the hybrid core's wedges skipped
  bbf::Hybrid hyb;
  bool hyb_scored;            // hybrid_choose's candidate scores computed (once per graph)
  uint32_t hyb_pick[2][2];    // chosen core sizes (global, per-vertex); {0, 0} = none
  uint32_t last_nc[2];        // core sizes of the last count (bbf_graph_hybrid_core)
  bbf::Plan plan_s[2];
  bbf::Plan plan_e[2];  // per-edge counts: route S(U) (ends after the start) and route 3 (ends before), all hub tier
  // scratch for the engine
  uint32_t* scratch;  // per-CTA middle arrays
  size_t scratch_words;
  unsigned long long* d_acc;  // [0]=B [1]=N [2..] misc counters, [8]=unit cursor, [9]=t1 cursor
  uint64_t* pv;              // 2*n per-vertex counts, (B, N) interleaved per row: pv[2r], pv[2r+1]
  uint64_t* pe;              // n packed end-role counts (B | N << 32) of "safe" ends, merged into pv
  uint64_t* pm;              // n packed middle-role counts of "safe" middles, merged into pv
  // stats
  uint64_t launches;
  uint64_t algo_bytes;  // algorithmic bytes of the last count's main kernel (sparse path)
  double algo_ops;      // algorithmic int8 ops of the last count's main kernel (dense path)
  float ms_main;
  int num_sms;
};

// error helpers (api.cu)
namespace bbf {
void set_error(const std::string& msg);
bbf_status cuda_status(cudaError_t e, const char* what);
}  // namespace bbf

#define BBF_CUDA(call)                                             \
  do {                                                             \
    cudaError_t e_ = (call);                                       \
    if (e_ != cudaSuccess) return bbf::cuda_status(e_, #call);     \
  } while (0)

#define BBF_TRY(call)                          \
  do {                                         \
    bbf_status s_ = (call);                    \
    if (s_ != BBF_OK) return s_;               \
  } while (0)

// internal entry points across translation units
namespace bbf {
// device-memory cache (mem.cu): stream-ordered like cudaMallocAsync / cudaFreeAsync
cudaError_t dmalloc_raw(void** out, size_t bytes, cudaStream_t st);
cudaError_t dmalloc_raw2(void** out, size_t bytes, cudaStream_t st, bool no_wait);
void dfree(void* p, cudaStream_t st);
// small device->host readbacks (mem.cu): enqueue with rb_add, complete with rb_sync(st), which
// synchronises the stream and then fills the host variables
cudaError_t rb_add(void* host, const void* dev, size_t n, cudaStream_t st);
cudaError_t rb_sync(cudaStream_t st);
// kernels launched by one CUB device-wide call (counted in bbf_graph_stats): a radix sort over
// `bits` key bits = histogram + exclusive sum + one onesweep pass per 8 bits; scans, selects and
// reductions launch two kernels each
constexpr uint32_t cub_sort_kernels(int bits) { return 2u + (uint32_t)((bits + 7) / 8); }
constexpr uint32_t kCubScanKernels = 2, kCubSelectKernels = 2, kCubReduceKernels = 2;
constexpr uint32_t kCubSortKernels64 = 10;  // onesweep radix sort of 64-bit keys: histogram, exclusive sum, 8 passes
template <class T>
inline cudaError_t dmalloc(T** out, size_t bytes, cudaStream_t st) {
  return dmalloc_raw(reinterpret_cast<void**>(out), bytes, st);
}
template <typename T>
cudaError_t dmalloc_nowait(T** out, size_t bytes, cudaStream_t st) {  // see mem.cu
  return dmalloc_raw2(reinterpret_cast<void**>(out), bytes, st, true);
}
bbf_status build_graph(bbf_graph* g, const uint64_t* row_ptr, const uint32_t* col,
                       const uint8_t* sign, bool device_ptrs);
bbf_status validate_csr(const uint64_t* d_rp, uint32_t n_u, const uint32_t* d_col, const uint8_t* d_sg,
                        uint64_t nnz, uint32_t n_v, cudaStream_t st);
bbf_status build_adj(bbf_graph* g, const uint64_t* d_rp, const uint32_t* d_col, const uint8_t* d_sg);
bbf_status ensure_adj(bbf_graph* g);
bbf_status build_dense_operands(bbf_graph* g, const uint64_t* d_rp, const uint32_t* d_col,
                                const uint8_t* d_sg);
bbf_status make_plan(bbf_graph* g, int route, Plan* p, bool all_t3 = false, const uint32_t* nc = nullptr);
void free_plan(Plan* p, cudaStream_t st);
// run the sparse engine for a route; per_vertex -> accumulate into g->pv (rank space)
bbf_status run_sparse(bbf_graph* g, Plan* p, bool per_vertex, int rank, int nranks,
                      unsigned long long* host_BN);
bbf_status run_sparse_impl(bbf_graph* g, Plan* p, bool per_vertex, bool pairs, int rank, int nranks,
                           unsigned long long* host_BN, unsigned long long* cb, unsigned long long* cn,
                           unsigned long long* cid, unsigned long long cap, unsigned long long* n_cand,
                           unsigned long long tau, unsigned long long* edge = nullptr);
bbf_status run_pairs_topk(bbf_graph* g, int side, uint32_t k, bbf_pair* out, uint32_t* n_out, int rank,
                          int nranks);
bbf_status run_dense(bbf_graph* g, bool per_vertex, int rank, int nranks,
                     unsigned long long* host_BN);
// Alg. 1 BB-Base (base.cu): explicit pair checks, the paper's baseline
bbf_status run_base(bbf_graph* g, Plan* p, int rank, int nranks, unsigned long long* host_BN);
bool dense_supported(bbf_graph* g);
// the (rank, nranks) shard of the work this process counts (communicator, or BBF_FAKE_WORLD)
void shard_of(const bbf_graph* g, int* rank, int* nranks);
bool dense_preferred(bbf_graph* g, bool per_vertex);
// hybrid dense core (hybrid.cu): core sizes to use for a count ({0,0} = plain sparse route), and
// the count itself (engine on plan_h + dense core + the mixed-pair correction)
void hybrid_choose(bbf_graph* g, bool per_vertex, uint32_t nc[2]);
bbf_status run_hybrid(bbf_graph* g, const uint32_t nc[2], bool per_vertex, int rank, int nranks,
                      unsigned long long* host_BN);
void free_hybrid(bbf_graph* g);
bbf_status dense_core_cross(bbf_graph* g, uint32_t n_rows, uint64_t rows_pad, uint64_t k, uint8_t* Ae, uint8_t* Se,
                            uint8_t** Ae4, uint8_t** Se4, uint8_t* A, uint8_t* S, uint8_t** A4, uint8_t** S4,
                            uint32_t* R, uint32_t r_ld, uint32_t pv_row0, bool per_vertex, uint32_t xlo,
                            uint32_t xhi, unsigned long long* acc, double* ops);
// one side's pair counts of a dense 0/1 / +-1 operand pair (dense_i8.cu): rows_pad x k u8
// operands, FP4 tensor-core kernels while exact (maxdeg <= 8192), else int8; adds (B, N) into
// acc[0..1] and, when pv, the per-row counts into pv rows pv_row0 + i
bbf_status dense_core_side(bbf_graph* g, uint32_t n_rows, uint64_t rows_pad, uint64_t k, uint8_t* A, uint8_t* S,
                           uint8_t** A4, uint8_t** S4, uint32_t maxdeg, uint32_t pv_row0, bool per_vertex,
                           int rank, int nranks, unsigned long long* acc, double* ops);
}  // namespace bbf
