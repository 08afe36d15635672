// dense_i8.cu — S10 of the hot path: the dense int8 tensor-core path (tcgen05, sm_100a).
//
// For one side s (rows = the side's vertices in rank order, K = the other side's vertices) let
// A in {0,1} be the adjacency and S in {-1,0,+1} the signed adjacency.  For a same-side pair
// (i, j): T_ij = (A A^T)_ij = #common neighbours and P_ij = (S S^T)_ij = #agreeing - #disagreeing
// common neighbours, so the agree / disagree wedge counts of Def. Symmetric / Asymmetric Wedge
// are a = (T+P)/2, d = (T-P)/2, and Lemma 2 gives the
// pair's balanced count C(a,2) + C(d,2), unbalanced a*d.  Summing over i < j
// counts every butterfly once (Alg. 2's global count); the row + column sums of the upper
// triangle are the per-vertex counts of the side (vBBFC semantics).
//
// Kernel k_dense_tiles: persistent, one CTA per SM, 6 warps:
//   warp 0     TMA producer: per K block of 128 B, A_i, S_i (128 rows) and A_j, S_j (256 rows)
//              into a 2-stage 128B-swizzled shared-memory ring (96 KB per stage);
//   warp 1     TMEM allocator + MMA issuer: tcgen05.mma.cta_group::1.kind::i8, M=128, N=256,
//              K=32 per instruction; T accumulates in TMEM columns [0,256) (u8 x u8), P in
//              [256,512) (s8 x s8), both exact s32;
//   warps 2-5  epilogue: tcgen05.ld 32 columns at a time, Lemma 2 per element, row sums in
//              registers, column sums by a lane-transposing butterfly + shared atomics, u64
//              atomics to the per-vertex array once per tile.
// Tiles (I, J) of 128 x 256 cover the upper triangle only (j > i masked on diagonal tiles).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "bbf_internal.cuh"

namespace bbf {
namespace {

constexpr uint32_t kBM = 128;       // rows i per tile (MMA M, TMEM lanes)
constexpr uint32_t kBN = 256;       // rows j per tile (MMA N)
constexpr uint32_t kBK = 128;       // K bytes per stage (one 128-B swizzle row)
constexpr uint32_t kStages = 2;
constexpr uint32_t kTileI = kBM * kBK;           // 16 KB
constexpr uint32_t kTileJ = kBN * kBK;           // 32 KB
constexpr uint32_t kStageBytes = 2 * kTileI + 2 * kTileJ;  // A_i, S_i, A_j, S_j = 96 KB
constexpr int kThreads = 192;
constexpr int kEpiWarp0 = 2;
constexpr size_t kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 2 * kBN * 8 /*col acc*/ + 256;

// ------------------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// K-major operand tile, 128-B swizzle, rows of 128 B, 8-row atoms 1024 B apart
// (SBO = 1024 B, LBO = 16 B (unused for swizzled K-major), version 1, layout SWIZZLE_128B = 2)
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) | ((uint64_t)64u << 32) |
         ((uint64_t)1u << 46) | ((uint64_t)2u << 61);
}

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// instruction descriptors: D s32 (bits 4-5 = 2), A/B format bits 7-9 / 10-12 (0 u8, 1 s8),
// K-major A and B, N >> 3 at bit 17, M >> 4 at bit 24
constexpr uint32_t kIdescT = (2u << 4) | (0u << 7) | (0u << 10) | ((kBN >> 3) << 17) | ((kBM >> 4) << 24);
constexpr uint32_t kIdescP = (2u << 4) | (1u << 7) | (1u << 10) | ((kBN >> 3) << 17) | ((kBM >> 4) << 24);

struct DenseArgs {
  const uint2* tiles;  // (I, J)
  uint32_t n_tiles;
  uint32_t n_rows;     // rows of this side
  uint32_t n_kb;       // K blocks of 128 B
  uint32_t pv_row0;    // pv index of row 0 (0 for U, n_u for V)
  uint32_t n;          // pv stride (N counts at pv[n + ...])
  int rank, nranks;
  unsigned long long* pv;  // nullptr: global only
  unsigned long long* acc; // [0] B, [1] N
  // hybrid cross terms (k_dense_f4q<true>, hybrid.cu): the pair words R[i * r_ld + j] hold the
  // non-core counts (a_r | d_r << 16); the tile's T, P give the core counts (a_c, d_c) and the
  // epilogue adds a_c a_r + d_c d_r / a_c d_r + a_r d_c, then stores (a_c | d_c << 16) in R
  uint32_t* R;
  uint32_t r_ld;
};

// Column sums of a warp's 32 x 32 block: lane L ends holding the sum over the 32 lanes (rows)
// of column L.  Recursive halving: each step exchanges half of the remaining columns.
template <int H>
__device__ __forceinline__ void xpose_step(unsigned long long (&v)[32], int lane) {
  const bool up = lane & H;
#pragma unroll
  for (int c = 0; c < H; ++c) {
    unsigned long long send = up ? v[c] : v[c + H];
    unsigned long long keep = up ? v[c + H] : v[c];
    v[c] = keep + __shfl_xor_sync(0xffffffffu, send, H);
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    k_dense_tiles(const __grid_constant__ CUtensorMap mA_i, const __grid_constant__ CUtensorMap mS_i,
                  const __grid_constant__ CUtensorMap mA_j, const __grid_constant__ CUtensorMap mS_j,
                  const DenseArgs a) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned operand ring (128-B swizzle atoms)
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned long long* colB = reinterpret_cast<unsigned long long*>(smem + kStages * kStageBytes);
  unsigned long long* colN = colB + kBN;
  __shared__ __align__(8) uint64_t bar_full[kStages], bar_empty[kStages], bar_tfull, bar_tempty;
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (uint32_t i = threadIdx.x; i < 2 * kBN; i += kThreads) colB[i] = 0;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < kStages; ++s) {
      mbar_init(smem_u32(&bar_full[s]), 1);
      mbar_init(smem_u32(&bar_empty[s]), 1);
    }
    mbar_init(smem_u32(&bar_tfull), 1);
    mbar_init(smem_u32(&bar_tempty), 4 * 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&tmem_base_sh))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0) {
    // ================================================================ TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mA_i)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mS_i)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mA_j)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mS_j)) : "memory");
      uint32_t stage = 0, phase = 0;
      for (uint32_t t = blockIdx.x * a.nranks + a.rank; t < a.n_tiles; t += gridDim.x * a.nranks) {
        const uint2 tile = a.tiles[t];
        const int32_t ri = (int32_t)(tile.x * kBM), rj = (int32_t)(tile.y * kBN);
        for (uint32_t kb = 0; kb < a.n_kb; ++kb) {
          mbar_wait(smem_u32(&bar_empty[stage]), phase ^ 1u);
          const uint32_t fb = smem_u32(&bar_full[stage]);
          mbar_arrive_expect_tx(fb, kStageBytes);
          const uint32_t base = smem_u32(smem + stage * kStageBytes);
          const int32_t k0 = (int32_t)(kb * kBK);
          tma_load_2d(base, &mA_i, fb, k0, ri);
          tma_load_2d(base + kTileI, &mS_i, fb, k0, ri);
          tma_load_2d(base + 2 * kTileI, &mA_j, fb, k0, rj);
          tma_load_2d(base + 2 * kTileI + kTileJ, &mS_j, fb, k0, rj);
          if (++stage == kStages) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    // ================================================================ MMA issuer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, lt = 0;
      for (uint32_t t = blockIdx.x * a.nranks + a.rank; t < a.n_tiles; t += gridDim.x * a.nranks, ++lt) {
        if (lt > 0) {
          mbar_wait(smem_u32(&bar_tempty), (lt - 1) & 1u);
          tc_fence_after();
        }
        for (uint32_t kb = 0; kb < a.n_kb; ++kb) {
          mbar_wait(smem_u32(&bar_full[stage]), phase);
          tc_fence_after();
          const uint32_t base = smem_u32(smem + stage * kStageBytes);
#pragma unroll
          for (uint32_t kk = 0; kk < kBK / 32; ++kk) {
            const uint32_t acc = (kb | kk) ? 1u : 0u;
            const uint32_t off = kk * 32;
            mma_i8(tmem, smem_desc(base + off), smem_desc(base + 2 * kTileI + off), kIdescT, acc);
            mma_i8(tmem + kBN, smem_desc(base + kTileI + off),
                   smem_desc(base + 2 * kTileI + kTileJ + off), kIdescP, acc);
          }
          mma_commit(smem_u32(&bar_empty[stage]));  // frees the stage when these MMAs finish
          if (++stage == kStages) { stage = 0; phase ^= 1u; }
        }
        mma_commit(smem_u32(&bar_tfull));
      }
    }
  } else {
    // ================================================================ epilogue (warps 2..5)
    const uint32_t q = (uint32_t)(warp & 3);  // TMEM lane quarter this warp may access
    const uint32_t etid = threadIdx.x - kEpiWarp0 * 32;  // 0..127
    unsigned long long totB = 0, totN = 0;
    uint32_t lt = 0;
    for (uint32_t t = blockIdx.x * a.nranks + a.rank; t < a.n_tiles; t += gridDim.x * a.nranks, ++lt) {
      const uint2 tile = a.tiles[t];
      const uint32_t i = tile.x * kBM + q * 32 + lane;  // this thread's row
      const uint32_t j0 = tile.y * kBN;
      const bool diag = j0 < tile.x * kBM + kBM;        // some j <= i in the tile
      mbar_wait(smem_u32(&bar_tfull), lt & 1u);
      tc_fence_after();
      unsigned long long rB = 0, rN = 0;
#pragma unroll 1
      for (uint32_t c = 0; c < kBN / 32; ++c) {
        uint32_t tv[32], pv[32];
        const uint32_t ta = tmem + ((q * 32) << 16) + c * 32;
        tmem_ld32(ta, tv);
        tmem_ld32(ta + kBN, pv);
        tmem_wait_ld();
        unsigned long long vb[32], vn[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const uint32_t tt = tv[e], pp = pv[e];
          const uint32_t ad = (tt + pp) >> 1, dd = (tt - pp) >> 1;  // a, d (t >= |p|)
          uint32_t fb = ((ad * (ad - 1u)) >> 1) + ((dd * (dd - 1u)) >> 1);
          uint32_t fn = ad * dd;
          if (diag && j0 + c * 32 + (uint32_t)e <= i) { fb = 0; fn = 0; }
          rB += fb;
          rN += fn;
          vb[e] = fb;
          vn[e] = fn;
        }
        if (a.pv) {
          xpose_step<16>(vb, lane); xpose_step<16>(vn, lane);
          xpose_step<8>(vb, lane);  xpose_step<8>(vn, lane);
          xpose_step<4>(vb, lane);  xpose_step<4>(vn, lane);
          xpose_step<2>(vb, lane);  xpose_step<2>(vn, lane);
          xpose_step<1>(vb, lane);  xpose_step<1>(vn, lane);
          if (vb[0]) atomicAdd(&colB[c * 32 + lane], vb[0]);
          if (vn[0]) atomicAdd(&colN[c * 32 + lane], vn[0]);
        }
      }
      // TMEM may be overwritten by the next tile's MMAs from here on
      tc_fence_before();
      mbar_arrive(smem_u32(&bar_tempty));
      totB += rB;
      totN += rN;
      if (a.pv) {
        if ((rB | rN) && i < a.n_rows) {
          atomicAdd(&a.pv[2ull * (a.pv_row0 + i)], rB);
          atomicAdd(&a.pv[2ull * (a.pv_row0 + i) + 1], rN);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        for (uint32_t jj = etid; jj < kBN; jj += 128) {
          const unsigned long long b = colB[jj], nn = colN[jj];
          colB[jj] = 0;
          colN[jj] = 0;
          const uint32_t j = j0 + jj;
          if ((b | nn) && j < a.n_rows) {
            atomicAdd(&a.pv[2ull * (a.pv_row0 + j)], b);
            atomicAdd(&a.pv[2ull * (a.pv_row0 + j) + 1], nn);
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
    }
    for (int o = 16; o; o >>= 1) {
      totB += __shfl_xor_sync(0xffffffffu, totB, o);
      totN += __shfl_xor_sync(0xffffffffu, totN, o);
    }
    if (lane == 0 && (totB | totN)) {
      atomicAdd(&a.acc[0], totB);
      atomicAdd(&a.acc[1], totN);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// ============================================================================ CTA-pair kernel
// k_dense_pair: the same computation on 256 x 256 tiles with tcgen05.mma.cta_group::2 (M = 256,
// N = 256) by a cluster of 2 CTAs on one TPC.  CTA r of the pair loads rows [128r, 128r + 128)
// of the i-block (A_i, S_i: the MMA's A operand halves) and of the j-block (A_j, S_j: the B
// operand halves) into its own 3-stage ring (64 KB per stage), both completing on the leader's
// full barrier; the leader issues the MMAs, which read both CTAs' shared memory and accumulate
// rows [128r, 128r + 128) of T and P in CTA r's TMEM.  Each CTA's epilogue handles its 128 rows
// exactly as in k_dense_tiles.  Operand traffic per MAC is 2/3 of the single-CTA kernel's.
constexpr uint32_t kPB = 256;                     // pair tile (rows i and rows j)
constexpr uint32_t kPStages = 3;
constexpr uint32_t kPHalf = 128 * kBK;            // 16 KB: one operand half (128 rows x 128 B)
constexpr uint32_t kPStageBytes = 4 * kPHalf;     // A_i, S_i, A_j, S_j halves = 64 KB
constexpr size_t kPSmemBytes = kPStages * kPStageBytes + 1024 + 2 * kBN * 8 + 256;
constexpr uint32_t kIdescT2 = (2u << 4) | (0u << 7) | (0u << 10) | ((kPB >> 3) << 17) | ((kPB >> 4) << 24);
constexpr uint32_t kIdescP2 = (2u << 4) | (1u << 7) | (1u << 10) | ((kPB >> 3) << 17) | ((kPB >> 4) << 24);

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA into this CTA's shared memory, completing on the leader's barrier (cluster address)
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar_cluster,
                                                 int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.cta_group::2"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mma_i8_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// commit: arrive on the barrier at this offset in both CTAs of the pair when the MMAs finish
__device__ __forceinline__ void mma_commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_dense_pair(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mS,
                 const DenseArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned long long* colB = reinterpret_cast<unsigned long long*>(smem + kPStages * kPStageBytes);
  unsigned long long* colN = colB + kBN;
  __shared__ __align__(8) uint64_t bar_full[kPStages], bar_empty[kPStages], bar_tfull, bar_tempty;
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_rank();
  const bool leader = crank == 0;
  const uint32_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  for (uint32_t i = threadIdx.x; i < 2 * kBN; i += kThreads) colB[i] = 0;
  if (threadIdx.x == 0) {
    for (uint32_t st = 0; st < kPStages; ++st) {
      mbar_init(smem_u32(&bar_full[st]), 1);
      mbar_init(smem_u32(&bar_empty[st]), 1);
    }
    mbar_init(smem_u32(&bar_tfull), 1);
    mbar_init(smem_u32(&bar_tempty), 2 * 4);  // one arrival per epilogue warp of both CTAs
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&tmem_base_sh))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0) {
    // ================================================================ TMA producer (both CTAs)
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mS)) : "memory");
      uint32_t stage = 0, phase = 0;
      for (uint32_t t = pair * a.nranks + a.rank; t < a.n_tiles; t += npairs * a.nranks) {
        const uint2 tile = a.tiles[t];
        const int32_t ri = (int32_t)(tile.x * kPB + crank * 128), rj = (int32_t)(tile.y * kPB + crank * 128);
        for (uint32_t kb = 0; kb < a.n_kb; ++kb) {
          mbar_wait(smem_u32(&bar_empty[stage]), phase ^ 1u);
          const uint32_t fb = mapa_rank(smem_u32(&bar_full[stage]), 0);
          if (leader) mbar_arrive_expect_tx(smem_u32(&bar_full[stage]), 2 * kPStageBytes);
          const uint32_t base = smem_u32(smem + stage * kPStageBytes);
          const int32_t k0 = (int32_t)(kb * kBK);
          tma_load_2d_pair(base, &mA, fb, k0, ri);
          tma_load_2d_pair(base + kPHalf, &mS, fb, k0, ri);
          tma_load_2d_pair(base + 2 * kPHalf, &mA, fb, k0, rj);
          tma_load_2d_pair(base + 3 * kPHalf, &mS, fb, k0, rj);
          if (++stage == kPStages) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    // ================================================================ MMA issuer (leader only)
    if (leader && lane == 0) {
      uint32_t stage = 0, phase = 0, lt = 0;
      for (uint32_t t = pair * a.nranks + a.rank; t < a.n_tiles; t += npairs * a.nranks, ++lt) {
        if (lt > 0) {
          mbar_wait(smem_u32(&bar_tempty), (lt - 1) & 1u);
          tc_fence_after();
        }
        for (uint32_t kb = 0; kb < a.n_kb; ++kb) {
          mbar_wait(smem_u32(&bar_full[stage]), phase);
          tc_fence_after();
          const uint32_t base = smem_u32(smem + stage * kPStageBytes);
#pragma unroll
          for (uint32_t kk = 0; kk < kBK / 32; ++kk) {
            const uint32_t acc = (kb | kk) ? 1u : 0u;
            const uint32_t off = kk * 32;
            mma_i8_pair(tmem, smem_desc(base + off), smem_desc(base + 2 * kPHalf + off), kIdescT2, acc);
            mma_i8_pair(tmem + kBN, smem_desc(base + kPHalf + off), smem_desc(base + 3 * kPHalf + off),
                        kIdescP2, acc);
          }
          mma_commit_pair(smem_u32(&bar_empty[stage]));  // frees the stage in both CTAs
          if (++stage == kPStages) { stage = 0; phase ^= 1u; }
        }
        mma_commit_pair(smem_u32(&bar_tfull));
      }
    }
  } else {
    // ================================================================ epilogue (warps 2..5)
    const uint32_t q = (uint32_t)(warp & 3);
    const uint32_t etid = threadIdx.x - kEpiWarp0 * 32;
    const uint32_t tempty_leader = mapa_rank(smem_u32(&bar_tempty), 0);
    unsigned long long totB = 0, totN = 0;
    uint32_t lt = 0;
    for (uint32_t t = pair * a.nranks + a.rank; t < a.n_tiles; t += npairs * a.nranks, ++lt) {
      const uint2 tile = a.tiles[t];
      const uint32_t i = tile.x * kPB + crank * 128 + q * 32 + lane;  // this thread's row
      const uint32_t j0 = tile.y * kPB;
      const bool diag = tile.x == tile.y;
      mbar_wait(smem_u32(&bar_tfull), lt & 1u);
      tc_fence_after();
      unsigned long long rB = 0, rN = 0;
#pragma unroll 1
      for (uint32_t c = 0; c < kBN / 32; ++c) {
        uint32_t tv[32], pv[32];
        const uint32_t ta = tmem + ((q * 32) << 16) + c * 32;
        tmem_ld32(ta, tv);
        tmem_ld32(ta + kBN, pv);
        tmem_wait_ld();
        unsigned long long vb[32], vn[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const uint32_t tt = tv[e], pp = pv[e];
          const uint32_t ad = (tt + pp) >> 1, dd = (tt - pp) >> 1;
          uint32_t fb = ((ad * (ad - 1u)) >> 1) + ((dd * (dd - 1u)) >> 1);
          uint32_t fn = ad * dd;
          if (diag && j0 + c * 32 + (uint32_t)e <= i) { fb = 0; fn = 0; }
          rB += fb;
          rN += fn;
          vb[e] = fb;
          vn[e] = fn;
        }
        if (a.pv) {
          xpose_step<16>(vb, lane); xpose_step<16>(vn, lane);
          xpose_step<8>(vb, lane);  xpose_step<8>(vn, lane);
          xpose_step<4>(vb, lane);  xpose_step<4>(vn, lane);
          xpose_step<2>(vb, lane);  xpose_step<2>(vn, lane);
          xpose_step<1>(vb, lane);  xpose_step<1>(vn, lane);
          if (vb[0]) atomicAdd(&colB[c * 32 + lane], vb[0]);
          if (vn[0]) atomicAdd(&colN[c * 32 + lane], vn[0]);
        }
      }
      // this warp is done with TMEM: one arrival on the leader's tmem_empty barrier
      tc_fence_before();
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(tempty_leader)
                     : "memory");
      totB += rB;
      totN += rN;
      if (a.pv) {
        if ((rB | rN) && i < a.n_rows) {
          atomicAdd(&a.pv[2ull * (a.pv_row0 + i)], rB);
          atomicAdd(&a.pv[2ull * (a.pv_row0 + i) + 1], rN);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        for (uint32_t jj = etid; jj < kBN; jj += 128) {
          const unsigned long long b = colB[jj], nn = colN[jj];
          colB[jj] = 0;
          colN[jj] = 0;
          const uint32_t j = j0 + jj;
          if ((b | nn) && j < a.n_rows) {
            atomicAdd(&a.pv[2ull * (a.pv_row0 + j)], b);
            atomicAdd(&a.pv[2ull * (a.pv_row0 + j) + 1], nn);
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
    }
    for (int o = 16; o; o >>= 1) {
      totB += __shfl_xor_sync(0xffffffffu, totB, o);
      totN += __shfl_xor_sync(0xffffffffu, totN, o);
    }
    if (lane == 0 && (totB | totN)) {
      atomicAdd(&a.acc[0], totB);
      atomicAdd(&a.acc[1], totN);
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// 8 x 8 nibble transpose in registers: w[k] = row k (nibble j = column j) becomes w[j] = column j
// (nibble k = row k), by swapping 2 x 2 blocks of nibbles, then bytes, then half-words
__device__ __forceinline__ void transpose8x8_nibbles(uint32_t (&w)[8]) {
#pragma unroll
  for (int k = 0; k < 8; k += 2) {
    const uint32_t t = ((w[k] >> 4) ^ w[k + 1]) & 0x0F0F0F0Fu;
    w[k + 1] ^= t;
    w[k] ^= t << 4;
  }
#pragma unroll
  for (int k = 0; k < 8; k += (k & 1) ? 3 : 1) {  // k = 0, 1, 4, 5
    const uint32_t t = ((w[k] >> 8) ^ w[k + 2]) & 0x00FF00FFu;
    w[k + 2] ^= t;
    w[k] ^= t << 8;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t t = ((w[k] >> 16) ^ w[k + 4]) & 0x0000FFFFu;
    w[k + 4] ^= t;
    w[k] ^= t << 16;
  }
}

// Av4 = Au4^T and Sv4 = Su4^T on the packed e2m1 operands, 128 x 128 element tiles: each thread
// loads an 8 x 8 nibble block (eight 4-byte row pieces), transposes it in registers and stages the
// words in shared memory (lanes spread so the staging stores hit 32 distinct banks); the tile is
// written as 64-byte row pieces.  U rows at or beyond rows_u read as zero.  Lets an FP4-only
// graph skip the u8 operands altogether.
__global__ void __launch_bounds__(256) k_dense_transpose_f4(const uint8_t* __restrict__ Au4,
                                                            const uint8_t* __restrict__ Su4, uint32_t ku4,
                                                            uint32_t rows_u, uint8_t* __restrict__ Av4,
                                                            uint8_t* __restrict__ Sv4, uint32_t kv4) {
  __shared__ uint32_t ta[128][17], ts[128][17];
  const uint32_t c0 = blockIdx.x * 128, r0 = blockIdx.y * 128;  // U rows c0.. (V columns), V rows r0..
  const uint32_t wp = threadIdx.x >> 5, l = threadIdx.x & 31;
  const uint32_t bi = 8 * (wp & 1) + (l & 7), bj = 4 * (wp >> 1) + (l >> 3);  // U rows c0 + 8 bi, V rows r0 + 8 bj
  uint32_t a[8], s[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t row = c0 + 8 * bi + k;
    const uint64_t src = (uint64_t)row * ku4 + r0 / 2 + 4 * bj;
    const bool in = row < rows_u && r0 / 2 + 4 * bj < ku4;
    a[k] = in ? __ldg(reinterpret_cast<const uint32_t*>(Au4 + src)) : 0u;
    s[k] = in ? __ldg(reinterpret_cast<const uint32_t*>(Su4 + src)) : 0u;
  }
  transpose8x8_nibbles(a);
  transpose8x8_nibbles(s);
#pragma unroll
  for (int k = 0; k < 8; ++k) { ta[8 * bj + k][bi] = a[k]; ts[8 * bj + k][bi] = s[k]; }
  __syncthreads();
  const uint32_t orow = threadIdx.x >> 1, h = 8 * (threadIdx.x & 1);  // V row r0 + orow, words h .. h + 7
  const uint64_t dst = (uint64_t)(r0 + orow) * kv4 + c0 / 2 + 4 * h;
  uint4* da = reinterpret_cast<uint4*>(Av4 + dst);
  uint4* ds = reinterpret_cast<uint4*>(Sv4 + dst);
  da[0] = make_uint4(ta[orow][h], ta[orow][h + 1], ta[orow][h + 2], ta[orow][h + 3]);
  da[1] = make_uint4(ta[orow][h + 4], ta[orow][h + 5], ta[orow][h + 6], ta[orow][h + 7]);
  ds[0] = make_uint4(ts[orow][h], ts[orow][h + 1], ts[orow][h + 2], ts[orow][h + 3]);
  ds[1] = make_uint4(ts[orow][h + 4], ts[orow][h + 5], ts[orow][h + 6], ts[orow][h + 7]);
}

// ================================================================================ FP4 variant
// The same pair kernel on the block-scaled FP4 tensor path (tcgen05.mma.cta_group::2.kind::mxf4,
// 2x the int8 rate, half the operand bytes): A and S as e2m1 (0, +1.0, -1.0) packed two per byte,
// every E8M0 block scale 1.0 (127), so T = A A^T and P = S S^T are integer sums of +-1 products,
// accumulated in fp32 — exact while every partial sum stays far below 2^24; the path is used only
// when the rows' maximum degree (which bounds |T|, |P| and every partial sum) is <= 8,192.
// TMEM: T in columns [0, 224), P in [224, 448) (N = 224: both accumulators and the scale factors
// must fit the 512 columns), scale factors in [448, 512), filled once with 0x7F bytes.
constexpr uint32_t kF4N = 224;                    // tile columns (MMA N); each CTA holds 112 B rows
constexpr uint32_t kF4JRows = kF4N / 2;
constexpr uint32_t kF4Stages = 3;
constexpr uint32_t kF4StageBytes = 4 * kPHalf;    // A_i, S_i (128 rows), A_j, S_j (112 rows) slots
constexpr size_t kF4SmemBytes = kF4Stages * kF4StageBytes + 1024 + 2 * kBN * 8 + 256;
constexpr uint32_t kF4SfCol = 2 * kF4N;           // 448
// block-scaled descriptor: a/b format E2M1 (MXF4Format 1) at bits 7 / 10, N >> 3 at 17, scale
// format E8M0 at bit 23, M >> 4 at 24, K = 64 (bit 31 clear), scale-factor ids 0
constexpr uint32_t kIdescF4 = (1u << 7) | (1u << 10) | ((kF4N >> 3) << 17) | (1u << 23) | ((256u >> 4) << 24);

__device__ __forceinline__ void mma_f4_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t sf,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(kIdescF4), "r"(acc), "r"(sf)
      : "memory");
}

__device__ __forceinline__ void tmem_st16_const(uint32_t taddr, uint32_t v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
      "r"(v)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_dense_f4(const __grid_constant__ CUtensorMap mAi, const __grid_constant__ CUtensorMap mSi,
               const __grid_constant__ CUtensorMap mAj, const __grid_constant__ CUtensorMap mSj,
               const DenseArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned long long* colB = reinterpret_cast<unsigned long long*>(smem + kF4Stages * kF4StageBytes);
  unsigned long long* colN = colB + kBN;
  __shared__ __align__(8) uint64_t bar_full[kF4Stages], bar_empty[kF4Stages], bar_tfull, bar_tempty;
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_rank();
  const bool leader = crank == 0;
  const uint32_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  for (uint32_t i = threadIdx.x; i < 2 * kBN; i += kThreads) colB[i] = 0;
  if (threadIdx.x == 0) {
    for (uint32_t st = 0; st < kF4Stages; ++st) {
      mbar_init(smem_u32(&bar_full[st]), 1);
      mbar_init(smem_u32(&bar_empty[st]), 1);
    }
    mbar_init(smem_u32(&bar_tfull), 1);
    mbar_init(smem_u32(&bar_tempty), 2 * 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&tmem_base_sh))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  if (warp >= kEpiWarp0) {  // scale factors: every byte of columns [448, 512) = 127 (2^0)
    const uint32_t q = (uint32_t)(warp & 3);
#pragma unroll
    for (uint32_t h = 0; h < 4; ++h) tmem_st16_const(tmem + ((q * 32) << 16) + kF4SfCol + 16 * h, 0x7F7F7F7Fu);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mAi)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mSi)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mAj)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mSj)) : "memory");
      uint32_t stage = 0, phase = 0;
      for (uint32_t t = pair * a.nranks + a.rank; t < a.n_tiles; t += npairs * a.nranks) {
        const uint2 tile = a.tiles[t];
        const int32_t ri = (int32_t)(tile.x * kPB + crank * 128);
        const int32_t rj = (int32_t)(tile.y * kF4N + crank * kF4JRows);
        for (uint32_t kb = 0; kb < a.n_kb; ++kb) {
          mbar_wait(smem_u32(&bar_empty[stage]), phase ^ 1u);
          const uint32_t fb = mapa_rank(smem_u32(&bar_full[stage]), 0);
          if (leader) mbar_arrive_expect_tx(smem_u32(&bar_full[stage]), 2 * (2 * kPHalf + 2 * kF4JRows * kBK));
          const uint32_t base = smem_u32(smem + stage * kF4StageBytes);
          const int32_t k0 = (int32_t)(kb * kBK);
          tma_load_2d_pair(base, &mAi, fb, k0, ri);
          tma_load_2d_pair(base + kPHalf, &mSi, fb, k0, ri);
          tma_load_2d_pair(base + 2 * kPHalf, &mAj, fb, k0, rj);
          tma_load_2d_pair(base + 3 * kPHalf, &mSj, fb, k0, rj);
          if (++stage == kF4Stages) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      uint32_t stage = 0, phase = 0, lt = 0;
      for (uint32_t t = pair * a.nranks + a.rank; t < a.n_tiles; t += npairs * a.nranks, ++lt) {
        if (lt > 0) {
          mbar_wait(smem_u32(&bar_tempty), (lt - 1) & 1u);
          tc_fence_after();
        }
        for (uint32_t kb = 0; kb < a.n_kb; ++kb) {
          mbar_wait(smem_u32(&bar_full[stage]), phase);
          tc_fence_after();
          const uint32_t base = smem_u32(smem + stage * kF4StageBytes);
#pragma unroll
          for (uint32_t kk = 0; kk < kBK / 32; ++kk) {  // 32 B = 64 e2m1 values per MMA
            const uint32_t acc = (kb | kk) ? 1u : 0u;
            const uint32_t off = kk * 32;
            mma_f4_pair(tmem, smem_desc(base + off), smem_desc(base + 2 * kPHalf + off), tmem + kF4SfCol, acc);
            mma_f4_pair(tmem + kF4N, smem_desc(base + kPHalf + off), smem_desc(base + 3 * kPHalf + off),
                        tmem + kF4SfCol, acc);
          }
          mma_commit_pair(smem_u32(&bar_empty[stage]));
          if (++stage == kF4Stages) { stage = 0; phase ^= 1u; }
        }
        mma_commit_pair(smem_u32(&bar_tfull));
      }
    }
  } else {
    const uint32_t q = (uint32_t)(warp & 3);
    const uint32_t etid = threadIdx.x - kEpiWarp0 * 32;
    const uint32_t tempty_leader = mapa_rank(smem_u32(&bar_tempty), 0);
    unsigned long long totB = 0, totN = 0;
    uint32_t lt = 0;
    for (uint32_t t = pair * a.nranks + a.rank; t < a.n_tiles; t += npairs * a.nranks, ++lt) {
      const uint2 tile = a.tiles[t];
      const uint32_t i = tile.x * kPB + crank * 128 + q * 32 + lane;  // this thread's row
      const uint32_t j0 = tile.y * kF4N;
      mbar_wait(smem_u32(&bar_tfull), lt & 1u);
      tc_fence_after();
      unsigned long long rB = 0, rN = 0;
#pragma unroll 1
      for (uint32_t c = 0; c < kF4N / 32; ++c) {
        uint32_t tv[32], pv[32];
        const uint32_t ta = tmem + ((q * 32) << 16) + c * 32;
        tmem_ld32(ta, tv);
        tmem_ld32(ta + kF4N, pv);
        tmem_wait_ld();
        unsigned long long vb[32], vn[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const uint32_t tt = (uint32_t)__float2int_rn(__int_as_float((int)tv[e]));
          const uint32_t pp = (uint32_t)__float2int_rn(__int_as_float((int)pv[e]));
          const uint32_t ad = (tt + pp) >> 1, dd = (tt - pp) >> 1;
          uint32_t fb = ((ad * (ad - 1u)) >> 1) + ((dd * (dd - 1u)) >> 1);
          uint32_t fn = ad * dd;
          if (j0 + c * 32 + (uint32_t)e <= i) { fb = 0; fn = 0; }  // pairs i < j only
          rB += fb;
          rN += fn;
          vb[e] = fb;
          vn[e] = fn;
        }
        if (a.pv) {
          xpose_step<16>(vb, lane); xpose_step<16>(vn, lane);
          xpose_step<8>(vb, lane);  xpose_step<8>(vn, lane);
          xpose_step<4>(vb, lane);  xpose_step<4>(vn, lane);
          xpose_step<2>(vb, lane);  xpose_step<2>(vn, lane);
          xpose_step<1>(vb, lane);  xpose_step<1>(vn, lane);
          if (vb[0]) atomicAdd(&colB[c * 32 + lane], vb[0]);
          if (vn[0]) atomicAdd(&colN[c * 32 + lane], vn[0]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(tempty_leader)
                     : "memory");
      totB += rB;
      totN += rN;
      if (a.pv) {
        if ((rB | rN) && i < a.n_rows) {
          atomicAdd(&a.pv[2ull * (a.pv_row0 + i)], rB);
          atomicAdd(&a.pv[2ull * (a.pv_row0 + i) + 1], rN);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        for (uint32_t jj = etid; jj < kF4N; jj += 128) {
          const unsigned long long b = colB[jj], nn = colN[jj];
          colB[jj] = 0;
          colN[jj] = 0;
          const uint32_t j = j0 + jj;
          if ((b | nn) && j < a.n_rows) {
            atomicAdd(&a.pv[2ull * (a.pv_row0 + j)], b);
            atomicAdd(&a.pv[2ull * (a.pv_row0 + j) + 1], nn);
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
    }
    for (int o = 16; o; o >>= 1) {
      totB += __shfl_xor_sync(0xffffffffu, totB, o);
      totN += __shfl_xor_sync(0xffffffffu, totN, o);
    }
    if (lane == 0 && (totB | totN)) {
      atomicAdd(&a.acc[0], totB);
      atomicAdd(&a.acc[1], totN);
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// ====================================================== FP4, one packed accumulator (k_dense_f4q)
// When the rows' max degree is < 2048, T and P are produced by ONE accumulation over a K axis of
// twice the length: the first half multiplies A_i by A_j with unit block scales, the second S_i by
// S_j with block scales 2^5 (A operand) and 2^6 (B operand), so the accumulator holds
// Q = T + 2048 P exactly (|Q| < 2^22, integer fp32 sums), decoded as P = floor(Q / 2048),
// T = Q - 2048 P (T in [0, 2047]).  One 224-column accumulator per tile leaves room for TWO in
// TMEM: tile t+1 accumulates into the other buffer while the epilogue drains tile t.
constexpr uint32_t kQStages = 6;
constexpr uint32_t kQStageBytes = 2 * kPHalf;     // i operand (128 rows), j operand (112-row slot)
constexpr size_t kQSmemBytes = kQStages * kQStageBytes + 1024 + 2 * kBN * 8 + 256;
constexpr uint32_t kQSf1 = 2 * kF4N, kQSfA = kQSf1 + 16, kQSfB = kQSf1 + 32;  // scale regions

__device__ __forceinline__ void mma_f4q(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t sfa, uint32_t sfb,
                                        uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(kIdescF4), "r"(acc), "r"(sfa), "r"(sfb)
      : "memory");
}

template <bool CROSS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_dense_f4q(const __grid_constant__ CUtensorMap mAi, const __grid_constant__ CUtensorMap mSi,
                const __grid_constant__ CUtensorMap mAj, const __grid_constant__ CUtensorMap mSj,
                const DenseArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned long long* colB = reinterpret_cast<unsigned long long*>(smem + kQStages * kQStageBytes);
  unsigned long long* colN = colB + kBN;
  __shared__ __align__(8) uint64_t bar_full[kQStages], bar_empty[kQStages], bar_tfull[2], bar_tempty[2];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_rank();
  const bool leader = crank == 0;
  const uint32_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const uint32_t nk = 2 * a.n_kb;  // K steps: A half, then S half

  for (uint32_t i = threadIdx.x; i < 2 * kBN; i += kThreads) colB[i] = 0;
  if (threadIdx.x == 0) {
    for (uint32_t st = 0; st < kQStages; ++st) {
      mbar_init(smem_u32(&bar_full[st]), 1);
      mbar_init(smem_u32(&bar_empty[st]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&bar_tfull[b]), 1);
      mbar_init(smem_u32(&bar_tempty[b]), 2 * 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&tmem_base_sh))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  if (warp >= kEpiWarp0) {  // scale regions: 2^0 everywhere, 2^5 (0x84) and 2^6 (0x85)
    const uint32_t lb = tmem + (((uint32_t)(warp & 3) * 32) << 16);
    tmem_st16_const(lb + kQSf1, 0x7F7F7F7Fu);
    tmem_st16_const(lb + kQSfA, 0x84848484u);
    tmem_st16_const(lb + kQSfB, 0x85858585u);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mAi)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mSi)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mAj)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mSj)) : "memory");
      uint32_t stage = 0, phase = 0;
      for (uint32_t t = pair * a.nranks + a.rank; t < a.n_tiles; t += npairs * a.nranks) {
        const uint2 tile = a.tiles[t];
        const int32_t ri = (int32_t)(tile.x * kPB + crank * 128);
        const int32_t rj = (int32_t)(tile.y * kF4N + crank * kF4JRows);
        for (uint32_t kb = 0; kb < nk; ++kb) {
          mbar_wait(smem_u32(&bar_empty[stage]), phase ^ 1u);
          const uint32_t fb = mapa_rank(smem_u32(&bar_full[stage]), 0);
          if (leader) mbar_arrive_expect_tx(smem_u32(&bar_full[stage]), 2 * (kPHalf + kF4JRows * kBK));
          const uint32_t base = smem_u32(smem + stage * kQStageBytes);
          const bool shalf = kb >= a.n_kb;
          const int32_t k0 = (int32_t)((shalf ? kb - a.n_kb : kb) * kBK);
          tma_load_2d_pair(base, shalf ? &mSi : &mAi, fb, k0, ri);
          tma_load_2d_pair(base + kPHalf, shalf ? &mSj : &mAj, fb, k0, rj);
          if (++stage == kQStages) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      uint32_t stage = 0, phase = 0, lt = 0;
      for (uint32_t t = pair * a.nranks + a.rank; t < a.n_tiles; t += npairs * a.nranks, ++lt) {
        const uint32_t b = lt & 1u;
        if (lt >= 2) {
          mbar_wait(smem_u32(&bar_tempty[b]), ((lt >> 1) - 1) & 1u);
          tc_fence_after();
        }
        const uint32_t dq = tmem + b * kF4N;
        for (uint32_t kb = 0; kb < nk; ++kb) {
          mbar_wait(smem_u32(&bar_full[stage]), phase);
          tc_fence_after();
          const uint32_t base = smem_u32(smem + stage * kQStageBytes);
          const bool shalf = kb >= a.n_kb;
          const uint32_t sfa = tmem + (shalf ? kQSfA : kQSf1), sfb = tmem + (shalf ? kQSfB : kQSf1);
#pragma unroll
          for (uint32_t kk = 0; kk < kBK / 32; ++kk) {  // 32 B = 64 e2m1 values per MMA
            const uint32_t off = kk * 32;
            mma_f4q(dq, smem_desc(base + off), smem_desc(base + kPHalf + off), sfa, sfb, (kb | kk) ? 1u : 0u);
          }
          mma_commit_pair(smem_u32(&bar_empty[stage]));
          if (++stage == kQStages) { stage = 0; phase ^= 1u; }
        }
        mma_commit_pair(smem_u32(&bar_tfull[b]));
      }
    }
  } else {
    const uint32_t q = (uint32_t)(warp & 3);
    const uint32_t etid = threadIdx.x - kEpiWarp0 * 32;
    unsigned long long totB = 0, totN = 0;
    uint32_t lt = 0;
    for (uint32_t t = pair * a.nranks + a.rank; t < a.n_tiles; t += npairs * a.nranks, ++lt) {
      const uint32_t b = lt & 1u;
      const uint2 tile = a.tiles[t];
      const uint32_t i = tile.x * kPB + crank * 128 + q * 32 + lane;  // this thread's row
      const uint32_t j0 = tile.y * kF4N;
      mbar_wait(smem_u32(&bar_tfull[b]), (lt >> 1) & 1u);
      tc_fence_after();
      unsigned long long rB = 0, rN = 0;
#pragma unroll 1
      for (uint32_t c = 0; c < kF4N / 32; ++c) {
        uint32_t qv[32];
        tmem_ld32(tmem + ((q * 32) << 16) + b * kF4N + c * 32, qv);
        uint32_t rw[32];
        uint32_t* rrow = nullptr;
        if (CROSS) {  // this row's 32 pair words (one 128-B line), zero outside the core
          const uint32_t jc = j0 + c * 32;
          rrow = a.R + (uint64_t)i * a.r_ld + jc;
          const bool full = i < a.n_rows && jc + 32 <= a.n_rows && !(reinterpret_cast<uintptr_t>(rrow) & 15);
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            uint4 v4 = make_uint4(0, 0, 0, 0);
            if (full) v4 = *reinterpret_cast<const uint4*>(rrow + e);
            else if (i < a.n_rows)
              for (int f = 0; f < 4; ++f)
                if (jc + e + f < a.n_rows) (&v4.x)[f] = rrow[e + f];
            rw[e] = v4.x; rw[e + 1] = v4.y; rw[e + 2] = v4.z; rw[e + 3] = v4.w;
          }
        }
        tmem_wait_ld();
        unsigned long long vb[32], vn[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int32_t qq = __float2int_rn(__int_as_float((int)qv[e]));
          const int32_t pp = qq >> 11;                          // floor(Q / 2048)
          const uint32_t tt = (uint32_t)(qq - (pp << 11));      // in [0, 2047]
          const uint32_t ad = (tt + (uint32_t)pp) >> 1, dd = (tt - (uint32_t)pp) >> 1;
          uint32_t fb, fn;
          if (CROSS) {  // a_c = ad, d_c = dd over the start's eligible core middles
            const uint32_t ar = rw[e] & 0xffffu, dr = rw[e] >> 16;
            fb = ad * ar + dd * dr;
            fn = ad * dr + ar * dd;
            if (rw[e] && j0 + c * 32 + (uint32_t)e > i) rrow[e] = ad | (dd << 16);
            if (!rw[e]) { fb = 0; fn = 0; }
          } else {
            fb = ((ad * (ad - 1u)) >> 1) + ((dd * (dd - 1u)) >> 1);
            fn = ad * dd;
          }
          if (j0 + c * 32 + (uint32_t)e <= i) { fb = 0; fn = 0; }  // pairs i < j only
          rB += fb;
          rN += fn;
          vb[e] = fb;
          vn[e] = fn;
        }
        if (a.pv) {
          xpose_step<16>(vb, lane); xpose_step<16>(vn, lane);
          xpose_step<8>(vb, lane);  xpose_step<8>(vn, lane);
          xpose_step<4>(vb, lane);  xpose_step<4>(vn, lane);
          xpose_step<2>(vb, lane);  xpose_step<2>(vn, lane);
          xpose_step<1>(vb, lane);  xpose_step<1>(vn, lane);
          if (vb[0]) atomicAdd(&colB[c * 32 + lane], vb[0]);
          if (vn[0]) atomicAdd(&colN[c * 32 + lane], vn[0]);
        }
      }
      // buffer b drained: one arrival per warp on the leader's tmem_empty[b]
      tc_fence_before();
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                         mapa_rank(smem_u32(&bar_tempty[b]), 0))
                     : "memory");
      totB += rB;
      totN += rN;
      if (a.pv) {
        if ((rB | rN) && i < a.n_rows) {
          atomicAdd(&a.pv[2ull * (a.pv_row0 + i)], rB);
          atomicAdd(&a.pv[2ull * (a.pv_row0 + i) + 1], rN);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        for (uint32_t jj = etid; jj < kF4N; jj += 128) {
          const unsigned long long bb = colB[jj], nn = colN[jj];
          colB[jj] = 0;
          colN[jj] = 0;
          const uint32_t j = j0 + jj;
          if ((bb | nn) && j < a.n_rows) {
            atomicAdd(&a.pv[2ull * (a.pv_row0 + j)], bb);
            atomicAdd(&a.pv[2ull * (a.pv_row0 + j) + 1], nn);
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
    }
    for (int o = 16; o; o >>= 1) {
      totB += __shfl_xor_sync(0xffffffffu, totB, o);
      totN += __shfl_xor_sync(0xffffffffu, totN, o);
    }
    if (lane == 0 && (totB | totN)) {
      atomicAdd(&a.acc[0], totB);
      atomicAdd(&a.acc[1], totN);
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// u8 A (0/1) / S (0, 1, 0xFF) rows -> e2m1 packed two per byte (element 2b in the low nibble):
// 0 -> 0x0, +1 -> 0x2 (1.0), -1 -> 0xA (-1.0); bytes beyond the u8 row are zero padding
__global__ void k_dense_pack_f4(const uint8_t* __restrict__ in, uint64_t k_in, uint8_t* __restrict__ out,
                                uint64_t k_out, uint64_t rows) {
  const uint64_t n8 = rows * (k_out / 8);  // 8 output bytes per thread
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n8; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = t / (k_out / 8), b0 = (t % (k_out / 8)) * 8;  // first output byte
    uint32_t w[2] = {0u, 0u};
    if (2 * b0 < k_in) {
      const uint4 q = *reinterpret_cast<const uint4*>(in + r * k_in + 2 * b0);  // 16 input bytes
      const uint32_t iw[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const uint32_t v = (iw[e >> 2] >> (8 * (e & 3))) & 0xFFu;
        const uint32_t nib = v == 1u ? 0x2u : (v == 0xFFu ? 0xAu : 0u);
        w[e >> 3] |= nib << (4 * (e & 7));
      }
    }
    *reinterpret_cast<uint2*>(out + r * k_out + b0) = make_uint2(w[0], w[1]);
  }
}

// tiles of the FP4 kernel: I over 256-row blocks, J over 224-row blocks, kept when the tile holds
// a pair i < j; super-tiles of 8 x 8 blocks for L2 reuse as in pair_tile_list
std::vector<uint2> f4_tile_list(uint32_t rows_pad) {
  std::vector<uint2> t;
  const uint32_t sb = getenv("BBF_F4_SB") ? std::max(1, atoi(getenv("BBF_F4_SB"))) : 8u;  // super-tile side (blocks)
  const uint32_t nI = rows_pad / kPB, nJ = (rows_pad + kF4N - 1) / kF4N;
  for (uint32_t JS = 0; JS < (nJ + sb - 1) / sb; ++JS)
    for (uint32_t IS = 0; IS < (nI + sb - 1) / sb; ++IS)
      for (uint32_t J = JS * sb; J < std::min(nJ, JS * sb + sb); ++J)
        for (uint32_t I = IS * sb; I < std::min(nI, IS * sb + sb); ++I)
          if (J * kF4N + kF4N - 1 > I * kPB) t.push_back(make_uint2(I, J));
  return t;
}

// upper-triangle pair tiles (I <= J over 256-row blocks) in super-tiles of 8 x 8 blocks, so the
// ~74 tiles in flight read ~16 distinct operand blocks (L2 reuse) instead of ~75
std::vector<uint2> pair_tile_list(uint32_t rows_pad) {
  std::vector<uint2> t;
  const uint32_t nb = rows_pad / kPB, sb = 8, ns = (nb + sb - 1) / sb;
  for (uint32_t JS = 0; JS < ns; ++JS)
    for (uint32_t IS = 0; IS <= JS; ++IS)
      for (uint32_t J = JS * sb; J < std::min(nb, JS * sb + sb); ++J)
        for (uint32_t I = IS * sb; I < std::min(nb, IS * sb + sb); ++I)
          if (I <= J) t.push_back(make_uint2(I, J));
  return t;
}

// A (0/1, u8) and S (+1/-1, s8) rows of both sides from the rank-space CSR: entry e of row x
// sets column l(y) of row x's side matrix
__global__ void k_dense_fill(const uint32_t* __restrict__ off, const uint32_t* __restrict__ adj,
                             uint32_t n, uint32_t n_u, uint64_t m, uint8_t* __restrict__ Au,
                             uint8_t* __restrict__ Su, uint64_t ku, uint8_t* __restrict__ Av,
                             uint8_t* __restrict__ Sv, uint64_t kv) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
       e += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = n;  // row: largest x with off[x] <= e
    while (hi - lo > 1) {
      uint32_t md = lo + (hi - lo) / 2;
      if (off[md] <= e) lo = md; else hi = md;
    }
    const uint32_t x = lo, w = adj[e];
    const uint8_t s = (w & kNegBit) ? (uint8_t)0xFF : (uint8_t)1;  // -1 / +1
    const uint64_t c = w & kMask;
    if (x < n_u) {
      if (Au) { Au[x * ku + c] = 1; Su[x * ku + c] = s; }
    } else {
      if (Av) { Av[(x - n_u) * kv + c] = 1; Sv[(x - n_u) * kv + c] = s; }
    }
  }
}

// 16 u8 operand bytes (0, 1 or 0xFF) -> 8 bytes of e2m1 pairs (element 2b in the low nibble):
// 0 -> 0x0, +1 -> 0x2 (1.0), -1 -> 0xA (-1.0)
__device__ __forceinline__ uint2 pack_e2m1(const uint4 q) {
  const uint32_t iw[4] = {q.x, q.y, q.z, q.w};
  uint32_t w[2] = {0u, 0u};
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const uint32_t v = (iw[e >> 2] >> (8 * (e & 3))) & 0xFFu;
    const uint32_t nib = v == 1u ? 0x2u : (v == 0xFFu ? 0xAu : 0u);
    w[e >> 3] |= nib << (4 * (e & 7));
  }
  return make_uint2(w[0], w[1]);
}

// A_U and S_U straight from the input U-side CSR, one CTA per rank row: the row is assembled in
// shared memory (A = 1, S = +1 / -1 per edge; weight 1 = +1, 0 = -1) and
// written out with 16-byte stores, so the operands need no memset and no scattered byte stores
__global__ void k_dense_rows(const uint64_t* __restrict__ rp, const uint32_t* __restrict__ col,
                             const uint8_t* __restrict__ sg, uint32_t n_u, const uint32_t* __restrict__ inv,
                             const uint32_t* __restrict__ lr_v, uint8_t* __restrict__ Au,
                             uint8_t* __restrict__ Su, uint32_t ku, unsigned long long* __restrict__ nz,
                             uint8_t* __restrict__ A4, uint8_t* __restrict__ S4, uint32_t k4) {
  extern __shared__ uint4 rowbuf[];
  uint8_t* ba = reinterpret_cast<uint8_t*>(rowbuf);
  uint8_t* bs = ba + ku;
  const uint32_t r = blockIdx.x, n16 = ku / 16;
  uint4* a4 = Au ? reinterpret_cast<uint4*>(Au + (uint64_t)r * ku) : nullptr;  // u8 copy optional
  uint4* s4 = Au ? reinterpret_cast<uint4*>(Su + (uint64_t)r * ku) : nullptr;
  if (r >= n_u) {  // padding rows
    if (a4)
      for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) { a4[i] = make_uint4(0u, 0u, 0u, 0u); s4[i] = a4[i]; }
    if (A4)
      for (uint32_t i = threadIdx.x; i < k4 / 8; i += blockDim.x) {
        reinterpret_cast<uint2*>(A4 + (uint64_t)r * k4)[i] = make_uint2(0u, 0u);
        reinterpret_cast<uint2*>(S4 + (uint64_t)r * k4)[i] = make_uint2(0u, 0u);
      }
    return;
  }
  for (uint32_t i = threadIdx.x; i < 2 * n16; i += blockDim.x) rowbuf[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();
  const uint32_t u = inv[r];
  for (uint64_t e = rp[u] + threadIdx.x; e < rp[u + 1]; e += blockDim.x) {
    const uint32_t c = lr_v[col[e]];
    ba[c] = 1;
    bs[c] = sg[e] ? (uint8_t)1 : (uint8_t)0xFF;
  }
  __syncthreads();
  uint32_t ones = 0;  // bytes are 0 / 1: a duplicate (u,v) sets one cell twice (count < nnz)
  for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) {
    const uint4 q = rowbuf[i];
    ones += __popc(q.x) + __popc(q.y) + __popc(q.z) + __popc(q.w);
    if (a4) {
      a4[i] = q;
      s4[i] = rowbuf[n16 + i];
    }
  }
  ones = __reduce_add_sync(0xffffffffu, ones);
  if ((threadIdx.x & 31) == 0 && ones) atomicAdd(nz, (unsigned long long)ones);
  if (A4)  // the FP4 path's packed copy of the row (zero beyond the u8 row)
    for (uint32_t i = threadIdx.x; i < k4 / 8; i += blockDim.x) {
      const bool in = 16u * i < ku;
      reinterpret_cast<uint2*>(A4 + (uint64_t)r * k4)[i] = in ? pack_e2m1(rowbuf[i]) : make_uint2(0u, 0u);
      reinterpret_cast<uint2*>(S4 + (uint64_t)r * k4)[i] = in ? pack_e2m1(rowbuf[n16 + i]) : make_uint2(0u, 0u);
    }
}

// FP4-only variant of k_dense_rows: the row is assembled directly as packed e2m1 nibbles in shared
// memory (A = 0x2, S = 0x2 / 0xA, set with shared atomicOr) and written with 16-byte stores; every
// present cell has exactly one set bit in A, so the popcount still counts distinct edges
__global__ void __launch_bounds__(256) k_dense_rows_f4(const uint64_t* __restrict__ rp,
                                                       const uint32_t* __restrict__ col,
                                                       const uint8_t* __restrict__ sg, uint32_t n_u,
                                                       const uint32_t* __restrict__ inv,
                                                       const uint32_t* __restrict__ lr_v,
                                                       unsigned long long* __restrict__ nz,
                                                       uint8_t* __restrict__ A4, uint8_t* __restrict__ S4,
                                                       uint32_t k4) {
  extern __shared__ uint4 rowbuf[];
  uint32_t* rw = reinterpret_cast<uint32_t*>(rowbuf);
  const uint32_t r = blockIdx.x, n16 = k4 / 16, nw = k4 / 4;
  uint4* a4 = reinterpret_cast<uint4*>(A4 + (uint64_t)r * k4);
  uint4* s4 = reinterpret_cast<uint4*>(S4 + (uint64_t)r * k4);
  if (r >= n_u) {  // padding rows
    for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) { a4[i] = make_uint4(0u, 0u, 0u, 0u); s4[i] = a4[i]; }
    return;
  }
  for (uint32_t i = threadIdx.x; i < 2 * n16; i += blockDim.x) rowbuf[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();
  const uint32_t u = inv[r];
  for (uint64_t e = rp[u] + threadIdx.x; e < rp[u + 1]; e += blockDim.x) {
    const uint32_t c = lr_v[col[e]], sh = 4 * (c & 7);
    atomicOr(&rw[c >> 3], 0x2u << sh);
    atomicOr(&rw[nw + (c >> 3)], (sg[e] ? 0x2u : 0xAu) << sh);  // weight 1 = +1, 0 = -1
  }
  __syncthreads();
  uint32_t ones = 0;
  for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) {
    const uint4 q = rowbuf[i];
    ones += __popc(q.x) + __popc(q.y) + __popc(q.z) + __popc(q.w);
    a4[i] = q;
    s4[i] = rowbuf[n16 + i];
  }
  ones = __reduce_add_sync(0xffffffffu, ones);
  if ((threadIdx.x & 31) == 0 && ones) atomicAdd(nz, (unsigned long long)ones);
}

// Av = Au^T and Sv = Su^T, 64 x 64 byte tiles: each thread loads a 4 x 4 byte block (four 4-byte
// row pieces), transposes it in registers (__byte_perm) and stages the words in shared memory so
// that the stores are 16-byte row pieces.  Av is rv x kv with rv >= n_v, kv >= n_u; rows of Av
// at or beyond ku (the width of Au) are zero.
__device__ __forceinline__ void transpose4x4(uint32_t (&w)[4]) {
  const uint32_t t0 = __byte_perm(w[0], w[1], 0x5140), t1 = __byte_perm(w[2], w[3], 0x5140);
  const uint32_t t2 = __byte_perm(w[0], w[1], 0x7362), t3 = __byte_perm(w[2], w[3], 0x7362);
  w[0] = __byte_perm(t0, t1, 0x5410);
  w[1] = __byte_perm(t0, t1, 0x7632);
  w[2] = __byte_perm(t2, t3, 0x5410);
  w[3] = __byte_perm(t2, t3, 0x7632);
}

__global__ void __launch_bounds__(256) k_dense_transpose(const uint8_t* __restrict__ Au,
                                                         const uint8_t* __restrict__ Su, uint32_t ku,
                                                         uint8_t* __restrict__ Av, uint8_t* __restrict__ Sv,
                                                         uint32_t kv, uint8_t* __restrict__ Av4,
                                                         uint8_t* __restrict__ Sv4, uint32_t kv4) {
  __shared__ uint32_t ta[64][17], ts[64][17];
  const uint32_t r0 = blockIdx.y * 64, c0 = blockIdx.x * 64;  // tile of Av: rows r0.., cols c0..
  const uint32_t t = threadIdx.x, bi = t >> 4, bj = t & 15;   // source rows c0 + 4 bi.., bytes r0 + 4 bj..
  uint32_t wa[4] = {0u, 0u, 0u, 0u}, ws[4] = {0u, 0u, 0u, 0u};
  if (r0 < ku) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t src = (uint64_t)(c0 + 4 * bi + k) * ku + r0 + 4 * bj;
      wa[k] = *reinterpret_cast<const uint32_t*>(Au + src);
      ws[k] = *reinterpret_cast<const uint32_t*>(Su + src);
    }
  }
  transpose4x4(wa);
  transpose4x4(ws);
#pragma unroll
  for (int k = 0; k < 4; ++k) { ta[4 * bj + k][bi] = wa[k]; ts[4 * bj + k][bi] = ws[k]; }
  __syncthreads();
  const uint32_t orow = t >> 2, oq = (t & 3) * 4;  // destination row r0 + orow, words oq .. oq + 3
  const uint64_t dst = (uint64_t)(r0 + orow) * kv + c0 + 4 * oq;
  const uint4 qa = make_uint4(ta[orow][oq], ta[orow][oq + 1], ta[orow][oq + 2], ta[orow][oq + 3]);
  const uint4 qs = make_uint4(ts[orow][oq], ts[orow][oq + 1], ts[orow][oq + 2], ts[orow][oq + 3]);
  if (Av) {  // u8 copy (int8 kernels); skipped when only the FP4 kernels will read this side
    *reinterpret_cast<uint4*>(Av + dst) = qa;
    *reinterpret_cast<uint4*>(Sv + dst) = qs;
  }
  if (Av4) {  // packed e2m1 copy (16 columns -> 8 bytes)
    const uint64_t d4 = (uint64_t)(r0 + orow) * kv4 + (c0 + 4 * oq) / 2;
    *reinterpret_cast<uint2*>(Av4 + d4) = pack_e2m1(qa);
    *reinterpret_cast<uint2*>(Sv4 + d4) = pack_e2m1(qs);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool make_map(CUtensorMap* m, void* base, uint64_t rows, uint64_t k, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {k, rows};
  cuuint64_t strides[1] = {k};
  cuuint32_t box[2] = {kBK, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

inline uint64_t round_up(uint64_t x, uint64_t m) { return (x + m - 1) / m * m; }

// upper-triangle tile list of one side (I over 128-row blocks, J over 256-row blocks), J outer
std::vector<uint2> tile_list(uint32_t rows_pad) {
  std::vector<uint2> t;
  const uint32_t nI = rows_pad / kBM, nJ = rows_pad / kBN;
  for (uint32_t J = 0; J < nJ; ++J)
    for (uint32_t I = 0; I < nI; ++I)
      if (J * kBN + kBN > I * kBM + 1) t.push_back(make_uint2(I, J));
  return t;
}

}  // namespace

// The dense path holds both sides' A and S (n_u_pad x n_v_pad bytes each, twice) and needs
// K = the other side padded to 128 to stay below 65,536 so every per-element count fits 32 bits.
bool dense_supported(bbf_graph* g) {
  const uint64_t ru = round_up(std::max<uint32_t>(g->n_u, 1), kBN), rv = round_up(std::max<uint32_t>(g->n_v, 1), kBN);
  const uint64_t ku = round_up(std::max<uint32_t>(g->n_v, 1), kBK), kv = round_up(std::max<uint32_t>(g->n_u, 1), kBK);
  if (ku > 65536 || kv > 65536) return false;
  const uint64_t bytes = 2 * (ru * ku + rv * kv);
  return bytes <= (16ull << 30);
}

// dense-vs-sparse choice: estimated int8 tensor time of both sides vs the
// sparse engine's measured wedge rate on W_pruned wedges
bool dense_preferred(bbf_graph* g, bool per_vertex) {
  if (!dense_supported(g) || (!g->wg_valid && !g->plan_g.valid)) return false;
  const double nu = g->n_u, nv = g->n_v;
  const double cu = nu * nu * round_up(g->n_v, kBK), cv = nv * nv * round_up(g->n_u, kBK);
  const double ops = 2.0 * (per_vertex ? cu + cv : std::min(cu, cv));
  // measured rates: the FP4 kernel ~5e15 int-ops/s (exact while max degree <= 8192), int8 ~3.5e15
  const bool f4 = std::max(g->maxdeg[0], g->maxdeg[1]) <= 8192u && !getenv("BBF_DENSE_I8");
  const double t_dense = ops / (f4 ? 5.0e15 : 3.5e15) + 1e-4;
  const double w = g->wg_valid ? (double)g->W_G : (double)g->plan_g.W_pruned;
  const double t_sparse = w / 2.0e11 + 1e-4;
  return t_dense < t_sparse;
}

bbf_status alloc_dense_operands(bbf_graph* g, bool zero) {
  cudaStream_t st = g->stream;
  g->drows[0] = round_up(std::max<uint32_t>(g->n_u, 1), kBN);
  g->drows[1] = round_up(std::max<uint32_t>(g->n_v, 1), kBN);
  g->dk[0] = round_up(std::max<uint32_t>(g->n_v, 1), kBK);
  g->dk[1] = round_up(std::max<uint32_t>(g->n_u, 1), kBK);
  for (int s2 = 0; s2 < 2; ++s2) {
    const uint64_t bytes = g->drows[s2] * g->dk[s2];
    BBF_CUDA(dmalloc(&g->dA[s2], bytes, st));
    BBF_CUDA(dmalloc(&g->dS[s2], bytes, st));
    if (zero) {
      BBF_CUDA(cudaMemsetAsync(g->dA[s2], 0, bytes, st));
      BBF_CUDA(cudaMemsetAsync(g->dS[s2], 0, bytes, st));
    }
  }
  return BBF_OK;
}

bbf_status build_dense_operands_f4(bbf_graph* g, const uint64_t* d_rp, const uint32_t* d_col,
                                   const uint8_t* d_sg) {
  cudaStream_t st = g->stream;
  g->drows[0] = round_up(std::max<uint32_t>(g->n_u, 1), kBN);
  g->drows[1] = round_up(std::max<uint32_t>(g->n_v, 1), kBN);
  g->dk[0] = round_up(std::max<uint32_t>(g->n_v, 1), kBK);
  g->dk[1] = round_up(std::max<uint32_t>(g->n_u, 1), kBK);
  for (int s2 = 0; s2 < 2; ++s2) {
    g->dk4[s2] = round_up(g->dk[s2], 256) / 2;
    BBF_CUDA(dmalloc(&g->dA4[s2], g->drows[s2] * g->dk4[s2], st));
    BBF_CUDA(dmalloc(&g->dS4[s2], g->drows[s2] * g->dk4[s2], st));
  }
  unsigned long long* d_nz;
  BBF_CUDA(dmalloc(&d_nz, 8, st));
  BBF_CUDA(cudaMemsetAsync(d_nz, 0, 8, st));
  const int smem = 2 * (int)g->dk4[0];
  if (smem > 48 * 1024)
    BBF_CUDA(cudaFuncSetAttribute(k_dense_rows_f4, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_dense_rows_f4<<<(unsigned)g->drows[0], 256, smem, st>>>(d_rp, d_col, d_sg, g->n_u, g->inv, g->lr + g->n_u,
                                                           d_nz, g->dA4[0], g->dS4[0], (uint32_t)g->dk4[0]);
  // V side: every V row (drows[1]) x every packed column (2 * dk4[1] elements)
  k_dense_transpose_f4<<<dim3((unsigned)(2 * g->dk4[1] / 128), (unsigned)(g->drows[1] / 128)), 256, 0, st>>>(
      g->dA4[0], g->dS4[0], (uint32_t)g->dk4[0], (uint32_t)g->drows[0], g->dA4[1], g->dS4[1], (uint32_t)g->dk4[1]);
  g->launches += 2;
  unsigned long long nz = 0;
  BBF_CUDA(rb_add(&nz, d_nz, 8, st)); g->launches++;
  BBF_CUDA(rb_sync(st));
  dfree(d_nz, st);
  if (nz != g->nnz) {
    set_error("duplicate (u,v) edge");
    return BBF_EDUP;
  }
  g->dense_built = true;
  g->dense_v_u8 = false;
  return BBF_OK;
}

// dense operands of both sides from the input CSR (device arrays), with the duplicate-edge check
// (SPEC.md:56): every edge sets one cell of A_U, so a duplicate leaves fewer than nnz ones
bbf_status build_dense_operands(bbf_graph* g, const uint64_t* d_rp, const uint32_t* d_col,
                                const uint8_t* d_sg) {
  cudaStream_t st = g->stream;
  // FP4-only graphs (both sides exact on the FP4 kernels, no int8 test hook): the packed operands
  // are built directly (rows, then a nibble transpose) and the u8 ones are skipped
  const bool f4_only = std::max(g->maxdeg[0], g->maxdeg[1]) <= 8192u && !getenv("BBF_DENSE_I8") &&
                       !getenv("BBF_DENSE_1CTA");
  if (f4_only) return build_dense_operands_f4(g, d_rp, d_col, d_sg);
  BBF_TRY(alloc_dense_operands(g, false));
  unsigned long long* d_nz;
  BBF_CUDA(dmalloc(&d_nz, 8, st));
  BBF_CUDA(cudaMemsetAsync(d_nz, 0, 8, st));
  {
    const uint32_t ku = (uint32_t)g->dk[0], kv = (uint32_t)g->dk[1];
    const int smem = 2 * (int)ku;
    if (smem > 48 * 1024)
      BBF_CUDA(cudaFuncSetAttribute(k_dense_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    // FP4 copies for the sides whose rows' max degree keeps the fp32 accumulation exact
    for (int s2 = 0; s2 < 2; ++s2) {
      if (g->maxdeg[s2] > 8192u || getenv("BBF_DENSE_I8") || g->dA4[s2]) continue;
      const uint64_t k4 = round_up(g->dk[s2], 256) / 2;
      BBF_CUDA(dmalloc(&g->dA4[s2], g->drows[s2] * k4, st));
      BBF_CUDA(dmalloc(&g->dS4[s2], g->drows[s2] * k4, st));
      g->dk4[s2] = k4;
      if (s2 == 1 && 2 * k4 > g->dk[1]) {  // the transpose leaves the padding columns unwritten
        BBF_CUDA(cudaMemsetAsync(g->dA4[1], 0, g->drows[1] * k4, st));
        BBF_CUDA(cudaMemsetAsync(g->dS4[1], 0, g->drows[1] * k4, st));
      }
    }
    k_dense_rows<<<(unsigned)g->drows[0], 256, smem, st>>>(d_rp, d_col, d_sg, g->n_u, g->inv, g->lr + g->n_u,
                                                          g->dA[0], g->dS[0], ku, d_nz, g->dA4[0], g->dS4[0],
                                                          (uint32_t)g->dk4[0]);
    const bool v_u8 = !g->dA4[1] || getenv("BBF_DENSE_1CTA");
    k_dense_transpose<<<dim3(kv / 64, (unsigned)(g->drows[1] / 64)), 256, 0, st>>>(
        g->dA[0], g->dS[0], ku, v_u8 ? g->dA[1] : nullptr, v_u8 ? g->dS[1] : nullptr, kv, g->dA4[1], g->dS4[1],
        (uint32_t)g->dk4[1]);
    g->dense_v_u8 = v_u8;
    g->launches += 2;
  }
  {
    unsigned long long nz = 0;
    BBF_CUDA(rb_add(&nz, d_nz, 8, st)); g->launches++;
    BBF_CUDA(rb_sync(st));
    dfree(d_nz, st);
    if (nz != g->nnz) {
      set_error("duplicate (u,v) edge");
      return BBF_EDUP;
    }
  }
  g->dense_built = true;
  return BBF_OK;
}

bbf_status run_dense(bbf_graph* g, bool per_vertex, int rank, int nranks, unsigned long long* host_BN) {
  NvtxRange nvtx_("bbf::dense_engine");
  cudaStream_t st = g->stream;
  if (!dense_supported(g)) {
    set_error("graph not supported by the dense int8 path");
    return BBF_EINVAL;
  }
  if (!encode_fn()) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return BBF_ECUDA;
  }
  // operands of both sides, built once per graph (at load for dense graphs, else here from the
  // rank-space adjacency) and kept until bbf_graph_free
  if (!g->dense_built) {
    if (g->in_rp) {
      BBF_TRY(build_dense_operands(g, g->in_rp, g->in_col, g->in_sg));
    } else {
      BBF_TRY(ensure_adj(g));
      BBF_TRY(alloc_dense_operands(g, true));
      const uint64_t m = 2 * g->nnz;
      if (m) {
        unsigned grid = (unsigned)std::min<uint64_t>((m + 255) / 256, 148u * 64u);
        k_dense_fill<<<grid, 256, 0, st>>>(g->off, g->adj, g->n, g->n_u, m, g->dA[0], g->dS[0], g->dk[0],
                                           g->dA[1], g->dS[1], g->dk[1]);
        g->launches++;
      }
      g->dense_built = true;
      g->dense_v_u8 = true;
    }
  }
  // an FP4-only graph asked for the int8 kernels (test hooks set after the load): u8 U side from
  // the kept input CSR; the V side follows from it on demand below
  if (!g->dA[0] && (getenv("BBF_DENSE_I8") || getenv("BBF_DENSE_1CTA") ||
                    std::max(g->maxdeg[0], g->maxdeg[1]) > 8192u)) {
    if (!g->in_rp) { set_error("internal: u8 dense operands requested without the input CSR"); return BBF_ECUDA; }
    BBF_TRY(alloc_dense_operands(g, false));
    unsigned long long* d_nz;
    BBF_CUDA(dmalloc(&d_nz, 8, st));
    const uint32_t ku = (uint32_t)g->dk[0];
    const int smem = 2 * (int)ku;
    if (smem > 48 * 1024)
      BBF_CUDA(cudaFuncSetAttribute(k_dense_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_dense_rows<<<(unsigned)g->drows[0], 256, smem, st>>>(g->in_rp, g->in_col, g->in_sg, g->n_u, g->inv,
                                                          g->lr + g->n_u, g->dA[0], g->dS[0], ku, d_nz, nullptr,
                                                          nullptr, 0u);
    g->launches++;
    dfree(d_nz, st);
    g->dense_v_u8 = false;
  }
  // global only: the cheaper side (cost ~ rows^2 * K); per-vertex: both sides
  const bool do_u = per_vertex || (uint64_t)g->n_u * g->n_u * g->n_v <= (uint64_t)g->n_v * g->n_v * g->n_u;
  const bool do_v = per_vertex || !do_u;
  const uint64_t ru = g->drows[0], rv = g->drows[1], ku = g->dk[0], kv = g->dk[1];
  uint8_t *Au = g->dA[0], *Su = g->dS[0], *Av = g->dA[1], *Sv = g->dS[1];
  BBF_CUDA(cudaMemsetAsync(g->d_acc, 0, 32 * sizeof(unsigned long long), st));
  BBF_CUDA(cudaFuncSetAttribute(k_dense_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes));
  BBF_CUDA(cudaFuncSetAttribute(k_dense_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPSmemBytes));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  unsigned long long BN_side[2][2] = {{0, 0}, {0, 0}};
  uint2* dtiles[2] = {nullptr, nullptr};
  bbf_status status = BBF_OK;
  double ops = 0;
  for (int side = 0; side < 2 && status == BBF_OK; ++side) {
    if (side == 0 ? !do_u : !do_v) continue;
    const uint64_t rows_pad = side ? rv : ru, k = side ? kv : ku;
    uint8_t* A = side ? Av : Au;
    uint8_t* S = side ? Sv : Su;
    const bool pair_kernel = !getenv("BBF_DENSE_1CTA");
    const bool f4_ok = pair_kernel && !getenv("BBF_DENSE_I8") && g->maxdeg[side] <= 8192u;
    if (side == 1 && !f4_ok && g->dense_built && !g->dense_v_u8) {  // int8 wanted: u8 V side on demand
      k_dense_transpose<<<dim3((unsigned)(kv / 64), (unsigned)(rv / 64)), 256, 0, st>>>(
          Au, Su, (uint32_t)ku, Av, Sv, (uint32_t)kv, nullptr, nullptr, 0u);
      g->launches++;
      g->dense_v_u8 = true;
    }
    // FP4 block-scaled path when exact (|T|, |P| and every partial sum <= the rows' max degree)
    const bool f4 = pair_kernel && !getenv("BBF_DENSE_I8") && g->maxdeg[side] <= 8192u;
    if (f4) {
      if (!g->dA4[side]) {  // packed operands, built once per graph
        const uint64_t k4 = round_up(k, 256) / 2;
        cudaError_t err = dmalloc(&g->dA4[side], rows_pad * k4, st);
        if (err == cudaSuccess) err = dmalloc(&g->dS4[side], rows_pad * k4, st);
        if (err != cudaSuccess) { status = cuda_status(err, "fp4 operands"); break; }
        const uint64_t n8 = rows_pad * (k4 / 8);
        const unsigned grid = (unsigned)std::min<uint64_t>((n8 + 255) / 256, 148ull * 32);
        k_dense_pack_f4<<<grid, 256, 0, st>>>(A, k, g->dA4[side], k4, rows_pad);
        k_dense_pack_f4<<<grid, 256, 0, st>>>(S, k, g->dS4[side], k4, rows_pad);
        g->launches += 2;
        g->dk4[side] = k4;
      }
      const uint64_t k4 = g->dk4[side];
      CUtensorMap fAi, fSi, fAj, fSj;
      if (!(make_map(&fAi, g->dA4[side], rows_pad, k4, 128) && make_map(&fSi, g->dS4[side], rows_pad, k4, 128) &&
            make_map(&fAj, g->dA4[side], rows_pad, k4, kF4JRows) && make_map(&fSj, g->dS4[side], rows_pad, k4, kF4JRows))) {
        set_error("cuTensorMapEncodeTiled failed");
        status = BBF_ECUDA;
        break;
      }
      std::vector<uint2> tl = f4_tile_list((uint32_t)rows_pad);
      cudaError_t err = dmalloc(&dtiles[side], sizeof(uint2) * (tl.size() + 1), st);
      if (err == cudaSuccess)
        err = cudaMemcpyAsync(dtiles[side], tl.data(), sizeof(uint2) * tl.size(), cudaMemcpyHostToDevice, st);
      if (err != cudaSuccess) { status = cuda_status(err, "dense tiles"); break; }
      DenseArgs da{};
      da.tiles = dtiles[side];
      da.n_tiles = (uint32_t)tl.size();
      da.n_rows = side ? g->n_v : g->n_u;
      da.n_kb = (uint32_t)(k4 / kBK);
      da.pv_row0 = side ? g->n_u : 0;
      da.n = g->n;
      da.rank = rank;
      da.nranks = nranks;
      da.pv = per_vertex ? (unsigned long long*)g->pv : nullptr;
      da.acc = g->d_acc + 2 * side;
      const unsigned pairs = (unsigned)std::min<uint64_t>(g->num_sms / 2, tl.size());
      if (g->maxdeg[side] < 2048u && !getenv("BBF_DENSE_F4_TP")) {  // one packed accumulator, double-buffered
        BBF_CUDA(cudaFuncSetAttribute(k_dense_f4q<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kQSmemBytes));
        k_dense_f4q<false><<<2 * pairs, kThreads, kQSmemBytes, st>>>(fAi, fSi, fAj, fSj, da);
      } else {
        BBF_CUDA(cudaFuncSetAttribute(k_dense_f4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kF4SmemBytes));
        k_dense_f4<<<2 * pairs, kThreads, kF4SmemBytes, st>>>(fAi, fSi, fAj, fSj, da);
      }
      g->launches++;
      const double nr = side ? g->n_v : g->n_u, kk = side ? g->n_u : g->n_v;
      ops += 2.0 * 2.0 * (nr * (nr - 1.0) / 2.0) * kk;
      err = cudaGetLastError();
      if (err != cudaSuccess) { status = cuda_status(err, "k_dense_f4 launch"); break; }
      continue;
    }
    CUtensorMap mAi, mSi, mAj, mSj;
    bool ok = pair_kernel ? (make_map(&mAi, A, rows_pad, k, 128) && make_map(&mSi, S, rows_pad, k, 128))
                          : (make_map(&mAi, A, rows_pad, k, kBM) && make_map(&mSi, S, rows_pad, k, kBM) &&
                             make_map(&mAj, A, rows_pad, k, kBN) && make_map(&mSj, S, rows_pad, k, kBN));
    if (!ok) {
      set_error("cuTensorMapEncodeTiled failed");
      status = BBF_ECUDA;
      break;
    }
    std::vector<uint2> tl = pair_kernel ? pair_tile_list((uint32_t)rows_pad) : tile_list((uint32_t)rows_pad);
    cudaError_t err = dmalloc(&dtiles[side], sizeof(uint2) * (tl.size() + 1), st);
    if (err == cudaSuccess)
      err = cudaMemcpyAsync(dtiles[side], tl.data(), sizeof(uint2) * tl.size(), cudaMemcpyHostToDevice, st);
    if (err != cudaSuccess) { status = cuda_status(err, "dense tiles"); break; }
    DenseArgs da{};
    da.tiles = dtiles[side];
    da.n_tiles = (uint32_t)tl.size();
    da.n_rows = side ? g->n_v : g->n_u;
    da.n_kb = (uint32_t)(k / kBK);
    da.pv_row0 = side ? g->n_u : 0;
    da.n = g->n;
    da.rank = rank;
    da.nranks = nranks;
    da.pv = per_vertex ? (unsigned long long*)g->pv : nullptr;
    da.acc = g->d_acc + 2 * side;
    if (pair_kernel) {
      const unsigned pairs = (unsigned)std::min<uint64_t>(g->num_sms / 2, tl.size());
      k_dense_pair<<<2 * pairs, kThreads, kPSmemBytes, st>>>(mAi, mSi, da);
    } else {
      const unsigned grid = (unsigned)std::min<uint64_t>(g->num_sms, tl.size());
      k_dense_tiles<<<grid, kThreads, kSmemBytes, st>>>(mAi, mSi, mAj, mSj, da);
    }
    g->launches++;
    // algorithmic int8 ops: T and P over the n(n-1)/2 pairs, K MACs each, 2 ops/MAC
    const double nr = side ? g->n_v : g->n_u, kk = side ? g->n_u : g->n_v;
    ops += 2.0 * 2.0 * (nr * (nr - 1.0) / 2.0) * kk;
    err = cudaGetLastError();
    if (err != cudaSuccess) { status = cuda_status(err, "k_dense_tiles launch"); break; }
  }
  cudaEventRecord(e1, st);
  unsigned long long h[4] = {0, 0, 0, 0};
  if (status == BBF_OK) {
    cudaError_t err = rb_add(h, g->d_acc, sizeof(h), st);
    g->launches++;
    if (err == cudaSuccess) err = rb_sync(st);
    if (err != cudaSuccess) status = cuda_status(err, "dense path");
  }
  float ms = 0;
  if (status == BBF_OK) cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  for (void* p : {(void*)dtiles[0], (void*)dtiles[1]})
    if (p) dfree(p, st);
  if (status != BBF_OK) return status;
  BN_side[0][0] = h[0]; BN_side[0][1] = h[1];
  BN_side[1][0] = h[2]; BN_side[1][1] = h[3];
  const int s0 = do_u ? 0 : 1;
  host_BN[0] = BN_side[s0][0];
  host_BN[1] = BN_side[s0][1];
  g->ms_main = ms;
  g->algo_bytes = 0;
  g->algo_ops = ops;
  if (getenv("BBF_DEBUG"))
    fprintf(stderr, "[bbf] dense: %.3f ms, %.3e int8 ops (%.1f TOPS), sides U=%d V=%d, B U/V %llu/%llu\n",
            ms, ops, ops / (ms * 1e-3) / 1e12, (int)do_u, (int)do_v, BN_side[0][0], BN_side[1][0]);
  return BBF_OK;
}

// One side of the hybrid path's dense core (hybrid.cu): the pair counts of the rows of a given u8
// operand pair, exactly as run_dense does for a whole side (same kernels, same epilogue, per-row
// counts into pv rows pv_row0 + i).  The FP4 copies are packed on first use into *A4 / *S4.
bbf_status dense_core_side(bbf_graph* g, uint32_t n_rows, uint64_t rows_pad, uint64_t k, uint8_t* A, uint8_t* S,
                           uint8_t** A4, uint8_t** S4, uint32_t maxdeg, uint32_t pv_row0, bool per_vertex,
                           int rank, int nranks, unsigned long long* acc, double* ops) {
  cudaStream_t st = g->stream;
  if (n_rows < 2) return BBF_OK;
  if (!encode_fn()) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return BBF_ECUDA;
  }
  const bool f4 = !getenv("BBF_DENSE_I8") && maxdeg <= 8192u;
  uint2* dt = nullptr;
  DenseArgs da{};
  da.n_rows = n_rows;
  da.pv_row0 = pv_row0;
  da.n = g->n;
  da.rank = rank;
  da.nranks = nranks;
  da.pv = per_vertex ? (unsigned long long*)g->pv : nullptr;
  da.acc = acc;
  std::vector<uint2> tl;
  CUtensorMap m0, m1, m2, m3;
  if (f4) {
    const uint64_t k4 = round_up(k, 256) / 2;
    if (!*A4) {
      BBF_CUDA(dmalloc(A4, rows_pad * k4, st));
      BBF_CUDA(dmalloc(S4, rows_pad * k4, st));
      const uint64_t n8 = rows_pad * (k4 / 8);
      const unsigned grid = (unsigned)std::min<uint64_t>((n8 + 255) / 256, 148ull * 32);
      k_dense_pack_f4<<<grid, 256, 0, st>>>(A, k, *A4, k4, rows_pad);
      k_dense_pack_f4<<<grid, 256, 0, st>>>(S, k, *S4, k4, rows_pad);
      g->launches += 2;
    }
    if (!(make_map(&m0, *A4, rows_pad, k4, 128) && make_map(&m1, *S4, rows_pad, k4, 128) &&
          make_map(&m2, *A4, rows_pad, k4, kF4JRows) && make_map(&m3, *S4, rows_pad, k4, kF4JRows))) {
      set_error("cuTensorMapEncodeTiled failed");
      return BBF_ECUDA;
    }
    tl = f4_tile_list((uint32_t)rows_pad);
    da.n_kb = (uint32_t)(k4 / kBK);
  } else {
    if (!(make_map(&m0, A, rows_pad, k, 128) && make_map(&m1, S, rows_pad, k, 128))) {
      set_error("cuTensorMapEncodeTiled failed");
      return BBF_ECUDA;
    }
    tl = pair_tile_list((uint32_t)rows_pad);
    da.n_kb = (uint32_t)(k / kBK);
  }
  BBF_CUDA(dmalloc(&dt, sizeof(uint2) * (tl.size() + 1), st));
  BBF_CUDA(cudaMemcpyAsync(dt, tl.data(), sizeof(uint2) * tl.size(), cudaMemcpyHostToDevice, st));
  da.tiles = dt;
  da.n_tiles = (uint32_t)tl.size();
  const unsigned pairs = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g->num_sms / 2, tl.size()));
  if (f4 && maxdeg < 2048u && !getenv("BBF_DENSE_F4_TP")) {
    BBF_CUDA(cudaFuncSetAttribute(k_dense_f4q<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kQSmemBytes));
    k_dense_f4q<false><<<2 * pairs, kThreads, kQSmemBytes, st>>>(m0, m1, m2, m3, da);
  } else if (f4) {
    BBF_CUDA(cudaFuncSetAttribute(k_dense_f4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kF4SmemBytes));
    k_dense_f4<<<2 * pairs, kThreads, kF4SmemBytes, st>>>(m0, m1, m2, m3, da);
  } else {
    BBF_CUDA(cudaFuncSetAttribute(k_dense_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPSmemBytes));
    k_dense_pair<<<2 * pairs, kThreads, kPSmemBytes, st>>>(m0, m1, da);
  }
  g->launches++;
  const cudaError_t err = cudaGetLastError();
  dfree(dt, st);
  if (err != cudaSuccess) return cuda_status(err, "dense core launch");
  const double nr = n_rows, kk = (double)k;
  *ops += 2.0 * 2.0 * (nr * (nr - 1.0) / 2.0) * kk;
  return BBF_OK;
}

// The hybrid path's mixed core pairs of one side (hybrid.cu), fused on the FP4 tensor cores:
// k_dense_f4q<true> over the I operand A', S' (each start row masked to its eligible core
// middles) and the J operand A, S, whose epilogue turns (T, P) into the core counts (a_c, d_c) of
// every pair i < j, adds the cross terms against the pair words R (row sums = the start's share,
// column sums = the end's, total = the global count) and leaves (a_c | d_c << 16) in R.  Exact
// while every row's core degree is < 2,048 (the packed accumulator); the caller checks.  Rows
// [xlo, xhi) (256-aligned: the caller's rank shard) are the I tiles launched.
bbf_status dense_core_cross(bbf_graph* g, uint32_t n_rows, uint64_t rows_pad, uint64_t k, uint8_t* Ae, uint8_t* Se,
                            uint8_t** Ae4, uint8_t** Se4, uint8_t* A, uint8_t* S, uint8_t** A4, uint8_t** S4,
                            uint32_t* R, uint32_t r_ld, uint32_t pv_row0, bool per_vertex, uint32_t xlo,
                            uint32_t xhi, unsigned long long* acc, double* ops) {
  cudaStream_t st = g->stream;
  if (n_rows < 2 || xhi <= xlo) return BBF_OK;
  if (!encode_fn()) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return BBF_ECUDA;
  }
  const uint64_t k4 = round_up(k, 256) / 2;
  const uint64_t n8 = rows_pad * (k4 / 8);
  const unsigned pgrid = (unsigned)std::min<uint64_t>((n8 + 255) / 256, 148ull * 32);
  uint8_t** outs[4] = {Ae4, Se4, A4, S4};
  uint8_t* ins[4] = {Ae, Se, A, S};
  for (int q = 0; q < 4; ++q)
    if (!*outs[q]) {
      BBF_CUDA(dmalloc(outs[q], rows_pad * k4, st));
      k_dense_pack_f4<<<pgrid, 256, 0, st>>>(ins[q], k, *outs[q], k4, rows_pad);
      g->launches++;
    }
  CUtensorMap m0, m1, m2, m3;
  if (!(make_map(&m0, *Ae4, rows_pad, k4, 128) && make_map(&m1, *Se4, rows_pad, k4, 128) &&
        make_map(&m2, *A4, rows_pad, k4, kF4JRows) && make_map(&m3, *S4, rows_pad, k4, kF4JRows))) {
    set_error("cuTensorMapEncodeTiled failed");
    return BBF_ECUDA;
  }
  // the I tiles (256-row blocks) of rows [xlo, xhi) only: the caller's pair words are zero elsewhere
  std::vector<uint2> tl;
  for (const uint2 t : f4_tile_list((uint32_t)rows_pad))
    if (t.x * kPB >= xlo && t.x * kPB < xhi) tl.push_back(t);
  if (tl.empty()) return BBF_OK;
  uint2* dt = nullptr;
  BBF_CUDA(dmalloc(&dt, sizeof(uint2) * (tl.size() + 1), st));
  BBF_CUDA(cudaMemcpyAsync(dt, tl.data(), sizeof(uint2) * tl.size(), cudaMemcpyHostToDevice, st));
  DenseArgs da{};
  da.tiles = dt;
  da.n_tiles = (uint32_t)tl.size();
  da.n_rows = n_rows;
  da.n_kb = (uint32_t)(k4 / kBK);
  da.pv_row0 = pv_row0;
  da.n = g->n;
  da.rank = 0;
  da.nranks = 1;
  da.pv = per_vertex ? (unsigned long long*)g->pv : nullptr;
  da.acc = acc;
  da.R = R;
  da.r_ld = r_ld;
  const unsigned pairs = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g->num_sms / 2, tl.size()));
  BBF_CUDA(cudaFuncSetAttribute(k_dense_f4q<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kQSmemBytes));
  k_dense_f4q<true><<<2 * pairs, kThreads, kQSmemBytes, st>>>(m0, m1, m2, m3, da);
  g->launches++;
  const cudaError_t err = cudaGetLastError();
  dfree(dt, st);
  if (err != cudaSuccess) return cuda_status(err, "dense cross launch");
  const double nr = n_rows;
  *ops += 2.0 * 2.0 * (nr * (nr - 1.0) / 2.0) * (double)k;
  return BBF_OK;
}

}  // namespace bbf
