// estimate.cu — NEXT-1 of SURVEY §8(f): SBESPAR one-shot sparsification (PAPER.md:1402-1438,
// §Approximation by Sparsification): keep every edge independently with probability rho, count
// the balanced butterflies of the sampled graph G' exactly (S1-S7 of the exact path, unchanged),
// and scale by rho^-4 (a butterfly survives iff its 4 edges do; reading R18).
//
// Edge draws come from a documented counter-based generator, so every sample is reproducible:
//   key_t = sm64(seed + t) for trial t, draw_e = sm64(key_t ^ e) for the e-th edge of the input
//   U-side CSR, keep iff rho >= 1 or draw_e < floor(rho * 2^64),
// with sm64 = SplitMix64 (one increment by the golden gamma, then the 30/27/31 xor-shift mixer).
#include <cub/cub.cuh>

#include <cmath>
#include <vector>

#include "bbf_internal.cuh"

namespace bbf {
namespace {

__host__ __device__ inline uint64_t sm64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_sample(uint64_t nnz, uint64_t key, uint64_t thr, bool all, uint32_t* __restrict__ keep) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (uint64_t)gridDim.x * blockDim.x)
    keep[e] = (all || sm64(key ^ e) < thr) ? 1u : 0u;
}

// pos = exclusive prefix of keep (nnz + 1 entries): new row_ptr[u] = pos[row_ptr[u]]
__global__ void k_sample_rows(const uint64_t* __restrict__ rp, uint32_t n_u, const uint32_t* __restrict__ pos,
                              uint64_t* __restrict__ nrp) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u <= n_u;
       u += (uint64_t)gridDim.x * blockDim.x)
    nrp[u] = pos[rp[u]];
}

__global__ void k_sample_compact(uint64_t nnz, const uint32_t* __restrict__ keep, const uint32_t* __restrict__ pos,
                                 const uint32_t* __restrict__ col, const uint8_t* __restrict__ sg,
                                 uint32_t* __restrict__ ncol, uint8_t* __restrict__ nsg) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (uint64_t)gridDim.x * blockDim.x)
    if (keep[e]) {
      ncol[pos[e]] = col[e];
      nsg[pos[e]] = sg[e];
    }
}

inline unsigned grid_for(uint64_t n) {
  uint64_t g = (n + 255) / 256;
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g, 148u * 64u));
}

}  // namespace
}  // namespace bbf

using namespace bbf;

extern "C" bbf_status bbf_estimate_global(uint32_t n_u, uint32_t n_v, const uint64_t* row_ptr,
                                          const uint32_t* col, const uint8_t* sign, uint32_t flags,
                                          double rho, uint32_t trials, uint64_t seed, int device,
                                          void* cuda_stream, bbf_comm* comm, uint64_t* sampled_balanced,
                                          uint64_t* sampled_unbalanced, double* estimates) {
  if (!row_ptr || !estimates) { set_error("null pointer"); return BBF_EINVAL; }
  if (!(rho > 0.0 && rho <= 1.0)) { set_error("rho must be in (0, 1]"); return BBF_EINVAL; }
  if (trials == 0) { set_error("trials == 0"); return BBF_EINVAL; }
  if (flags & ~(uint32_t)(BBF_PTR_DEVICE | BBF_FORCE_SPARSE | BBF_FORCE_DENSE)) { set_error("unknown flags"); return BBF_EINVAL; }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    set_error("no usable sm_100 CUDA device");
    return BBF_ECUDA;
  }
  BBF_CUDA(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  bool own_stream = false;
  if (!st) { BBF_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)); own_stream = true; }
  const bool dptr = flags & BBF_PTR_DEVICE;
  uint64_t nnz = 0;
  if (dptr) {
    BBF_CUDA(rb_add(&nnz, row_ptr + n_u, 8, st));
    BBF_CUDA(rb_sync(st));
  } else {
    nnz = row_ptr[n_u];
  }
  if (nnz >= (1ull << 31)) { set_error("nnz >= 2^31"); return BBF_ERANGE; }
  // device copies of the input, validated once (S1) before the sampling kernels read them
  // (each sample is validated again by its own load)
  uint64_t *d_rp = nullptr, *n_rp = nullptr;
  uint32_t *d_col = nullptr, *keep = nullptr, *pos = nullptr, *n_col = nullptr;
  uint8_t *d_sg = nullptr, *n_sg = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  bbf_status s = BBF_OK;
  auto fail = [&](cudaError_t e, const char* what) { s = cuda_status(e, what); };
  cudaError_t e = cudaSuccess;
  if (!dptr) {
    e = dmalloc(&d_rp, 8ull * (n_u + 1), st);
    if (e == cudaSuccess) e = dmalloc(&d_col, 4ull * (nnz + 1), st);
    if (e == cudaSuccess) e = dmalloc(&d_sg, nnz + 1, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_rp, row_ptr, 8ull * (n_u + 1), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && nnz) e = cudaMemcpyAsync(d_col, col, 4ull * nnz, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && nnz) e = cudaMemcpyAsync(d_sg, sign, nnz, cudaMemcpyHostToDevice, st);
  }
  const uint64_t* rp = dptr ? row_ptr : d_rp;
  const uint32_t* cl = dptr ? col : d_col;
  const uint8_t* sg = dptr ? sign : d_sg;
  if (e == cudaSuccess) e = dmalloc(&keep, 4ull * (nnz + 1), st);
  if (e == cudaSuccess) e = dmalloc(&pos, 4ull * (nnz + 1), st);
  if (e == cudaSuccess) e = dmalloc(&n_rp, 8ull * (n_u + 1), st);
  if (e == cudaSuccess) e = dmalloc(&n_col, 4ull * (nnz + 1), st);
  if (e == cudaSuccess) e = dmalloc(&n_sg, nnz + 1, st);
  if (e == cudaSuccess) {
    cub::DeviceScan::ExclusiveSum(nullptr, tb, keep, pos, (int64_t)(nnz + 1), st);
    e = dmalloc(&tmp, tb + 16, st);
  }
  if (e != cudaSuccess) fail(e, "estimate setup");
  if (s == BBF_OK) s = validate_csr(rp, n_u, cl, sg, nnz, n_v, st);
  const bool all = rho >= 1.0;
  const uint64_t thr = all ? ~0ull : (uint64_t)(rho * 18446744073709551616.0);  // floor(rho * 2^64)
  const double scale = 1.0 / (rho * rho * rho * rho);
  for (uint32_t t = 0; t < trials && s == BBF_OK; ++t) {
    const uint64_t key = sm64(seed + t);
    if (nnz) k_sample<<<grid_for(nnz), 256, 0, st>>>(nnz, key, thr, all, keep);
    e = cudaMemsetAsync(keep + nnz, 0, 4, st);
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(tmp, tb, keep, pos, (int64_t)(nnz + 1), st);
    if (e != cudaSuccess) { fail(e, "sample scan"); break; }
    k_sample_rows<<<grid_for(n_u + 1), 256, 0, st>>>(rp, n_u, pos, n_rp);
    if (nnz) k_sample_compact<<<grid_for(nnz), 256, 0, st>>>(nnz, keep, pos, cl, sg, n_col, n_sg);
    e = cudaGetLastError();
    if (e != cudaSuccess) { fail(e, "sample kernels"); break; }
    bbf_graph* g = nullptr;
    s = bbf_graph_load_csr(n_u, n_v, n_rp, n_col, n_sg,
                           BBF_PTR_DEVICE | (flags & (BBF_FORCE_SPARSE | BBF_FORCE_DENSE)), device, st,
                           comm, &g);
    if (s != BBF_OK) break;
    bbf_counts c;
    s = bbf_count_global(g, &c);
    bbf_graph_free(g);
    if (s != BBF_OK) break;
    if (sampled_balanced) sampled_balanced[t] = c.balanced;
    if (sampled_unbalanced) sampled_unbalanced[t] = c.unbalanced;
    estimates[t] = (double)c.balanced * scale;
  }
  for (void* p : {(void*)d_rp, (void*)d_col, (void*)d_sg, (void*)keep, (void*)pos, (void*)n_rp, (void*)n_col,
                  (void*)n_sg, tmp})
    if (p) dfree(p, st);
  cudaStreamSynchronize(st);
  if (own_stream) cudaStreamDestroy(st);
  return s;
}
