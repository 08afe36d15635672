// microbenchmark: V-degree histogram variants over a col array (tools only, not the product)
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_plain(const uint32_t* __restrict__ col, uint64_t n, uint32_t* __restrict__ d) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n; e += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&d[col[e]], 1u);
}
// block-local hash aggregation: 4096-slot smem table (key, count), flush per block chunk
template <int kSlots, int P>
__global__ void k_hash(const uint32_t* __restrict__ col, uint64_t n, uint32_t* __restrict__ d, uint32_t chunk) {
  __shared__ uint32_t key[kSlots], cnt[kSlots];
  for (uint64_t c0 = (uint64_t)blockIdx.x * chunk; c0 < n; c0 += (uint64_t)gridDim.x * chunk) {
    for (int i = threadIdx.x; i < kSlots; i += blockDim.x) { key[i] = 0xffffffffu; cnt[i] = 0; }
    __syncthreads();
    uint64_t c1 = c0 + chunk < n ? c0 + chunk : n;
    for (uint64_t e = c0 + threadIdx.x; e < c1; e += blockDim.x) {
      uint32_t v = col[e];
      uint32_t h = (v * 2654435761u) >> (32 - __popc(kSlots - 1));
      bool done = false;
      for (int p = 0; p < P && !done; ++p) {
        uint32_t s = (h + p) & (kSlots - 1);
        uint32_t k = key[s];
        if (k == 0xffffffffu) k = atomicCAS(&key[s], 0xffffffffu, v);
        if (k == 0xffffffffu || k == v) { atomicAdd(&cnt[s], 1u); done = true; }
      }
      if (!done) atomicAdd(&d[v], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kSlots; i += blockDim.x)
      if (cnt[i]) atomicAdd(&d[key[i]], cnt[i]);
    __syncthreads();
  }
}
extern "C" float run(int variant, const uint32_t* col, uint64_t n, uint32_t* d, uint32_t nv, int reps, uint32_t chunk) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < reps; ++r) {
    cudaMemset(d, 0, 4ull * nv);
    cudaEventRecord(a);
    if (variant == 0) k_plain<<<(unsigned)((n + 255) / 256), 256>>>(col, n, d);
    else if (variant == 1) k_hash<4096, 8><<<148 * 4, 512>>>(col, n, d, chunk);
    else if (variant == 2) k_hash<4096, 1><<<148 * 4, 512>>>(col, n, d, chunk);
    else if (variant == 3) k_hash<4096, 2><<<148 * 2, 1024>>>(col, n, d, chunk);
    else if (variant == 4) k_hash<2048, 2><<<148 * 8, 256>>>(col, n, d, chunk);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}
