// Microbenchmarks that size the sparse wedge-aggregation design on sm_100a:
// shared-memory atomic increments at random addresses (the S6 counter update),
// the same as plain warp-private read-modify-write, and L2 (global) reductions.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atomics atomics.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t lcg(uint32_t& s) { s = s * 1664525u + 1013904223u; return s >> 8; }

template <int NW>
__global__ void k_smem_atomic(uint32_t* out, int iters) {
  extern __shared__ uint32_t s[];
  for (int i = threadIdx.x; i < NW; i += blockDim.x) s[i] = 0;
  __syncthreads();
  uint32_t st = blockIdx.x * 7919u + threadIdx.x * 104729u + 1;
  #pragma unroll 8
  for (int i = 0; i < iters; ++i) {
    uint32_t a = lcg(st) % NW;
    atomicAdd(&s[a], (st & 1) ? 1u : 65536u);
  }
  __syncthreads();
  uint32_t acc = 0;
  for (int i = threadIdx.x; i < NW; i += blockDim.x) acc += s[i];
  if (acc == 0xdeadbeef) out[0] = acc;
}

// consecutive addresses per warp (one list segment of 32 distinct ends, in order)
template <int NW>
__global__ void k_smem_atomic_run(uint32_t* out, int iters) {
  extern __shared__ uint32_t s[];
  for (int i = threadIdx.x; i < NW; i += blockDim.x) s[i] = 0;
  __syncthreads();
  uint32_t st = blockIdx.x * 7919u + (threadIdx.x >> 5) * 104729u + 1;
  int lane = threadIdx.x & 31;
  #pragma unroll 8
  for (int i = 0; i < iters; ++i) {
    uint32_t base = lcg(st) % (NW - 64);
    atomicAdd(&s[base + lane * 2], 1u);  // a sorted run with gaps (typical list)
  }
  __syncthreads();
  uint32_t acc = 0;
  for (int i = threadIdx.x; i < NW; i += blockDim.x) acc += s[i];
  if (acc == 0xdeadbeef) out[0] = acc;
}

template <int NW>
__global__ void k_smem_rmw(uint32_t* out, int iters) {
  extern __shared__ uint32_t s[];
  const int nwarps = blockDim.x >> 5;
  const int per = NW / nwarps;
  uint32_t* mine = s + (threadIdx.x >> 5) * per;
  for (int i = threadIdx.x; i < NW; i += blockDim.x) s[i] = 0;
  __syncthreads();
  uint32_t st = blockIdx.x * 7919u + threadIdx.x * 104729u + 1;
  #pragma unroll 8
  for (int i = 0; i < iters; ++i) {
    uint32_t a = lcg(st) % per;
    uint32_t v = mine[a];
    mine[a] = v + ((st & 1) ? 1u : 65536u);
  }
  __syncthreads();
  uint32_t acc = 0;
  for (int i = threadIdx.x; i < NW; i += blockDim.x) acc += s[i];
  if (acc == 0xdeadbeef) out[0] = acc;
}

__global__ void k_gred(uint32_t* arr, uint32_t n, int iters) {
  uint32_t st = blockIdx.x * 7919u + threadIdx.x * 104729u + 1;
  #pragma unroll 8
  for (int i = 0; i < iters; ++i) {
    uint32_t a = (uint32_t)(((uint64_t)lcg(st) * 2654435761ull) % n);
    atomicAdd(&arr[a], 1u);
  }
}

__global__ void k_lds_random(uint32_t* out, int iters) {
  extern __shared__ uint32_t s[];
  const int NW = 12288;
  for (int i = threadIdx.x; i < NW; i += blockDim.x) s[i] = i;
  __syncthreads();
  uint32_t st = blockIdx.x * 7919u + threadIdx.x * 104729u + 1, acc = 0;
  #pragma unroll 8
  for (int i = 0; i < iters; ++i) acc += s[(lcg(st) ^ acc) % NW];
  if (acc == 0xdeadbeef) out[0] = acc;
}

template <typename K>
float timeit(K launch, int reps = 5) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int nsm = p.multiProcessorCount;
  int l2 = 0; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"gpu\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"clock_khz\":%d,\"smem_optin\":%zu}\n", p.name, nsm, l2, clk, p.sharedMemPerBlockOptin);
  uint32_t* out; CK(cudaMalloc(&out, 4));
  const int iters = 4096;
  // shared atomics, varying CTA size / window
  {
    const int NW = 12288;  // 48 KB per CTA, 4 CTAs/SM
    CK(cudaFuncSetAttribute(k_smem_atomic<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, NW * 4));
    for (int threads : {256, 512, 1024}) {
      int blocks = nsm * (2048 / threads);
      float ms = timeit([&] { k_smem_atomic<NW><<<blocks, threads, NW * 4>>>(out, iters); });
      double ops = (double)blocks * threads * iters;
      printf("{\"bench\":\"smem_atomic_random\",\"window_words\":%d,\"threads\":%d,\"blocks\":%d,\"Gops\":%.1f,\"ops_per_clk_per_sm\":%.3f}\n",
             NW, threads, blocks, ops / ms / 1e6, ops / (ms * 1e-3) / nsm / (clk * 1e3));
    }
  }
  {
    const int NW = 49152;  // 192 KB per CTA, 1 CTA/SM
    CK(cudaFuncSetAttribute(k_smem_atomic<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, NW * 4));
    int blocks = nsm, threads = 1024;
    float ms = timeit([&] { k_smem_atomic<NW><<<blocks, threads, NW * 4>>>(out, iters); });
    double ops = (double)blocks * threads * iters;
    printf("{\"bench\":\"smem_atomic_random\",\"window_words\":%d,\"threads\":%d,\"blocks\":%d,\"Gops\":%.1f,\"ops_per_clk_per_sm\":%.3f}\n",
           NW, threads, blocks, ops / ms / 1e6, ops / (ms * 1e-3) / nsm / (clk * 1e3));
    CK(cudaFuncSetAttribute(k_smem_atomic_run<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, NW * 4));
    ms = timeit([&] { k_smem_atomic_run<NW><<<blocks, threads, NW * 4>>>(out, iters); });
    printf("{\"bench\":\"smem_atomic_run\",\"window_words\":%d,\"threads\":%d,\"blocks\":%d,\"Gops\":%.1f,\"ops_per_clk_per_sm\":%.3f}\n",
           NW, threads, blocks, ops / ms / 1e6, ops / (ms * 1e-3) / nsm / (clk * 1e3));
    CK(cudaFuncSetAttribute(k_smem_rmw<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, NW * 4));
    ms = timeit([&] { k_smem_rmw<NW><<<blocks, threads, NW * 4>>>(out, iters); });
    printf("{\"bench\":\"smem_rmw_warp_private\",\"window_words\":%d,\"threads\":%d,\"blocks\":%d,\"Gops\":%.1f,\"ops_per_clk_per_sm\":%.3f}\n",
           NW, threads, blocks, ops / ms / 1e6, ops / (ms * 1e-3) / nsm / (clk * 1e3));
  }
  {
    CK(cudaFuncSetAttribute(k_lds_random, cudaFuncAttributeMaxDynamicSharedMemorySize, 12288 * 4));
    int blocks = nsm * 4, threads = 512;
    float ms = timeit([&] { k_lds_random<<<blocks, threads, 12288 * 4>>>(out, iters); });
    double ops = (double)blocks * threads * iters;
    printf("{\"bench\":\"lds_random\",\"Gops\":%.1f,\"ops_per_clk_per_sm\":%.3f}\n", ops / ms / 1e6, ops / (ms * 1e-3) / nsm / (clk * 1e3));
  }
  for (size_t bytes : {(size_t)2 << 20, (size_t)8 << 20, (size_t)32 << 20, (size_t)256 << 20}) {
    uint32_t* arr; CK(cudaMalloc(&arr, bytes)); cudaMemset(arr, 0, bytes);
    int blocks = nsm * 4, threads = 512;
    int it = 1024;
    float ms = timeit([&] { k_gred<<<blocks, threads>>>(arr, (uint32_t)(bytes / 4), it); });
    double ops = (double)blocks * threads * it;
    printf("{\"bench\":\"global_red_random\",\"array_MB\":%zu,\"Gops\":%.1f,\"ops_per_clk_per_sm\":%.3f}\n",
           bytes >> 20, ops / ms / 1e6, ops / (ms * 1e-3) / nsm / (clk * 1e3));
    cudaFree(arr);
  }
  return 0;
}
