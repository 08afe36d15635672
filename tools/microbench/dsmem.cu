// Microbenchmark: distributed-shared-memory (DSMEM) atomics across a thread-block cluster on
// sm_100a — the candidate for cluster-wide counter windows in the hub kernel.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem dsmem.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t lcg(uint32_t& s) { s = s * 1664525u + 1013904223u; return s >> 8; }

__device__ __forceinline__ void red_cluster(uint32_t saddr_cluster, uint32_t v) {
  asm volatile("red.shared::cluster.add.u32 [%0], %1;" :: "r"(saddr_cluster), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}

template <int NW>
__global__ void k_dsmem(uint32_t* out, int iters, int remote_mode) {
  extern __shared__ uint32_t s[];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t csize = cl.num_blocks();
  for (int i = threadIdx.x; i < NW; i += blockDim.x) s[i] = 0;
  cl.sync();
  uint32_t st = blockIdx.x * 7919u + threadIdx.x * 104729u + 1;
  uint32_t base = (uint32_t)__cvta_generic_to_shared(s);
  uint32_t myrank = cl.block_rank();
  #pragma unroll 4
  for (int i = 0; i < iters; ++i) {
    uint32_t r = lcg(st);
    uint32_t a = r % NW;
    uint32_t rank = remote_mode ? (r >> 20) % csize : myrank;
    red_cluster(mapa(base + 4 * a, rank), 1u);
  }
  cl.sync();
  uint32_t acc = 0;
  for (int i = threadIdx.x; i < NW; i += blockDim.x) acc += s[i];
  if (acc == 0xdeadbeef) out[0] = acc;
}

template <typename K>
float timeit(K launch, int reps = 5) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  launch(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* out; cudaMalloc(&out, 4);
  const int NW = 48 * 1024;
  auto kern = k_dsmem<NW>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, NW * 4);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int iters = 2048;
  for (int cs : {1, 2, 4, 8, 16}) {
    for (int remote = 0; remote < 2; ++remote) {
      if (cs == 1 && remote) continue;
      int threads = 1024;
      cudaLaunchConfig_t cfg{};
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = NW * 4;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr; cfg.numAttrs = 1;
      int nclusters = 0;
      cfg.gridDim = dim3(cs);
      cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg);
      if (nclusters <= 0) { printf("{\"bench\":\"dsmem\",\"cluster\":%d,\"error\":\"cannot launch (max clusters %d): %s\"}\n", cs, nclusters, cudaGetErrorString(cudaGetLastError())); continue; }
      cfg.gridDim = dim3(cs * nclusters);
      float ms = timeit([&] { cudaLaunchKernelEx(&cfg, kern, out, iters, remote); });
      cudaError_t e = cudaGetLastError();
      double ops = (double)cs * nclusters * threads * iters;
      printf("{\"bench\":\"dsmem_red\",\"cluster\":%d,\"clusters\":%d,\"remote\":%d,\"Gops\":%.1f,\"ops_per_clk_per_sm\":%.3f,\"err\":\"%s\"}\n",
             cs, nclusters, remote, ops / ms / 1e6, ops / (ms * 1e-3) / (cs * nclusters) / (clk * 1e3), cudaGetErrorString(e));
    }
  }
  return 0;
}
