// mem.cu — the library's device-memory cache.  Every device buffer of libbbf.so (graph arrays,
// plan and build temporaries, hub-kernel scratch) comes from here: blocks released by dfree go
// to a per-device free list (with an event recorded on the releasing stream) and are handed
// out again to later requests of similar size, so repeated load / count / free cycles never go
// back to the driver.  Fresh blocks come from cudaMallocAsync; cached blocks are never returned
// (they live until process exit).  Thread-safe.
#include <map>
#include <mutex>
#include <unordered_map>

#include "bbf_internal.cuh"

namespace bbf {
namespace {

struct Block {
  void* p;
  size_t size;
  cudaStream_t st;
  cudaEvent_t ev;
};

struct Cache {
  std::mutex mu;
  std::multimap<size_t, Block> free_by_size[64];        // per device
  std::unordered_map<void*, std::pair<int, size_t>> live;  // ptr -> (device, size)
};

Cache& cache() {
  static Cache* c = new Cache();  // intentionally leaked: blocks outlive static destruction
  return *c;
}

inline size_t round_size(size_t b) {
  if (b <= 512) return 512;
  if (b <= (1u << 20)) {  // powers of two up to 1 MiB
    size_t r = 1024;
    while (r < b) r <<= 1;
    return r;
  }
  return (b + (2u << 20) - 1) & ~size_t((2u << 20) - 1);  // 2 MiB granules
}

}  // namespace

cudaError_t dmalloc_raw(void** out, size_t bytes, cudaStream_t st) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  const size_t need = round_size(bytes ? bytes : 1);
  Cache& c = cache();
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto& fl = c.free_by_size[dev];
    auto it = fl.lower_bound(need);
    // reuse a cached block no larger than 1.25x the request (+ 64 MiB slack for big ones)
    if (it != fl.end() && it->first <= need + need / 4 + (64u << 20)) {
      Block b = it->second;
      fl.erase(it);
      cudaStreamWaitEvent(st, b.ev, 0);  // no-op wait when already ordered / complete
      cudaEventDestroy(b.ev);
      c.live[b.p] = {dev, b.size};
      *out = b.p;
      return cudaSuccess;
    }
  }
  void* p = nullptr;
  e = cudaMallocAsync(&p, need, st);
  if (e == cudaErrorMemoryAllocation) {
    // out of memory: give every cached block of this device back to the pool and retry
    std::lock_guard<std::mutex> lk(c.mu);
    for (auto& kv : c.free_by_size[dev]) {
      cudaStreamWaitEvent(st, kv.second.ev, 0);
      cudaEventDestroy(kv.second.ev);
      cudaFreeAsync(kv.second.p, st);
    }
    c.free_by_size[dev].clear();
    cudaGetLastError();
    e = cudaMallocAsync(&p, need, st);
  }
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(c.mu);
  c.live[p] = {dev, need};
  *out = p;
  return cudaSuccess;
}

void dfree(void* p, cudaStream_t st) {
  if (!p) return;
  Cache& c = cache();
  std::lock_guard<std::mutex> lk(c.mu);
  auto it = c.live.find(p);
  if (it == c.live.end()) return;  // not ours
  const int dev = it->second.first;
  const size_t size = it->second.second;
  c.live.erase(it);
  cudaEvent_t ev;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
    cudaFreeAsync(p, st);
    return;
  }
  cudaEventRecord(ev, st);
  c.free_by_size[dev].emplace(size, Block{p, size, st, ev});
}

}  // namespace bbf
