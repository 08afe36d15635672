// mem.cu — the library's device-memory cache.  Every device buffer of libbbf.so (graph arrays,
// plan and build temporaries, hub-kernel scratch) comes from here: blocks released by dfree go
// to a per-device free list (with an event recorded on the releasing stream) and are handed
// out again to later requests of similar size, so repeated load / count / free cycles never go
// back to the driver.  Fresh blocks come from cudaMallocAsync; cached blocks are never returned
// (they live until process exit).  Thread-safe.
#include <map>
#include <mutex>
#include <unordered_map>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "bbf_internal.cuh"

namespace bbf {
namespace {

struct Block {
  void* p;
  size_t size;
  cudaStream_t st;
  cudaEvent_t ev;
};

struct Live {
  int dev;
  size_t size;   // block size
  void* base;    // block start (the returned pointer is base + kGuard in guard mode)
  size_t bytes;  // requested bytes
};
struct Cache {
  std::mutex mu;
  std::multimap<size_t, Block> free_by_size[64];  // per device
  std::unordered_map<void*, Live> live;            // returned ptr -> block
};

// Guard mode (BBF_GUARD=1, a debugging aid in place of compute-sanitizer, which this pool does
// not offer): every block gets kGuard bytes of 0xA5 before the returned pointer and from the end
// of the requested bytes to the end of the block; dfree synchronises the stream, reads both
// guards back and aborts the process on any changed byte (an out-of-bounds write by a kernel).
constexpr size_t kGuard = 256;
constexpr uint8_t kGuardByte = 0xA5;
bool guard_mode() {
  static const bool on = [] { const char* e = getenv("BBF_GUARD"); return e && atoi(e) != 0; }();
  return on;
}

void guard_check(const Live& L, cudaStream_t st) {
  if (cudaStreamSynchronize(st) != cudaSuccess) return;  // the error surfaces elsewhere
  const size_t tail_off = kGuard + L.bytes, tail = L.size - tail_off;
  std::vector<uint8_t> h(kGuard + tail);
  if (cudaMemcpy(h.data(), L.base, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(h.data() + kGuard, (uint8_t*)L.base + tail_off, tail, cudaMemcpyDeviceToHost) != cudaSuccess)
    return;
  for (size_t i = 0; i < h.size(); ++i)
    if (h[i] != kGuardByte) {
      const bool front = i < kGuard;
      fprintf(stderr, "[bbf] BBF_GUARD: out-of-bounds write %s a block of %zu bytes (guard byte %zd: 0x%02x)\n",
              front ? "before" : "after", L.bytes, front ? (ssize_t)i - (ssize_t)kGuard : (ssize_t)(i - kGuard),
              h[i]);
      abort();
    }
}

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

cudaError_t dmalloc_raw(void** out, size_t bytes, cudaStream_t st) { return dmalloc_raw2(out, bytes, st, false); }

// A request reuses a cached block of similar size (<= 1.25x + 64 MiB) that needs no wait: released
// on `st` itself, or released on another stream whose work has already completed.  Otherwise it
// takes fresh memory rather than making `st` wait for another stream's pending work (e.g. an
// asynchronous output copy that is meant to overlap the next graph's build); only when the device
// is out of memory does it reuse a busy block behind a stream wait (never, with no_wait), and then
// give the whole cache back to the driver.
cudaError_t dmalloc_raw2(void** out, size_t bytes, cudaStream_t st, bool no_wait) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  Cache& c = cache();
  const bool gm = guard_mode();
  const size_t need = round_size((bytes ? bytes : 1) + (gm ? 2 * kGuard : 0));
  const size_t lim = need + need / 4 + (64u << 20);
  auto hand_out = [&](void* base, size_t size) {  // caller holds c.mu
    void* user = gm ? (void*)((uint8_t*)base + kGuard) : base;
    c.live[user] = Live{dev, size, base, bytes};
    if (gm) {
      cudaMemsetAsync(base, kGuardByte, kGuard, st);
      cudaMemsetAsync((uint8_t*)base + kGuard + bytes, kGuardByte, size - kGuard - bytes, st);
    }
    *out = user;
  };
  auto take = [&](std::multimap<size_t, Block>& fl, std::multimap<size_t, Block>::iterator it) {
    Block b = it->second;
    fl.erase(it);
    cudaStreamWaitEvent(st, b.ev, 0);  // no-op when complete or already ordered
    cudaEventDestroy(b.ev);
    hand_out(b.p, b.size);
  };
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto& fl = c.free_by_size[dev];
    for (auto jt = fl.lower_bound(need); jt != fl.end() && jt->first <= lim; ++jt) {
      if (jt->second.st == st || cudaEventQuery(jt->second.ev) == cudaSuccess) {
        take(fl, jt);
        return cudaSuccess;
      }
    }
  }
  void* p = nullptr;
  e = cudaMallocAsync(&p, need, st);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    std::lock_guard<std::mutex> lk(c.mu);
    auto& fl = c.free_by_size[dev];
    auto it = fl.lower_bound(need);
    if (!no_wait && it != fl.end() && it->first <= lim) {  // a busy block, behind a stream wait
      take(fl, it);
      return cudaSuccess;
    }
    // give every cached block of this device back to the pool and retry
    for (auto& kv : fl) {
      cudaStreamWaitEvent(st, kv.second.ev, 0);
      cudaEventDestroy(kv.second.ev);
      cudaFreeAsync(kv.second.p, st);
    }
    fl.clear();
    e = cudaMallocAsync(&p, need, st);
  }
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(c.mu);
  hand_out(p, need);
  return cudaSuccess;
}

void dfree(void* p, cudaStream_t st) {
  if (!p) return;
  Cache& c = cache();
  std::lock_guard<std::mutex> lk(c.mu);
  auto it = c.live.find(p);
  if (it == c.live.end()) return;  // not ours
  const Live L = it->second;
  const int dev = L.dev;
  const size_t size = L.size;
  p = L.base;
  c.live.erase(it);
  if (guard_mode()) guard_check(L, st);
  cudaEvent_t ev;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
    cudaFreeAsync(p, st);
    return;
  }
  cudaEventRecord(ev, st);
  c.free_by_size[dev].emplace(size, Block{p, size, st, ev});
}

// ---------------------------------------------------------------------------- small readbacks
// Host values the library needs mid-build (error flags, counts, sizes) are read back through
// mapped pinned memory by a one-warp copy kernel instead of cudaMemcpyAsync: a copy command
// would queue behind large asynchronous copies of other streams on the same copy engine (e.g.
// BBF_OUTPUT_ASYNC outputs of the previous graph), stalling the build for their whole duration.
namespace {
__global__ void k_rb_copy(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, uint32_t n) {
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}
struct RbEntry {
  void* host;
  size_t off, n;
  cudaStream_t st;
};
struct RbState {
  uint8_t* hbuf = nullptr;  // mapped pinned, kRbBytes
  uint8_t* dbuf = nullptr;  // its device address
  size_t used = 0;
  std::vector<RbEntry> pending;
};
constexpr size_t kRbBytes = 1 << 16;
thread_local RbState t_rb;
}  // namespace

cudaError_t rb_add(void* host, const void* dev, size_t n, cudaStream_t st) {
  RbState& r = t_rb;
  if (!r.hbuf) {
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&r.hbuf), kRbBytes, cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) { r.hbuf = nullptr; return e; }
    e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&r.dbuf), r.hbuf, 0);
    if (e != cudaSuccess) return e;
  }
  const size_t off = (r.used + 15) & ~size_t(15);
  if (n == 0) return cudaSuccess;
  if (off + n > kRbBytes) {  // too large for the slots: an ordinary copy
    return cudaMemcpyAsync(host, dev, n, cudaMemcpyDeviceToHost, st);
  }
  k_rb_copy<<<1, 32, 0, st>>>(r.dbuf + off, reinterpret_cast<const uint8_t*>(dev), (uint32_t)n);
  r.used = off + n;
  r.pending.push_back(RbEntry{host, off, n, st});
  return cudaGetLastError();
}

cudaError_t rb_sync(cudaStream_t st) {
  cudaError_t e = cudaStreamSynchronize(st);
  RbState& r = t_rb;
  std::vector<RbEntry> keep;
  for (const RbEntry& x : r.pending) {
    if (x.st == st) {
      if (e == cudaSuccess) std::memcpy(x.host, r.hbuf + x.off, x.n);
    } else {
      keep.push_back(x);
    }
  }
  r.pending.swap(keep);
  if (r.pending.empty()) r.used = 0;
  return e;
}

}  // namespace bbf
