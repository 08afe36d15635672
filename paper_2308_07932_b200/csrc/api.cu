// api.cu — the C ABI of libbbf.so (include/bbf.h): handle lifetime, status codes, the count
// entry points, per-vertex output mapping (S9) and the multi-GPU reduction (S12, NCCL u64 sum).
#include <cub/cub.cuh>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "bbf_internal.cuh"

namespace bbf {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

bbf_status cuda_status(cudaError_t e, const char* what) {
  g_last_error = std::string("CUDA error: ") + cudaGetErrorString(e) + " in " + what;
  if (e == cudaErrorMemoryAllocation) return BBF_ENOMEM;
  return BBF_ECUDA;
}

// ---------------------------------------------------------------------------- NCCL (dlopen)
namespace {
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
    api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
    api.CommGetAsyncError = (decltype(api.CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
    api.CommAbort = (decltype(api.CommAbort))dlsym(h, "ncclCommAbort");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.AllGather &&
             api.CommGetAsyncError && api.CommAbort;
  });
  return api;
}

bbf_status nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return BBF_OK;
  const char* s = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
  set_error(std::string("NCCL error: ") + s + " in " + what);
  return BBF_ENCCL;
}

bool device_ok(int device, int* num_sms) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) return false;
  int major = 0, sms = 0;  // attributes, not cudaGetDeviceProperties (milliseconds per call)
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess) return false;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return false;
  if (major < 10) return false;
  if (num_sms) *num_sms = sms;
  return true;
}

// Keep freed stream-ordered memory in the device's default pool: a graph's buffers are
// re-allocated on every load, and returning them to the driver at each synchronisation costs
// more than the count itself on large graphs.
void keep_pool(int device) {
  static std::once_flag flags[64];
  if (device < 0 || device >= 64) return;
  std::call_once(flags[device], [device] {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
}

// rank space -> input ids (S9)
__global__ void k_scatter_pv(const unsigned long long* __restrict__ pv, const uint32_t* __restrict__ inv,
                             uint32_t row0, uint32_t cnt, uint32_t n, unsigned long long* __restrict__ ob,
                             unsigned long long* __restrict__ on) {
  uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= cnt) return;
  uint32_t id = inv[row0 + r];
  if (ob) ob[id] = pv[2ull * (row0 + r)];       // (B, N) interleaved per row
  if (on) on[id] = pv[2ull * (row0 + r) + 1];
}

// per-edge counts, rank space -> input CSR order: edge i = (u, col[i]) of the caller's CSR; its
// slot is u's rank-space row entry holding l(col[i]) (rows ascending by local rank, bit 31 = sign)
__global__ void k_edge_out(uint32_t n_u, uint32_t n_v, const uint64_t* __restrict__ rp, const uint32_t* __restrict__ col,
                           uint64_t nnz, const uint32_t* __restrict__ lr, const uint32_t* __restrict__ off,
                           const uint32_t* __restrict__ adj, const unsigned long long* __restrict__ edge,
                           unsigned long long* __restrict__ ob, unsigned long long* __restrict__ on,
                           uint32_t* __restrict__ err) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nnz; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = n_u;  // u: the row with rp[u] <= i < rp[u + 1]
    while (hi - lo > 1) {
      const uint32_t md = lo + (hi - lo) / 2;
      if (rp[md] <= i) lo = md; else hi = md;
    }
    if (col[i] >= n_v) { atomicOr(err, 1u); continue; }
    const uint32_t r = lr[lo], lv = lr[n_u + col[i]];
    uint32_t a = off[r], b = off[r + 1];  // first entry with local rank >= lv
    while (a < b) {
      const uint32_t md = a + (b - a) / 2;
      if ((adj[md] & kMask) < lv) a = md + 1; else b = md;
    }
    if (a >= off[r + 1] || (adj[a] & kMask) != lv) { atomicOr(err, 1u); continue; }
    if (ob) ob[i] = edge[2ull * a];
    if (on) on[i] = edge[2ull * a + 1];
  }
}

// per-vertex score (balanced count or degree) of one side in input-id order, ids ascending
__global__ void k_rank_scores(const unsigned long long* __restrict__ pv, const uint32_t* __restrict__ degs,
                              const uint32_t* __restrict__ inv, uint32_t row0, uint32_t cnt, bool degree,
                              unsigned long long* __restrict__ score, uint32_t* __restrict__ id) {
  uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= cnt) return;
  const uint32_t i = inv[row0 + r];
  score[i] = degree ? (unsigned long long)degs[row0 + r] : pv[2ull * (row0 + r)];
  id[i] = i;
}

// a communicator is attached (also with one rank: the collectives then run as single-rank NCCL
// operations, which is how the N > 1 code path is exercised on a one-GPU box)
bool multi_rank(const bbf_graph* g) { return g->comm && g->comm->nccl; }

bbf_status allreduce_u64(bbf_graph* g, unsigned long long* dbuf, size_t count, ncclRedOp_t op = ncclSum) {
  if (!multi_rank(g) || !count) return BBF_OK;
  return nccl_status(nccl().AllReduce(dbuf, dbuf, count, ncclUint64, op, (ncclComm_t)g->comm->nccl, g->stream),
                     "ncclAllReduce");
}

// Wait for the graph's stream.  With a communicator the wait polls ncclCommGetAsyncError, so a
// peer that failed (or a network error) surfaces as BBF_ENCCL instead of a hang; the
// communicator is then aborted and unusable (bbf_comm_free still releases it).
bbf_status sync_stream(bbf_graph* g) {
  if (!multi_rank(g)) {
    BBF_CUDA(cudaStreamSynchronize(g->stream));
    return BBF_OK;
  }
  while (true) {
    const cudaError_t e = cudaStreamQuery(g->stream);
    if (e == cudaSuccess) return BBF_OK;
    if (e != cudaErrorNotReady) return cuda_status(e, "stream wait");
    ncclResult_t ar = ncclSuccess;
    nccl().CommGetAsyncError((ncclComm_t)g->comm->nccl, &ar);
    if (ar != ncclSuccess && ar != ncclInProgress) {
      nccl().CommAbort((ncclComm_t)g->comm->nccl);
      g->comm->nccl = nullptr;
      return nccl_status(ar, "communicator (asynchronous error)");
    }
  }
}

// Collective completion of a count on every rank: every rank enters the same
// collectives whatever its local status — the local (B, N) partials are summed, the per-vertex
// array (per_vertex) is summed, and the ranks' status codes are max-reduced — so a rank that
// failed locally (an allocation, a table limit) makes every rank return that error instead of
// leaving the others blocked in the all-reduce.  BN: host (B, N), replaced by the global sums.
bbf_status finish_collective(bbf_graph* g, bbf_status local, bool per_vertex, unsigned long long* BN) {
  NvtxRange nvtx_("bbf::collective");
  if (!multi_rank(g)) return local;
  unsigned long long h[3] = {local == BBF_OK ? BN[0] : 0ull, local == BBF_OK ? BN[1] : 0ull,
                             (unsigned long long)local};
  const std::string msg = local == BBF_OK ? std::string() : g_last_error;
  BBF_CUDA(cudaMemcpyAsync(g->d_acc + 12, h, 24, cudaMemcpyHostToDevice, g->stream));
  BBF_TRY(allreduce_u64(g, g->d_acc + 12, 2));
  BBF_TRY(allreduce_u64(g, g->d_acc + 14, 1, ncclMax));
  // per-vertex sums: only the rows of degree >= 2 (a prefix of each side's rank-space rows,
  // [0, L4)); a vertex of degree <= 1 lies on no butterfly, so its row is 0 on every rank
  if (per_vertex) {
    BBF_TRY(allreduce_u64(g, (unsigned long long*)g->pv, 2ull * g->L4[0]));
    BBF_TRY(allreduce_u64(g, (unsigned long long*)g->pv + 2ull * g->n_u, 2ull * g->L4[1]));
  }
  BBF_CUDA(cudaMemcpyAsync(h, g->d_acc + 12, 24, cudaMemcpyDeviceToHost, g->stream));
  BBF_TRY(sync_stream(g));
  if (h[2] != BBF_OK) {
    set_error(local != BBF_OK ? msg : "a peer rank failed (status " + std::to_string(h[2]) + ")");
    return (bbf_status)h[2];
  }
  BN[0] = h[0];
  BN[1] = h[1];
  return BBF_OK;
}

// two CUDA events, destroyed on every return path
struct EventPair {
  cudaEvent_t a = nullptr, b = nullptr;
  EventPair() { cudaEventCreate(&a); cudaEventCreate(&b); }
  ~EventPair() { if (a) cudaEventDestroy(a); if (b) cudaEventDestroy(b); }
  EventPair(const EventPair&) = delete;
  EventPair& operator=(const EventPair&) = delete;
};

}  // namespace
// the (rank, nranks) shard this process counts: the communicator's, or the BBF_FAKE_WORLD test
// hook's ("r/N": count rank r's shard of an N-rank job on this single GPU, no collective)
void shard_of(const bbf_graph* g, int* rank, int* nranks) {
  *rank = g->comm ? g->comm->rank : 0;
  *nranks = g->comm ? g->comm->nranks : 1;
  if (!g->comm && getenv("BBF_FAKE_WORLD")) {
    int r = 0, N = 1;
    if (sscanf(getenv("BBF_FAKE_WORLD"), "%d/%d", &r, &N) == 2 && N >= 1 && r >= 0 && r < N) {
      *rank = r;
      *nranks = N;
    }
  }
}
namespace {

bbf_status check_overflow(bbf_graph* g) {
  if (g->ws_bound >= 18446744073709551615.0L) {
    set_error("counts could exceed 2^64-1 (bound (maxdeg-1)/2 * W_S)");
    return BBF_EOVERFLOW;
  }
  return BBF_OK;
}

bbf_status ensure_plan_g(bbf_graph* g) {
  BBF_TRY(ensure_adj(g));
  int rank, nranks;
  shard_of(g, &rank, &nranks);
  if (g->plan_g.valid && g->plan_g.nranks != nranks) free_plan(&g->plan_g, g->stream);  // units sized per N
  if (!g->plan_g.valid) BBF_TRY(make_plan(g, 0, &g->plan_g));
  return BBF_OK;
}

// the paper's wedge count W_G of the graph (the "wedges" of wedges/s, reading R20)
bbf_status wedges_g(bbf_graph* g, unsigned long long* w) {
  if (g->wg_valid) { *w = g->W_G; return BBF_OK; }
  BBF_TRY(ensure_plan_g(g));
  *w = g->plan_g.W_full;
  return BBF_OK;
}

// dense (tcgen05) vs sparse dispatch
bool use_dense(bbf_graph* g, uint32_t flags, bool per_vertex) {
  if (flags & BBF_FORCE_SPARSE) return false;
  if (flags & BBF_FORCE_DENSE) return true;
  if (getenv("BBF_HYBRID_CORE")) return false;  // test hook: a forced hybrid core (hybrid.cu)
  return dense_preferred(g, per_vertex);
}

bbf_status do_count_local(bbf_graph* g, bool per_vertex, uint32_t flags, int rank, int nranks,
                          unsigned long long* BN) {
  if (per_vertex) {
    BBF_CUDA(cudaMemsetAsync(g->pv, 0, 16ull * g->n, g->stream));
    BBF_CUDA(cudaMemsetAsync(g->pe, 0, 8ull * g->n, g->stream));
    BBF_CUDA(cudaMemsetAsync(g->pm, 0, 8ull * g->n, g->stream));
  }
  g->last_nc[0] = g->last_nc[1] = 0;
  // a dense core, if the graph has one worth it (hybrid.cu); graphs loaded as dense candidates
  // (W_G known at load) first get the whole-graph dense check
  const bool dense_first = (g->dense_cand && !getenv("BBF_HYBRID_CORE")) || (flags & BBF_FORCE_DENSE);
  if (!dense_first && !(flags & BBF_FORCE_SPARSE)) {
    BBF_TRY(ensure_adj(g));
    uint32_t nc[2];
    hybrid_choose(g, per_vertex, nc);
    if (nc[0] && nc[1]) {
      g->last_nc[0] = nc[0];
      g->last_nc[1] = nc[1];
      BBF_TRY(run_hybrid(g, nc, per_vertex, rank, nranks, BN));
      g->W_G = g->plan_h.W_full;  // the hybrid plan's unclamped count is the paper's W_G
      g->wg_valid = true;
      return BBF_OK;
    }
  }
  if (!g->wg_valid) BBF_TRY(ensure_plan_g(g));  // W_G of the graph (and the sparse plan)
  if (use_dense(g, flags, per_vertex)) {
    if (!dense_supported(g)) {
      set_error("BBF_FORCE_DENSE: graph not supported by the dense int8 path");
      return BBF_EINVAL;
    }
    return run_dense(g, per_vertex, rank, nranks, BN);
  }
  BBF_TRY(ensure_plan_g(g));
  return run_sparse(g, &g->plan_g, per_vertex, rank, nranks, BN);
}

bbf_status do_count(bbf_graph* g, bool per_vertex, uint32_t flags, unsigned long long* BN,
                    float* ms) {
  BBF_TRY(check_overflow(g));  // a property of the graph: identical on every rank
  int rank, nranks;
  shard_of(g, &rank, &nranks);
  EventPair ev;
  cudaEventRecord(ev.a, g->stream);
  const bbf_status local = do_count_local(g, per_vertex, flags, rank, nranks, BN);
  BBF_TRY(finish_collective(g, local, per_vertex, BN));
  cudaEventRecord(ev.b, g->stream);
  BBF_TRY(sync_stream(g));
  cudaEventElapsedTime(ms, ev.a, ev.b);
  return BBF_OK;
}

}  // namespace
}  // namespace bbf

using namespace bbf;

extern "C" {

int bbf_abi_version(void) { return BBF_ABI_VERSION; }

const char* bbf_last_error(void) { return g_last_error.c_str(); }

bbf_status bbf_nccl_unique_id(uint8_t id[128]) {
  if (!id) { set_error("null id"); return BBF_EINVAL; }
  if (!nccl().ok) { set_error("libnccl.so.2 not loadable"); return BBF_ENCCL; }
  ncclUniqueId u;
  BBF_TRY(nccl_status(nccl().GetUniqueId(&u), "ncclGetUniqueId"));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(id, &u, 128);
  return BBF_OK;
}

bbf_status bbf_comm_init(const uint8_t id[128], int nranks, int rank, int device, bbf_comm** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) { set_error("bad comm args"); return BBF_EINVAL; }
  if (!device_ok(device, nullptr)) { set_error("no sm_100 device"); return BBF_ECUDA; }
  if (!nccl().ok) { set_error("libnccl.so.2 not loadable"); return BBF_ENCCL; }
  BBF_CUDA(cudaSetDevice(device));
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclComm_t c;
  BBF_TRY(nccl_status(nccl().CommInitRank(&c, nranks, u, rank), "ncclCommInitRank"));
  bbf_comm* cm = new bbf_comm{(void*)c, nranks, rank, device};
  *out = cm;
  return BBF_OK;
}

bbf_status bbf_comm_free(bbf_comm* comm) {
  if (!comm) return BBF_OK;
  if (comm->nccl && nccl().ok) nccl().CommDestroy((ncclComm_t)comm->nccl);
  delete comm;
  return BBF_OK;
}

namespace {
// per-device library streams for asynchronous host<->device copies (uploads, async outputs)
cudaStream_t copy_stream(int device, int which) {
  static std::once_flag once[64][2];
  static cudaStream_t st[64][2];
  if (device < 0 || device >= 64) return nullptr;
  std::call_once(once[device][which], [device, which] {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaStreamCreateWithFlags(&st[device][which], cudaStreamNonBlocking);
    cudaSetDevice(prev);
  });
  return st[device][which];
}

bbf_status load_impl(uint32_t n_u, uint32_t n_v, const uint64_t* row_ptr, const uint32_t* col,
                     const uint8_t* sign, uint32_t flags, int device, void* cuda_stream, bbf_comm* comm,
                     bbf_graph** out, const uint64_t* known_nnz);
}  // namespace

struct bbf_upload {
  int device;
  uint32_t n_u, n_v;
  uint64_t nnz;
  uint64_t* rp;
  uint32_t* col;
  uint8_t* sg;
  cudaEvent_t done;
};

bbf_status bbf_upload_csr(uint32_t n_u, uint32_t n_v, const uint64_t* row_ptr, const uint32_t* col,
                          const uint8_t* sign, int device, bbf_upload** out) {
  if (!out || !row_ptr) { set_error("null pointer"); return BBF_EINVAL; }
  *out = nullptr;
  if ((uint64_t)n_u + n_v >= (1ull << 31)) { set_error("n_u + n_v >= 2^31"); return BBF_ERANGE; }
  const uint64_t nnz = row_ptr[n_u];
  if (nnz >= (1ull << 31)) { set_error("nnz >= 2^31"); return BBF_ERANGE; }
  if (nnz && (!col || !sign)) { set_error("null col/sign"); return BBF_EINVAL; }
  if (!device_ok(device, nullptr)) { set_error("no usable sm_100 CUDA device"); return BBF_ECUDA; }
  BBF_CUDA(cudaSetDevice(device));
  keep_pool(device);
  cudaStream_t cs = copy_stream(device, 0);
  bbf_upload* u = new bbf_upload();
  std::memset(u, 0, sizeof(*u));
  u->device = device; u->n_u = n_u; u->n_v = n_v; u->nnz = nnz;
  // blocks that need no wait on other streams: the copy must not queue behind the current count
  cudaError_t e = dmalloc_nowait(&u->rp, 8ull * (n_u + 1), cs);
  if (e == cudaSuccess) e = dmalloc_nowait(&u->col, 4ull * (nnz + 1), cs);
  if (e == cudaSuccess) e = dmalloc_nowait(&u->sg, nnz + 1, cs);
  if (e == cudaSuccess) e = cudaMemcpyAsync(u->rp, row_ptr, 8ull * (n_u + 1), cudaMemcpyHostToDevice, cs);
  if (e == cudaSuccess && nnz) e = cudaMemcpyAsync(u->col, col, 4ull * nnz, cudaMemcpyHostToDevice, cs);
  if (e == cudaSuccess && nnz) e = cudaMemcpyAsync(u->sg, sign, nnz, cudaMemcpyHostToDevice, cs);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&u->done, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(u->done, cs);
  if (e != cudaSuccess) {
    if (u->rp) dfree(u->rp, cs);
    if (u->col) dfree(u->col, cs);
    if (u->sg) dfree(u->sg, cs);
    delete u;
    return cuda_status(e, "upload");
  }
  *out = u;
  return BBF_OK;
}

bbf_status bbf_upload_free(bbf_upload* u) {
  if (!u) return BBF_OK;
  cudaSetDevice(u->device);
  cudaStream_t cs = copy_stream(u->device, 0);
  dfree(u->rp, cs);
  dfree(u->col, cs);
  dfree(u->sg, cs);
  if (u->done) cudaEventDestroy(u->done);
  delete u;
  return BBF_OK;
}

bbf_status bbf_graph_load_upload(bbf_upload* up, uint32_t flags, void* cuda_stream, bbf_comm* comm,
                                 bbf_graph** out) {
  if (!up || !out) { set_error("null pointer"); return BBF_EINVAL; }
  *out = nullptr;
  if (flags & BBF_PTR_DEVICE) { set_error("BBF_PTR_DEVICE is implied by an upload"); return BBF_EINVAL; }
  BBF_CUDA(cudaSetDevice(up->device));
  // the build waits for the copies on the device, not on the host
  if (cuda_stream) BBF_CUDA(cudaStreamWaitEvent((cudaStream_t)cuda_stream, up->done, 0));
  else BBF_CUDA(cudaEventSynchronize(up->done));
  const uint64_t nnz = up->nnz;
  bbf_status s = load_impl(up->n_u, up->n_v, up->rp, up->col, up->sg, flags | BBF_PTR_DEVICE, up->device,
                           cuda_stream, comm, out, &nnz);
  bbf_upload_free(up);  // stream-ordered: the device buffers are reused only after the build
  return s;
}

bbf_status bbf_device_sync(int device) {
  BBF_CUDA(cudaSetDevice(device));
  BBF_CUDA(cudaDeviceSynchronize());
  return BBF_OK;
}

bbf_status bbf_graph_load_csr(uint32_t n_u, uint32_t n_v, const uint64_t* row_ptr, const uint32_t* col,
                              const uint8_t* sign, uint32_t flags, int device, void* cuda_stream,
                              bbf_comm* comm, bbf_graph** out) {
  return load_impl(n_u, n_v, row_ptr, col, sign, flags, device, cuda_stream, comm, out, nullptr);
}

namespace {
bbf_status load_impl(uint32_t n_u, uint32_t n_v, const uint64_t* row_ptr, const uint32_t* col,
                     const uint8_t* sign, uint32_t flags, int device, void* cuda_stream, bbf_comm* comm,
                     bbf_graph** out, const uint64_t* known_nnz) {
  if (!out || !row_ptr) { set_error("null pointer"); return BBF_EINVAL; }
  *out = nullptr;
  if (flags & ~(uint32_t)(BBF_PTR_DEVICE | BBF_POSITIVE_ONLY | BBF_FORCE_SPARSE | BBF_FORCE_DENSE)) {
    set_error("unknown flags");
    return BBF_EINVAL;
  }
  if ((flags & BBF_FORCE_SPARSE) && (flags & BBF_FORCE_DENSE)) {
    set_error("BBF_FORCE_SPARSE and BBF_FORCE_DENSE are exclusive");
    return BBF_EINVAL;
  }
  if ((uint64_t)n_u + n_v >= (1ull << 31)) { set_error("n_u + n_v >= 2^31"); return BBF_ERANGE; }
  int num_sms = 0;
  if (!device_ok(device, &num_sms)) { set_error("no usable sm_100 CUDA device"); return BBF_ECUDA; }
  BBF_CUDA(cudaSetDevice(device));
  const bool dptr = flags & BBF_PTR_DEVICE;
  uint64_t nnz = 0;
  if (known_nnz) {
    nnz = *known_nnz;
  } else if (dptr) {
    // ordered after the caller's work on its stream (a plain cudaMemcpy would run on the legacy
    // default stream, which does not wait for non-blocking streams)
    if (cuda_stream) {
      BBF_CUDA(rb_add(&nnz, row_ptr + n_u, 8, (cudaStream_t)cuda_stream));
      BBF_CUDA(rb_sync((cudaStream_t)cuda_stream));
    } else {
      BBF_CUDA(cudaDeviceSynchronize());
      BBF_CUDA(cudaMemcpy(&nnz, row_ptr + n_u, 8, cudaMemcpyDeviceToHost));
    }
  } else {
    nnz = row_ptr[n_u];
  }
  if (nnz >= (1ull << 31)) { set_error("nnz >= 2^31"); return BBF_ERANGE; }
  if (nnz && (!col || !sign)) { set_error("null col/sign"); return BBF_EINVAL; }
  bbf_graph* g = new bbf_graph();
  std::memset(g, 0, sizeof(*g));
  g->device = device;
  g->num_sms = num_sms;
  g->load_flags = flags & (uint32_t)(BBF_FORCE_SPARSE | BBF_FORCE_DENSE);
  g->positive_only = flags & BBF_POSITIVE_ONLY;
  g->comm = comm;
  g->n_u = n_u; g->n_v = n_v; g->n = n_u + n_v; g->nnz = nnz;
  if (cuda_stream) {
    g->stream = (cudaStream_t)cuda_stream;
  } else {
    cudaError_t e = cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) { delete g; return cuda_status(e, "cudaStreamCreate"); }
    g->own_stream = true;
  }
  bbf_status s = BBF_OK;
  keep_pool(device);
  cudaError_t e = dmalloc(&g->d_acc, 32 * sizeof(unsigned long long), g->stream);
  if (e == cudaSuccess) e = dmalloc(&g->pv, 16ull * (g->n + 1), g->stream);
  if (e == cudaSuccess) e = dmalloc(&g->pe, 8ull * (g->n + 1), g->stream);
  if (e == cudaSuccess) e = dmalloc(&g->pm, 8ull * (g->n + 1), g->stream);
  if (e != cudaSuccess) s = cuda_status(e, "cudaMalloc");
  if (s == BBF_OK) s = build_graph(g, row_ptr, col, sign, dptr);
  if (s == BBF_OK) {
    e = cudaStreamSynchronize(g->stream);
    if (e != cudaSuccess) s = cuda_status(e, "graph build");
  }
  if (s != BBF_OK) {
    std::string msg = g_last_error;
    bbf_graph_free(g);
    g_last_error = msg;
    return s;
  }
  *out = g;
  return BBF_OK;
}
}  // namespace

bbf_status bbf_graph_free(bbf_graph* g) {
  if (!g) return BBF_OK;
  cudaSetDevice(g->device);
  free_hybrid(g);
  free_plan(&g->plan_g, g->stream);
  free_plan(&g->plan_s[0], g->stream);
  free_plan(&g->plan_s[1], g->stream);
  free_plan(&g->plan_e[0], g->stream);
  free_plan(&g->plan_e[1], g->stream);
  void* ptrs[] = {g->off, g->adj, g->erow, g->rev, g->rlast, g->mid, g->end1, g->inv, g->degs, g->degpre, g->scratch, g->d_acc, g->pv, g->pe, g->pm,
                  g->adjc, g->runid, g->runs, g->skey, g->lr, g->in_rp, g->in_col, g->in_sg,
                  g->dA[0], g->dA[1], g->dS[0], g->dS[1], g->dA4[0], g->dA4[1], g->dS4[0], g->dS4[1]};
  for (void* p : ptrs)
    if (p) dfree(p, g->stream);
  cudaStreamSynchronize(g->stream);
  if (g->own_stream) cudaStreamDestroy(g->stream);
  delete g;
  return BBF_OK;
}

bbf_status bbf_count_global(bbf_graph* g, bbf_counts* out) {
  if (!g || !out) { set_error("null pointer"); return BBF_EINVAL; }
  BBF_CUDA(cudaSetDevice(g->device));
  unsigned long long BN[2] = {0, 0};
  float ms = 0;
  BBF_TRY(do_count(g, false, g->load_flags, BN, &ms));
  unsigned long long wg = 0;
  BBF_TRY(wedges_g(g, &wg));
  out->balanced = BN[0];
  out->unbalanced = BN[1];
  out->total = BN[0] + BN[1];
  out->wedges_G = wg;
  out->ms_count = ms;
  return BBF_OK;
}

bbf_status bbf_count_global_base(bbf_graph* g, bbf_counts* out) {
  if (!g || !out) { set_error("null pointer"); return BBF_EINVAL; }
  BBF_CUDA(cudaSetDevice(g->device));
  BBF_TRY(check_overflow(g));
  int rank, nranks;
  shard_of(g, &rank, &nranks);
  EventPair ev;
  cudaEventRecord(ev.a, g->stream);
  unsigned long long BN[2] = {0, 0};
  // every rank enters the collective whatever its local status (a table-limit or allocation
  // failure on one rank is returned by all of them, none is left blocked in the all-reduce)
  bbf_status local = ensure_plan_g(g);
  if (local == BBF_OK) local = run_base(g, &g->plan_g, rank, nranks, BN);
  BBF_TRY(finish_collective(g, local, false, BN));
  cudaEventRecord(ev.b, g->stream);
  BBF_TRY(sync_stream(g));
  float ms = 0;
  cudaEventElapsedTime(&ms, ev.a, ev.b);
  unsigned long long wg = 0;
  BBF_TRY(wedges_g(g, &wg));
  out->balanced = BN[0];
  out->unbalanced = BN[1];
  out->total = BN[0] + BN[1];
  out->wedges_G = wg;
  out->ms_count = ms;
  return BBF_OK;
}

bbf_status bbf_count_per_vertex(bbf_graph* g, uint64_t* bal_u, uint64_t* unb_u, uint64_t* bal_v,
                                uint64_t* unb_v, uint32_t flags, bbf_counts* totals) {
  if (!g) { set_error("null graph"); return BBF_EINVAL; }
  if (flags & ~(uint32_t)(BBF_PTR_DEVICE | BBF_FORCE_SPARSE | BBF_FORCE_DENSE | BBF_OUTPUT_ASYNC)) {
    set_error("unknown flags");
    return BBF_EINVAL;
  }
  BBF_CUDA(cudaSetDevice(g->device));
  unsigned long long BN[2] = {0, 0};
  float ms = 0;
  if ((flags & (BBF_FORCE_SPARSE | BBF_FORCE_DENSE)) == 0) flags |= g->load_flags;
  BBF_TRY(do_count(g, true, flags, BN, &ms));
  cudaStream_t st = g->stream;
  const bool dptr = flags & BBF_PTR_DEVICE;
  // S9: rank space -> input ids, straight into device outputs or via one staging buffer
  unsigned long long* stage = nullptr;
  uint64_t* outs[4] = {bal_u, unb_u, bal_v, unb_v};
  if (!dptr && (bal_u || unb_u || bal_v || unb_v)) BBF_CUDA(dmalloc(&stage, 16ull * (g->n + 1), st));
  for (int side = 0; side < 2; ++side) {
    uint32_t cnt = side ? g->n_v : g->n_u, row0 = side ? g->n_u : 0;
    uint64_t* ob = outs[2 * side];
    uint64_t* on = outs[2 * side + 1];
    if (!cnt || (!ob && !on)) continue;
    unsigned long long* db = dptr ? (unsigned long long*)ob : (ob ? stage + 2ull * row0 : nullptr);
    unsigned long long* dn = dptr ? (unsigned long long*)on : (on ? stage + 2ull * row0 + cnt : nullptr);
    k_scatter_pv<<<(cnt + 255) / 256, 256, 0, st>>>((const unsigned long long*)g->pv, g->inv, row0, cnt,
                                                   g->n, db, dn);
    g->launches++;
  }
  // host outputs: one D2H per array, on the graph's stream, or with BBF_OUTPUT_ASYNC on the
  // library's download stream (ordered after the scatter by an event; the call returns without
  // waiting, bbf_device_sync completes it) so the copy overlaps the caller's next work
  cudaStream_t dst = st;
  const bool async_out = !dptr && stage && (flags & BBF_OUTPUT_ASYNC);
  if (async_out) {
    dst = copy_stream(g->device, 1);
    cudaEvent_t ev;
    BBF_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    BBF_CUDA(cudaEventRecord(ev, st));
    BBF_CUDA(cudaStreamWaitEvent(dst, ev, 0));
    cudaEventDestroy(ev);  // released once the recorded work completes
  }
  if (!dptr) {
    for (int side = 0; side < 2; ++side) {
      uint32_t cnt = side ? g->n_v : g->n_u, row0 = side ? g->n_u : 0;
      uint64_t* ob = outs[2 * side];
      uint64_t* on = outs[2 * side + 1];
      if (!cnt) continue;
      if (ob) BBF_CUDA(cudaMemcpyAsync(ob, stage + 2ull * row0, 8ull * cnt, cudaMemcpyDeviceToHost, dst));
      if (on) BBF_CUDA(cudaMemcpyAsync(on, stage + 2ull * row0 + cnt, 8ull * cnt, cudaMemcpyDeviceToHost, dst));
    }
  }
  if (stage) dfree(stage, dst);
  BBF_CUDA(cudaStreamSynchronize(st));
  if (totals) {
    unsigned long long wg = 0;
    BBF_TRY(wedges_g(g, &wg));
    totals->balanced = BN[0];
    totals->unbalanced = BN[1];
    totals->total = BN[0] + BN[1];
    totals->wedges_G = wg;
    totals->ms_count = ms;
  }
  return BBF_OK;
}

bbf_status bbf_count_pairs_topk(bbf_graph* g, int side, uint32_t k, bbf_pair* out, uint32_t* n_out,
                                uint32_t flags) {
  if (!g || !out || !n_out) { set_error("null pointer"); return BBF_EINVAL; }
  if (k == 0) { set_error("k == 0"); return BBF_EINVAL; }
  if (side != BBF_SIDE_U && side != BBF_SIDE_V) { set_error("bad side"); return BBF_EINVAL; }
  if (flags & ~(uint32_t)(BBF_FORCE_SPARSE)) { set_error("unsupported flags for topk"); return BBF_EINVAL; }
  BBF_CUDA(cudaSetDevice(g->device));
  BBF_TRY(check_overflow(g));
  int rank, nranks;
  shard_of(g, &rank, &nranks);
  *n_out = 0;
  bbf_status local = ensure_adj(g);
  if (local == BBF_OK) local = run_pairs_topk(g, side, k, out, n_out, rank, nranks);
  if (!multi_rank(g)) return local;
  // S12: all-gather of every rank's local top-k (k slots of (balanced, unbalanced, a << 32 | b),
  // empty slots zero, plus the rank's status) and a deterministic merge, identical on all ranks
  const int N = g->comm->nranks;
  const size_t rec = 3ull * k + 1;
  std::vector<unsigned long long> mine(rec, 0ull), all(rec * N, 0ull);
  if (local == BBF_OK)
    for (uint32_t i = 0; i < *n_out; ++i) {
      mine[3 * i] = out[i].balanced;
      mine[3 * i + 1] = out[i].unbalanced;
      mine[3 * i + 2] = ((unsigned long long)out[i].a << 32) | out[i].b;
    }
  mine[3ull * k] = (unsigned long long)local;
  unsigned long long* d = nullptr;
  BBF_CUDA(dmalloc(&d, 8ull * rec * (N + 1), g->stream));
  BBF_CUDA(cudaMemcpyAsync(d, mine.data(), 8ull * rec, cudaMemcpyHostToDevice, g->stream));
  bbf_status s = nccl_status(nccl().AllGather(d, d + rec, rec, ncclUint64, (ncclComm_t)g->comm->nccl, g->stream),
                             "ncclAllGather");
  if (s == BBF_OK) {
    cudaError_t e = cudaMemcpyAsync(all.data(), d + rec, 8ull * rec * N, cudaMemcpyDeviceToHost, g->stream);
    if (e != cudaSuccess) s = cuda_status(e, "cudaMemcpyAsync");
  }
  if (s == BBF_OK) s = sync_stream(g);
  dfree(d, g->stream);
  if (s != BBF_OK) return s;
  unsigned long long worst = 0;
  std::vector<bbf_pair> cand;
  for (int r = 0; r < N; ++r) {
    const unsigned long long* q = all.data() + rec * r;
    worst = std::max(worst, q[3ull * k]);
    for (uint32_t i = 0; i < k; ++i)
      if (q[3 * i])  // balanced > 0: a listed pair (reading R11 lists only those)
        cand.push_back(bbf_pair{(uint32_t)(q[3 * i + 2] >> 32), (uint32_t)(q[3 * i + 2] & 0xffffffffu), q[3 * i],
                                q[3 * i + 1]});
  }
  if (worst != BBF_OK) {
    if (local == BBF_OK) set_error("a peer rank failed (status " + std::to_string(worst) + ")");
    *n_out = 0;
    return (bbf_status)worst;
  }
  std::sort(cand.begin(), cand.end(), [](const bbf_pair& x, const bbf_pair& y) {
    if (x.balanced != y.balanced) return x.balanced > y.balanced;
    if (x.a != y.a) return x.a < y.a;
    return x.b < y.b;
  });
  *n_out = (uint32_t)std::min<size_t>(k, cand.size());
  for (uint32_t i = 0; i < *n_out; ++i) out[i] = cand[i];
  return BBF_OK;
}

bbf_status bbf_count_per_edge(bbf_graph* g, const uint64_t* row_ptr, const uint32_t* col, uint64_t* bal,
                              uint64_t* unb, uint32_t flags, bbf_counts* totals) {
  if (!g || !row_ptr) { set_error("null pointer"); return BBF_EINVAL; }
  if (flags & ~(uint32_t)BBF_PTR_DEVICE) { set_error("unknown flags"); return BBF_EINVAL; }
  BBF_CUDA(cudaSetDevice(g->device));
  BBF_TRY(check_overflow(g));
  cudaStream_t st = g->stream;
  const bool dptr = flags & BBF_PTR_DEVICE;
  const uint64_t nnz = g->nnz, m = 2 * nnz;
  if (nnz && !col) { set_error("null col"); return BBF_EINVAL; }
  {  // the CSR must have the graph's edge count (its edges are checked against the graph below)
    uint64_t c_nnz = 0;
    if (dptr) {
      BBF_CUDA(rb_add(&c_nnz, row_ptr + g->n_u, 8, st));
      BBF_CUDA(rb_sync(st));
    } else {
      c_nnz = row_ptr[g->n_u];
    }
    if (c_nnz != nnz) { set_error("per-edge counts: the CSR passed is not the loaded graph's"); return BBF_EINVAL; }
  }
  int rank, nranks;
  shard_of(g, &rank, &nranks);
  EventPair ev;
  cudaEventRecord(ev.a, st);
  // the edge slots: one (balanced, unbalanced) pair per rank-space adjacency entry of the U rows
  unsigned long long* d_edge = nullptr;
  BBF_CUDA(dmalloc(&d_edge, 16ull * (m + 1), st));
  BBF_CUDA(cudaMemsetAsync(d_edge, 0, 16ull * (m + 1), st));
  unsigned long long BN[2] = {0, 0}, BN2[2] = {0, 0};
  // route S(U) with the ends after the start, then with the ends before it: every U-pair (u, w)
  // is seen from both u and w, so each start->middle edge collects the shares of all its pairs
  // (reading R24); the hub kernel runs every start (its records carry the start->middle entry)
  bbf_status local = ensure_adj(g);
  for (int k = 0; k < 2 && local == BBF_OK; ++k) {
    Plan* p = &g->plan_e[k];
    if (p->valid && p->nranks != nranks) free_plan(p, st);
    if (!p->valid) local = make_plan(g, k == 0 ? 1 : 3, p, false);
    if (local == BBF_OK) {
      cudaError_t e = cudaMemsetAsync(g->pv, 0, 16ull * g->n, st);
      if (e != cudaSuccess) local = cuda_status(e, "memset");
    }
    if (local == BBF_OK)
      local = run_sparse_impl(g, p, true, false, rank, nranks, k == 0 ? BN : BN2, nullptr, nullptr, nullptr, 0, nullptr,
                              1ull, d_edge);
  }
  if (multi_rank(g)) {  // every rank enters: status max-reduce, (B, N), the edge slots
    BBF_TRY(finish_collective(g, local, false, BN));
    BBF_TRY(allreduce_u64(g, d_edge, 2 * m));
  } else if (local != BBF_OK) {
    dfree(d_edge, st);
    return local;
  }
  // the caller's CSR order
  const uint64_t* d_rp = row_ptr;
  const uint32_t* d_col = col;
  uint64_t* stage_rp = nullptr;
  uint32_t* stage_col = nullptr;
  if (!dptr) {
    BBF_CUDA(dmalloc(&stage_rp, 8ull * (g->n_u + 1), st));
    BBF_CUDA(dmalloc(&stage_col, 4ull * (nnz + 1), st));
    BBF_CUDA(cudaMemcpyAsync(stage_rp, row_ptr, 8ull * (g->n_u + 1), cudaMemcpyHostToDevice, st));
    if (nnz) BBF_CUDA(cudaMemcpyAsync(stage_col, col, 4ull * nnz, cudaMemcpyHostToDevice, st));
    d_rp = stage_rp;
    d_col = stage_col;
  }
  unsigned long long *ob = nullptr, *on = nullptr;
  if (dptr) {
    ob = (unsigned long long*)bal;
    on = (unsigned long long*)unb;
  } else {
    BBF_CUDA(dmalloc(&ob, 16ull * (nnz + 1), st));
    on = ob + nnz;
  }
  uint32_t* d_err;
  BBF_CUDA(dmalloc(&d_err, 4, st));
  BBF_CUDA(cudaMemsetAsync(d_err, 0, 4, st));
  if (nnz && g->n_u) {
    k_edge_out<<<(unsigned)std::min<uint64_t>((nnz + 255) / 256, 148ull * 64), 256, 0, st>>>(
        g->n_u, g->n_v, d_rp, d_col, nnz, g->lr, g->off, g->adj, d_edge, (dptr && !bal) ? nullptr : ob,
        (dptr && !unb) ? nullptr : on, d_err);
    g->launches++;
  }
  uint32_t h_err = 0;
  BBF_CUDA(cudaMemcpyAsync(&h_err, d_err, 4, cudaMemcpyDeviceToHost, st));
  if (!dptr && nnz) {
    if (bal) BBF_CUDA(cudaMemcpyAsync(bal, ob, 8ull * nnz, cudaMemcpyDeviceToHost, st));
    if (unb) BBF_CUDA(cudaMemcpyAsync(unb, on, 8ull * nnz, cudaMemcpyDeviceToHost, st));
  }
  cudaEventRecord(ev.b, st);
  BBF_TRY(sync_stream(g));
  for (void* q : {(void*)d_edge, (void*)stage_rp, (void*)stage_col, (void*)d_err}) if (q) dfree(q, st);
  if (!dptr) dfree(ob, st);
  if (h_err) { set_error("per-edge counts: the CSR passed is not the loaded graph's"); return BBF_EINVAL; }
  if (totals) {
    unsigned long long wg = 0;
    BBF_TRY(wedges_g(g, &wg));
    totals->balanced = BN[0];
    totals->unbalanced = BN[1];
    totals->total = BN[0] + BN[1];
    totals->wedges_G = wg;
    cudaEventElapsedTime(&totals->ms_count, ev.a, ev.b);
  }
  return BBF_OK;
}

bbf_status bbf_topk_vertices(bbf_graph* g, int side, int metric, uint32_t k, uint32_t* ids,
                             uint64_t* scores, uint32_t* n_out) {
  if (!g || !ids || !scores || !n_out) { set_error("null pointer"); return BBF_EINVAL; }
  if (k == 0) { set_error("k == 0"); return BBF_EINVAL; }
  if (side != BBF_SIDE_U && side != BBF_SIDE_V) { set_error("bad side"); return BBF_EINVAL; }
  if (metric != BBF_METRIC_BALANCED && metric != BBF_METRIC_DEGREE) { set_error("bad metric"); return BBF_EINVAL; }
  BBF_CUDA(cudaSetDevice(g->device));
  cudaStream_t st = g->stream;
  const uint32_t cnt = side ? g->n_v : g->n_u, row0 = side ? g->n_u : 0;
  *n_out = 0;
  if (cnt == 0) return BBF_OK;
  if (metric == BBF_METRIC_BALANCED) {
    unsigned long long BN[2];
    float ms;
    BBF_TRY(do_count(g, true, g->load_flags, BN, &ms));
  }
  unsigned long long *sc, *sc2;
  uint32_t *id, *id2;
  BBF_CUDA(dmalloc(&sc, 8ull * cnt, st));
  BBF_CUDA(dmalloc(&sc2, 8ull * cnt, st));
  BBF_CUDA(dmalloc(&id, 4ull * cnt, st));
  BBF_CUDA(dmalloc(&id2, 4ull * cnt, st));
  k_rank_scores<<<(cnt + 255) / 256, 256, 0, st>>>((const unsigned long long*)g->pv, g->degs, g->inv, row0, cnt,
                                                   metric == BBF_METRIC_DEGREE, sc, id);
  g->launches++;
  // one stable radix sort by score descending over ids generated in ascending order
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, sc, sc2, id, id2, (int)cnt, 0, 64, st);
  void* tmp;
  BBF_CUDA(dmalloc(&tmp, tb + 16, st));
  BBF_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp, tb, sc, sc2, id, id2, (int)cnt, 0, 64, st));
  g->launches += 4;
  const uint32_t take = std::min(k, cnt);
  BBF_CUDA(cudaMemcpyAsync(ids, id2, 4ull * take, cudaMemcpyDeviceToHost, st));
  BBF_CUDA(cudaMemcpyAsync(scores, sc2, 8ull * take, cudaMemcpyDeviceToHost, st));
  BBF_CUDA(cudaStreamSynchronize(st));
  for (void* p : {(void*)sc, (void*)sc2, (void*)id, (void*)id2, tmp}) dfree(p, st);
  *n_out = take;
  return BBF_OK;
}

bbf_status bbf_graph_hybrid_core(bbf_graph* g, uint32_t* core_u, uint32_t* core_v) {
  if (!g) { set_error("null graph"); return BBF_EINVAL; }
  if (core_u) *core_u = g->last_nc[0];
  if (core_v) *core_v = g->last_nc[1];
  return BBF_OK;
}

bbf_status bbf_graph_stats(bbf_graph* g, uint64_t* kernel_launches, uint64_t* algo_bytes,
                           double* algo_ops, float* ms_main_kernel) {
  if (!g) { set_error("null graph"); return BBF_EINVAL; }
  if (kernel_launches) *kernel_launches = g->launches;
  if (algo_bytes) *algo_bytes = g->algo_bytes;
  if (algo_ops) *algo_ops = g->algo_ops;
  if (ms_main_kernel) *ms_main_kernel = g->ms_main;
  return BBF_OK;
}

}  // extern "C"
