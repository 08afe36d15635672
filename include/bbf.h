/*
 * bbf.h — C ABI of libbbf.so: exact balanced / unbalanced butterfly counting in a signed
 * bipartite graph on NVIDIA B200 (sm_100a).  Hot path of arXiv 2308.07932
 * (/root/reference/PAPER.md), re-designed for the GPU; see DESIGN.md.
 *
 * Definitions the library computes (all exact, integer):
 *   - signed bipartite graph G = (U, V, E), E ⊆ U x V, one sign per edge (PAPER.md:571,
 *     §Problem Definition); the ABI sign byte is 1 = positive, 0 = negative (PAPER.md:1031,
 *     "weight 1 ... positive");
 *   - butterfly: 4-cycle u_i - v_i - u_j - v_j (Def. Butterfly);
 *   - balanced butterfly: an even number of negative edges (Def. Balanced
 *     butterfly); unbalanced otherwise;
 *   - per same-side pair (z, y): a = #common neighbours c with sigma(z,c) = sigma(y,c)
 *     ("symmetric wedges"), d = #with opposite signs ("asymmetric wedges",
 *     PAPER.md:660-664); balanced(z,y) = C(a,2) + C(d,2) (Lemma 2) and
 *     unbalanced(z,y) = a*d (Theorem proof);
 *   - global counts: every butterfly once (Alg. 2 BB-Bucket);
 *   - per-vertex counts: butterflies containing the vertex (vBBFC);
 *   - top-k pairs: the k same-side pairs with the largest balanced(z,y) > 0 (case study,
 *     PAPER.md:26-27), ordered by balanced desc, then smaller id asc, then larger id asc
 *     (reading R11).
 *
 * Conventions
 *   Ownership: input arrays are borrowed for the duration of the call and copied; a
 *     bbf_graph owns its device memory until bbf_graph_free.  Outputs are caller-allocated,
 *     host memory unless BBF_PTR_DEVICE is passed (then device pointers on the graph's
 *     device, written stream-ordered on the graph's stream).
 *   Synchronisation: calls return after host outputs are written.
 *   Threading: calls on one handle must be serialised; distinct handles are independent.
 *   Collectives: with a bbf_comm, every rank calls the same functions in the same order with
 *     the same graph; each rank counts its shard of the work (work item i on rank i mod N) and
 *     the library all-reduces (NCCL, u64 sum) so every rank receives the full results; top-k
 *     pairs are all-gathered per rank and merged.  Every rank enters the collectives whatever
 *     its local status and the ranks' status codes are max-reduced, so a local failure (an
 *     allocation, a table limit) is returned by every rank instead of blocking the others.
 *     Waits on a communicator poll ncclCommGetAsyncError: an asynchronous NCCL failure returns
 *     BBF_ENCCL and aborts the communicator (free it with bbf_comm_free).
 *   Errors: every function returns a bbf_status; on failure outputs are unspecified, the
 *     message is available from bbf_last_error() (thread-local), and the handle stays valid
 *     except after BBF_ECUDA.  No C++ exception crosses the ABI.
 *   Empty graphs are valid and count zero.  There is no CPU fallback: without a usable
 *     sm_100 device every counting call returns BBF_ECUDA.
 */
#ifndef BBF_H_
#define BBF_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BBF_ABI_VERSION 1

typedef struct bbf_graph bbf_graph; /* opaque; one graph resident on one GPU (one rank)   */
typedef struct bbf_upload bbf_upload; /* opaque; a host CSR being copied to one GPU          */
typedef struct bbf_comm bbf_comm;   /* opaque NCCL communicator                          */

typedef enum {
  BBF_OK = 0,
  BBF_EINVAL = 1,    /* null pointer, sign byte not in {0,1}, k == 0, bad flags/side      */
  BBF_ERANGE = 2,    /* col >= n_v, row_ptr[0] != 0 or not monotone, n or nnz >= 2^31    */
  BBF_EDUP = 3,      /* duplicate (u,v) edge (SPEC.md:56 DuplicateEdge)                   */
  BBF_ENOMEM = 4,    /* device or host allocation failed                                  */
  BBF_ECUDA = 5,     /* CUDA error / no sm_100 device                                     */
  BBF_ENCCL = 6,     /* NCCL error or library built without NCCL                          */
  BBF_EOVERFLOW = 7  /* a count could exceed 2^64-1 ("report, do not wrap")  */
} bbf_status;

enum { BBF_SIDE_U = 0, BBF_SIDE_V = 1 };
enum { BBF_METRIC_BALANCED = 0, BBF_METRIC_DEGREE = 1 };

enum {
  BBF_PTR_DEVICE = 1u << 0,   /* input (load) / output (count) pointers are device pointers */
  BBF_POSITIVE_ONLY = 1u << 1, /* load: keep only the positive edges (case-study analytics,   */
                               /* PAPER.md:15-27 "only formed by the edges with sign 1")       */
  BBF_FORCE_SPARSE = 1u << 2, /* count: use the sparse wedge-aggregation kernels            */
  BBF_FORCE_DENSE = 1u << 3,  /* count: use the dense int8 tensor-core path (tcgen05)       */
  BBF_OUTPUT_ASYNC = 1u << 4  /* bbf_count_per_vertex: host outputs are written by an        */
                              /* asynchronous copy, complete after bbf_device_sync()          */
};

/* Results of one count.  wedges_G is the paper's wedge count for Alg. 2 on this graph
 * (priority-eligible wedges) — the "wedges" of the wedges/s metric,
 * independent of which kernels ran.  ms_count is the device time of the count call. */
typedef struct {
  uint64_t balanced, unbalanced, total, wedges_G;
  float ms_count;
} bbf_counts;

/* One same-side pair (input ids, a < b) and its Lemma-2 counts. */
typedef struct {
  uint32_t a, b;
  uint64_t balanced, unbalanced;
} bbf_pair;

int bbf_abi_version(void);

/* Thread-local message of the last failure on this thread ("" if none). */
const char *bbf_last_error(void);

/* NCCL bootstrap: rank 0 creates the 128-byte id, the caller broadcasts it (e.g. over a
 * torch.distributed process group), every rank calls bbf_comm_init with it. */
bbf_status bbf_nccl_unique_id(uint8_t id[128]);
bbf_status bbf_comm_init(const uint8_t id[128], int nranks, int rank, int device, bbf_comm **out);
bbf_status bbf_comm_free(bbf_comm *comm);

/* Load a signed bipartite graph given as a U-side CSR and build the device representation
 * (degree priority ranks per Def. Vertex Priority PAPER.md:601-609, both-direction adjacency
 * sorted by priority per Alg. 2 line 3 PAPER.md:747, sign bit packed into each column word,
 * and the work plan).
 *   n_u, n_v  : |U|, |V|; n_u + n_v < 2^31.
 *   row_ptr   : n_u+1 entries, row_ptr[0] == 0, non-decreasing, row_ptr[n_u] = nnz < 2^31.
 *   col       : nnz V-side indices (< n_v), any order within a row, no duplicate (u,v).
 *   sign      : nnz bytes, 1 = positive, 0 = negative.
 *   flags     : BBF_PTR_DEVICE if the three arrays are device pointers on `device`;
 *               BBF_POSITIVE_ONLY: the graph is restricted to its positive edges after
 *               validation (every count then describes the positive subgraph, where every
 *               butterfly is balanced; a duplicate pair with a negative copy is not detected);
 *               BBF_FORCE_SPARSE or BBF_FORCE_DENSE (exclusive) fix the path every count on this
 *               handle uses unless the count call passes its own (default: the dispatch rule
 *               of DESIGN.md §6 picks the faster path; both give bit-identical results).
 *   device    : CUDA device ordinal.  cuda_stream: cudaStream_t to order work on (NULL =
 *               the library creates its own stream).  comm: NULL for a single GPU.
 * Errors: BBF_EINVAL, BBF_ERANGE, BBF_EDUP, BBF_ENOMEM, BBF_ECUDA. */
bbf_status bbf_graph_load_csr(uint32_t n_u, uint32_t n_v, const uint64_t *row_ptr,
                              const uint32_t *col, const uint8_t *sign, uint32_t flags,
                              int device, void *cuda_stream, bbf_comm *comm, bbf_graph **out);
bbf_status bbf_graph_free(bbf_graph *g);

/* Pipelined loading (a stream of graphs): bbf_upload_csr starts copying a host CSR (same
 * arguments and checks as bbf_graph_load_csr without flags; pinned host memory gives a truly
 * asynchronous copy) to device buffers on the library's per-device upload stream and returns at
 * once, so the copy of the next graph overlaps the counting of the current one.  The host arrays
 * must stay valid and unmodified until the upload is consumed or freed.  bbf_graph_load_upload
 * builds the graph from it exactly like bbf_graph_load_csr (flags without BBF_PTR_DEVICE; the
 * build stream waits on the copy on the device) and consumes the upload, whatever the status;
 * bbf_upload_free discards an unconsumed one.  Errors: those of bbf_graph_load_csr. */
bbf_status bbf_upload_csr(uint32_t n_u, uint32_t n_v, const uint64_t *row_ptr, const uint32_t *col,
                          const uint8_t *sign, int device, bbf_upload **out);
bbf_status bbf_graph_load_upload(bbf_upload *up, uint32_t flags, void *cuda_stream, bbf_comm *comm,
                                 bbf_graph **out);
bbf_status bbf_upload_free(bbf_upload *up);

/* Waits for all of the library's work on `device`, including the copies of BBF_OUTPUT_ASYNC. */
bbf_status bbf_device_sync(int device);

/* Global balanced / unbalanced counts (each butterfly once; Alg. 2).  out: host.  Path: the
 * load flags' BBF_FORCE_* if any, else the dispatch rule.
 * Limits and errors (also for bbf_count_per_vertex and bbf_count_pairs_topk):
 *   BBF_EINVAL if BBF_FORCE_DENSE was given for a graph the dense path does not support (other
 *     side > 65,536 vertices, or operands > 16 GB);
 *   BBF_ERANGE (at load) if one side needs more than 2^23 - 1 counter words for the sparse hub
 *     kernel's 23-bit counter address: ends (degree >= 2) take degree-zoned (a, d) fields, 8
 *     ends of degree 2-3 per word down to one end of degree >= 256 per word (two words above
 *     65,535), so a side holds at most ~8.4M words (161 windows of 52,224 words) — e.g. 67M ends
 *     of degree <= 3, or 8.4M ends of degree >= 256; (at count) if the hub kernel's window table
 *     (256 windows) would be exceeded, which the address limit already rules out;
 *   BBF_EOVERFLOW if B + N could exceed 2^64 - 1 (host bound, reading R13);
 *   BBF_ENOMEM, BBF_ECUDA, BBF_ENCCL.
 * The dense path's block-scaled FP4 kernels (tcgen05 kind::mxf4) multiply exact +-1/0 e2m1
 * operands with unit scales and accumulate in fp32; they are used only while every partial sum
 * is an integer of magnitude <= 2^13 (rows' max degree <= 8,192; packed-accumulator variant
 * |T + 2048 P| < 2^22 for degree < 2,048), where fp32 — even a reduced-precision tensor-core
 * accumulator — is exact; beyond that the int8 kernels (exact s32) run. */
bbf_status bbf_count_global(bbf_graph *g, bbf_counts *out);

/* The same global counts by Alg. 1 BB-Base, the paper's baseline: per start
 * the middles of every end w are collected in a list H(w) and every pair of a list is checked
 * for balance one by one (cost = the number of butterflies instead of the number of wedges).
 * Kept to reproduce the BB-Base vs BB-Bucket regime; results equal
 * bbf_count_global's.  Sparse path only; starts sharded over the ranks of comm like
 * bbf_count_global, counts all-reduced.  out: host (ms_count = device time of this call).
 * Errors: BBF_EINVAL if a start has more than 8,192 distinct ends (the per-CTA table),
 * BBF_ENOMEM if a start has 2^32 or more wedges (32-bit list offsets; the 8 GiB scratch holds
 * them), BBF_EOVERFLOW, BBF_ECUDA, BBF_ENCCL. */
bbf_status bbf_count_global_base(bbf_graph *g, bbf_counts *out);

/* Per-vertex counts (butterflies containing each vertex; vBBFC semantics),
 * indexed by input ids.  Any of the four arrays may be NULL.  Host arrays unless
 * BBF_PTR_DEVICE.  totals (nullable, host) receives the global counts as well.  With
 * BBF_OUTPUT_ASYNC (host arrays) the call returns once the counts exist on the device and the
 * arrays are filled by a copy on the library's download stream: read them after
 * bbf_device_sync(device); the graph may be freed before that. */
bbf_status bbf_count_per_vertex(bbf_graph *g, uint64_t *bal_u, uint64_t *unb_u, uint64_t *bal_v,
                                uint64_t *unb_v, uint32_t flags, bbf_counts *totals);

/* Top-k same-side pairs by balanced count on `side` (BBF_SIDE_U / BBF_SIDE_V).  out: host
 * array of k slots; *n_out receives min(k, #pairs with balanced > 0).  k >= 1.  With a comm,
 * each rank finds the top-k of its shard of the pairs (every pair lies in exactly one work item)
 * and the ranks' lists are all-gathered and merged (the global top-k is within their union).
 * Errors: BBF_EINVAL (k == 0, side, flags, null pointers), and those of bbf_count_global. */
bbf_status bbf_count_pairs_topk(bbf_graph *g, int side, uint32_t k, bbf_pair *out,
                                uint32_t *n_out, uint32_t flags);

/* Per-edge counts: for every edge e of the graph, the balanced / unbalanced butterflies containing
 * it ("count the number of balanced butterflies containing the edge e = (u,v)";
 * DESIGN.md reading R24).  row_ptr / col: the U-side CSR the graph was loaded from (the same
 * arrays, or any CSR of the same edge set) — its edge order is the output order: bal[i], unb[i]
 * belong to edge (u, col[i]) with row_ptr[u] <= i < row_ptr[u + 1].  Host pointers unless
 * BBF_PTR_DEVICE (then row_ptr, col, bal, unb are device pointers); bal / unb nullable.  totals
 * (nullable, host): global counts.  Each edge's counts are the Lemma-2 middle shares of its V
 * endpoint summed over all U-pairs containing its U endpoint (route S(U) in both directions on the
 * sparse engine's hub kernel), so they satisfy sum_e = 4 (B, N) and, per vertex z, the sum over
 * z's edges = 2 x z's per-vertex count.  With a comm the work is sharded and the slots all-reduced.
 * A graph loaded with BBF_POSITIVE_ONLY holds only the positive edges: pass that edge set's CSR.
 * Errors: BBF_EINVAL (null pointers, flags, a CSR whose edges are not the graph's), those of
 * bbf_count_global. */
bbf_status bbf_count_per_edge(bbf_graph *g, const uint64_t *row_ptr, const uint32_t *col, uint64_t *bal,
                              uint64_t *unb, uint32_t flags, bbf_counts *totals);

/* Top-k vertices of one side (case study, "top-10 actors with most number of
 * positive butterflies / positive edges"): metric BBF_METRIC_BALANCED ranks by
 * the per-vertex balanced count (bbf_count_per_vertex), BBF_METRIC_DEGREE by degree in the loaded
 * graph (with BBF_POSITIVE_ONLY at load: positive degree).  Order: score desc, then input id asc;
 * every vertex of the side is ranked (zero scores included).  ids, scores: host arrays of k
 * slots; *n_out = min(k, |side|).  Errors: BBF_EINVAL (side, metric, k == 0, null pointers). */
bbf_status bbf_topk_vertices(bbf_graph *g, int side, int metric, uint32_t k, uint32_t *ids,
                             uint64_t *scores, uint32_t *n_out);

/* SBESPAR one-shot sparsification estimate of the global balanced count (PAPER.md:1402-1438,
 * §Approximation by Sparsification): for trial t = 0..trials-1, keep each edge of the input CSR
 * independently with probability rho, count the sampled graph exactly (the same path as
 * bbf_count_global) and scale its balanced count by rho^-4 (reading R18: a butterfly survives iff
 * its 4 edges do).  Edge e of the U-side CSR is kept iff rho >= 1 or
 * sm64(sm64(seed + t) ^ e) < floor(rho * 2^64), sm64 = SplitMix64, so the draws are reproducible.
 *   n_u, n_v, row_ptr, col, sign, flags (BBF_PTR_DEVICE, BBF_FORCE_*), device, cuda_stream, comm:
 *     as bbf_graph_load_csr; rho in (0, 1]; trials >= 1.
 *   sampled_balanced / sampled_unbalanced: host u64[trials] (nullable) — exact counts of each
 *     sampled graph; estimates: host double[trials] — sampled balanced count * rho^-4.  (The
 *     mean and spread over trials are the caller's statistics; the Python binding reports them
 *     next to the per-trial estimates.)
 * Errors: BBF_EINVAL (rho, trials, null estimates), those of bbf_graph_load_csr. */
bbf_status bbf_estimate_global(uint32_t n_u, uint32_t n_v, const uint64_t *row_ptr, const uint32_t *col,
                               const uint8_t *sign, uint32_t flags, double rho, uint32_t trials,
                               uint64_t seed, int device, void *cuda_stream, bbf_comm *comm,
                               uint64_t *sampled_balanced, uint64_t *sampled_unbalanced,
                               double *estimates);

/* Introspection for tests and the bench (no effect on results).  kernel_launches: GPU kernels the
 * library launched on this handle since load.  For the last count call's main kernel (the hub
 * wedge-aggregation kernel k_t3 on the sparse path, k_dense_tiles on the dense path):
 * algo_bytes = algorithmic bytes (sparse path; 0 on the dense path), algo_ops = algorithmic
 * int8 tensor ops (dense path; 0 on the sparse path), ms_main_kernel = its device time
 * (DESIGN.md §5).  Any pointer may be NULL. */
bbf_status bbf_graph_stats(bbf_graph *g, uint64_t *kernel_launches, uint64_t *algo_bytes,
                           double *algo_ops, float *ms_main_kernel);

/* Hybrid dense-core dispatch of the last bbf_count_global / bbf_count_per_vertex on this handle
 * (NEXT-3, BASELINE north-star (3)): core_u / core_v = the number of top-priority
 * vertices of U / V (side-local ranks, Def. Vertex Priority PAPER.md:600-609) whose induced
 * subgraph was counted on the tensor cores while the rest of Alg. 2 ran on
 * the sparse engine, the pairs between the two merged per pair before Lemma 2's f
 * (PAPER.md:720-733); 0, 0 = no hybrid (plain sparse or whole-graph dense).  The counts are
 * identical either way.  The dispatch is automatic (estimated engine time of the core's wedges
 * vs the core's tensor time); env BBF_NO_HYBRID disables it, BBF_FORCE_SPARSE / BBF_FORCE_DENSE
 * (at load or count) bypass it.  Requires every degree < 65,536 (pair counts packed 16 | 16)
 * and cores of at most 8,192 per side.  Device memory of a hybrid count: ~2.5 GB for 8,192 x 8,192
 * cores (pair-word matrices nc^2 x 4 B per side, core operands, GEMM temporaries); an allocation
 * failure returns BBF_ENOMEM from the count call.  Errors: BBF_EINVAL on a null handle. */
bbf_status bbf_graph_hybrid_core(bbf_graph *g, uint32_t *core_u, uint32_t *core_v);

#ifdef __cplusplus
}
#endif
#endif /* BBF_H_ */
