/*
 * bbf_oracle.c — plain, slow, obviously-correct CPU oracle for balanced butterfly counting
 * in signed bipartite graphs (arXiv 2308.07932, /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or helper with the CUDA path (paper_2308_07932_b200/csrc), and never
 * reads anything the CUDA path produced.
 *
 * Every routine follows a definition or an algorithm of the paper, in its order:
 *   oracle_brute     Def. Butterfly + Def. Balanced butterfly: enumerate
 *                    all {u_i,u_j} x {v_i,v_j}, keep 4-cycles, classify by the parity of
 *                    negative edges.  B, N, per-vertex counts (both sides), per-pair counts.
 *   oracle_route_g   Alg. 2 BB-Bucket with the ForPar decomposition of
 *                    ParBB-Bucket over start vertices, private buckets per
 *                    thread.  Global B; N = sum B1[w]*B2[w] (Theorem proof, PAPER.md:784:
 *                    "one symmetric and one asymmetric wedge are an unbalanced butterfly");
 *                    W_G = number of priority-eligible wedges.
 *   oracle_route_g_pv  the same Alg. 2 buckets plus the 4-role scatter (SURVEY.md §8(c) O4.3,
 *                    DESIGN.md reading R22): per-vertex B_z, N_z for every vertex of both sides.
 *   oracle_route_s  Alg. vBBFC for a list of vertices: all wedges
 *                    u-v-w, no rank comparison, w != u (reading R9),
 *                    buckets H1/H2, sum C(H1,2)+C(H2,2); the unbalanced count H1*H2 alongside.
 *   oracle_bb_base   Alg. 1 BB-Base: per start, lists H(w) of middles, every
 *                    pair of a list checked for balance explicitly (the paper's baseline).
 *   oracle_pairs     Lemma 2 per same-side pair: C(l,2)+C(m,2) with l / m
 *                    symmetric / asymmetric wedges between the pair, each unordered pair once.
 *   oracle_edge_brute  per-edge counts by brute force: every butterfly of the 4-tuple enumeration
 *                    adds one to each of its four edges (Def. Butterfly).
 *   oracle_edge      per-edge counts by the definition, edge by edge (the butterflies containing
 *                    e = (u,v), "count the number of balanced butterflies
 *                    containing the edge e = (u,v)"; the section's eBBFC pseudocode sits in a block
 *                    the authors removed and indexes its buckets inconsistently, so the oracle
 *                    follows the sentence, reading R24): for each w in Γ(v) \ {u} and each
 *                    x in Γ(w) \ {v} with x in Γ(u), the 4-cycle u-v-w-x is classified by its signs.
 *
 * Arithmetic: wedge buckets are uint32 (a bucket is bounded by a vertex degree); every sum of
 * butterflies is accumulated in unsigned __int128 and checked to fit uint64 (SPEC.md:223,
 * "128-bit accumulation"; "report, do not wrap").
 *
 * Return codes: 0 ok, 1 invalid argument (sign byte not 0/1, null pointer), 2 out of range
 * (col >= n_v, row_ptr not monotone), 3 duplicate edge, 4 out of memory, 7 overflow,
 * 8 output buffer too small (oracle_pairs: *n_pairs holds the required count).
 */
#include <pthread.h>
#include <time.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------------------------------
 * Graph: both sides' adjacency, global ids gid(u) = u for u in U, gid(v) = n_u + v for v in V
 * (SPEC.md:100 global_id scheme).  sgn = +1 / -1 per directed entry.
 * ---------------------------------------------------------------------------------------- */
typedef struct {
  uint32_t n_u, n_v, n;
  uint64_t *off;   /* n+1 */
  uint32_t *nbr;   /* 2*nnz, global ids */
  int8_t *sgn;     /* 2*nnz, +1 / -1 */
  uint64_t *prio;  /* n: priority key, larger = higher priority (Def. Vertex Priority) */
} graph_t;

static void graph_free(graph_t *g) {
  free(g->off); free(g->nbr); free(g->sgn); free(g->prio);
  memset(g, 0, sizeof(*g));
}

static int cmp_u32(const void *a, const void *b) {
  uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
  return (x > y) - (x < y);
}

/* Validate the U-side CSR and build both adjacency lists.  Duplicate check: sort a copy of
 * every row and compare neighbours (DuplicateEdge). */
static int graph_build(graph_t *g, uint32_t n_u, uint32_t n_v, const uint64_t *row_ptr,
                       const uint32_t *col, const uint8_t *sign) {
  memset(g, 0, sizeof(*g));
  if (!row_ptr) return 1;
  if (row_ptr[0] != 0) return 2;
  for (uint32_t u = 0; u < n_u; ++u)
    if (row_ptr[u + 1] < row_ptr[u]) return 2;
  uint64_t nnz = row_ptr[n_u];
  if (nnz && (!col || !sign)) return 1;
  for (uint64_t e = 0; e < nnz; ++e) {
    if (col[e] >= n_v) return 2;
    if (sign[e] > 1) return 1;
  }
  uint32_t maxdeg = 0;
  for (uint32_t u = 0; u < n_u; ++u)
    if (row_ptr[u + 1] - row_ptr[u] > maxdeg) maxdeg = (uint32_t)(row_ptr[u + 1] - row_ptr[u]);
  uint32_t *tmp = (uint32_t *)malloc(sizeof(uint32_t) * (maxdeg + 1));
  if (!tmp) return 4;
  for (uint32_t u = 0; u < n_u; ++u) {
    uint64_t d = row_ptr[u + 1] - row_ptr[u];
    memcpy(tmp, col + row_ptr[u], d * sizeof(uint32_t));
    qsort(tmp, d, sizeof(uint32_t), cmp_u32);
    for (uint64_t i = 1; i < d; ++i)
      if (tmp[i] == tmp[i - 1]) { free(tmp); return 3; }
  }
  free(tmp);

  g->n_u = n_u; g->n_v = n_v; g->n = n_u + n_v;
  g->off = (uint64_t *)calloc((size_t)g->n + 1, sizeof(uint64_t));
  g->nbr = (uint32_t *)malloc(sizeof(uint32_t) * (2 * nnz + 1));
  g->sgn = (int8_t *)malloc(2 * nnz + 1);
  g->prio = (uint64_t *)malloc(sizeof(uint64_t) * ((size_t)g->n + 1));
  if (!g->off || !g->nbr || !g->sgn || !g->prio) { graph_free(g); return 4; }
  /* degrees */
  for (uint32_t u = 0; u < n_u; ++u) g->off[u + 1] = row_ptr[u + 1] - row_ptr[u];
  for (uint64_t e = 0; e < nnz; ++e) g->off[n_u + col[e] + 1] += 1;
  for (uint32_t x = 0; x < g->n; ++x) g->off[x + 1] += g->off[x];
  uint64_t *fill = (uint64_t *)malloc(sizeof(uint64_t) * ((size_t)g->n + 1));
  if (!fill) { graph_free(g); return 4; }
  memcpy(fill, g->off, sizeof(uint64_t) * ((size_t)g->n + 1));
  for (uint32_t u = 0; u < n_u; ++u) {
    for (uint64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
      uint32_t v = n_u + col[e];
      int8_t s = sign[e] ? 1 : -1;  /* weight 1 = positive, 0 = negative */
      g->nbr[fill[u]] = v; g->sgn[fill[u]] = s; fill[u]++;
      g->nbr[fill[v]] = u; g->sgn[fill[v]] = s; fill[v]++;
    }
  }
  free(fill);
  /* Def. Vertex Priority: p(a) > p(b) iff deg(a) > deg(b), or equal degree
   * and id(a) > id(b).  Encoded as the integer key deg * 2^32 + gid. */
  for (uint32_t x = 0; x < g->n; ++x)
    g->prio[x] = ((g->off[x + 1] - g->off[x]) << 32) | (uint64_t)x;
  return 0;
}

/* ------------------------------------------------------------------------------------------
 * Brute force over all 4-tuples (definition).  Dense sign matrix S[u][v] in {-1,0,+1}.
 * Outputs: out[0]=B, out[1]=N; per-vertex arrays (nullable); pair_b (nullable) is an n_u*n_u
 * row-major matrix of per-U-pair balanced counts (upper triangle u<w filled).
 * ---------------------------------------------------------------------------------------- */
int oracle_brute(uint32_t n_u, uint32_t n_v, const uint64_t *row_ptr, const uint32_t *col,
                 const uint8_t *sign, uint64_t *out, uint64_t *bal_u, uint64_t *unb_u,
                 uint64_t *bal_v, uint64_t *unb_v, uint64_t *pair_b_u) {
  graph_t g;
  int rc = graph_build(&g, n_u, n_v, row_ptr, col, sign);
  if (rc) return rc;
  graph_free(&g);
  int8_t *S = (int8_t *)calloc((size_t)n_u * n_v + 1, 1);
  if (!S) return 4;
  for (uint32_t u = 0; u < n_u; ++u)
    for (uint64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e)
      S[(size_t)u * n_v + col[e]] = sign[e] ? 1 : -1;
  u128 B = 0, N = 0;
  if (bal_u) memset(bal_u, 0, sizeof(uint64_t) * n_u);
  if (unb_u) memset(unb_u, 0, sizeof(uint64_t) * n_u);
  if (bal_v) memset(bal_v, 0, sizeof(uint64_t) * n_v);
  if (unb_v) memset(unb_v, 0, sizeof(uint64_t) * n_v);
  if (pair_b_u) memset(pair_b_u, 0, sizeof(uint64_t) * (size_t)n_u * n_u);
  for (uint32_t ui = 0; ui < n_u; ++ui) {
    for (uint32_t uj = ui + 1; uj < n_u; ++uj) {
      const int8_t *ri = S + (size_t)ui * n_v, *rj = S + (size_t)uj * n_v;
      for (uint32_t vi = 0; vi < n_v; ++vi) {
        if (!ri[vi] || !rj[vi]) continue;
        for (uint32_t vj = vi + 1; vj < n_v; ++vj) {
          if (!ri[vj] || !rj[vj]) continue;
          /* cycle v_i-u_i-v_j-u_j (Def. Butterfly); balanced iff an even number of negative
           * edges (Def. Balanced butterfly), i.e. the product of the four signs is +1 */
          int prod = ri[vi] * ri[vj] * rj[vi] * rj[vj];
          int balanced = prod > 0;
          if (balanced) B++; else N++;
          uint64_t *bu = balanced ? bal_u : unb_u, *bv = balanced ? bal_v : unb_v;
          if (bu) { bu[ui]++; bu[uj]++; }
          if (bv) { bv[vi]++; bv[vj]++; }
          if (balanced && pair_b_u) pair_b_u[(size_t)ui * n_u + uj]++;
        }
      }
    }
  }
  free(S);
  if (B >> 64 || N >> 64) return 7;
  out[0] = (uint64_t)B; out[1] = (uint64_t)N;
  return 0;
}

/* ------------------------------------------------------------------------------------------
 * Alg. 2 BB-Bucket, parallel over start vertices as ParBB-Bucket
 * ("ForPar u in U u V"), each worker with private B1/B2.
 * ---------------------------------------------------------------------------------------- */
typedef struct {
  const graph_t *g;
  const uint32_t *starts;  /* NULL: all vertices */
  uint64_t n_starts;
  int tid, nthreads;
  uint64_t *cursor;        /* shared start cursor: starts are handed out in chunks (ForPar) */
  u128 B, N, W;
  int rc;
} rg_task;

#define ORACLE_CHUNK 4u  /* small chunks: the hubs (low ids of the Chung-Lu configs) spread over the threads */

static const graph_t *g_sort_graph;  /* qsort context for line 3 of Alg. 2 */
static int cmp_by_prio(const void *a, const void *b) {
  /* entries are indices into nbr[]; ascending priority of the neighbour */
  uint64_t pa = g_sort_graph->prio[g_sort_graph->nbr[*(const uint64_t *)a]];
  uint64_t pb = g_sort_graph->prio[g_sort_graph->nbr[*(const uint64_t *)b]];
  return (pa > pb) - (pa < pb);
}

/* Line 3: "Rearrange Γ(u) for each u in ascending order" (of priority, reading R8). */
static int sort_adjacency_by_priority(graph_t *g) {
  uint64_t maxd = 0;
  for (uint32_t x = 0; x < g->n; ++x)
    if (g->off[x + 1] - g->off[x] > maxd) maxd = g->off[x + 1] - g->off[x];
  uint64_t *idx = (uint64_t *)malloc(sizeof(uint64_t) * (maxd + 1));
  uint32_t *nb = (uint32_t *)malloc(sizeof(uint32_t) * (maxd + 1));
  int8_t *sg = (int8_t *)malloc(maxd + 1);
  if (!idx || !nb || !sg) { free(idx); free(nb); free(sg); return 4; }
  g_sort_graph = g;
  for (uint32_t x = 0; x < g->n; ++x) {
    uint64_t o = g->off[x], d = g->off[x + 1] - o;
    for (uint64_t i = 0; i < d; ++i) idx[i] = o + i;
    qsort(idx, d, sizeof(uint64_t), cmp_by_prio);
    for (uint64_t i = 0; i < d; ++i) { nb[i] = g->nbr[idx[i]]; sg[i] = g->sgn[idx[i]]; }
    memcpy(g->nbr + o, nb, d * sizeof(uint32_t));
    memcpy(g->sgn + o, sg, d);
  }
  free(idx); free(nb); free(sg);
  return 0;
}

static void *route_g_worker(void *arg) {
  rg_task *t = (rg_task *)arg;
  const graph_t *g = t->g;
  uint32_t *B1 = (uint32_t *)calloc((size_t)g->n + 1, sizeof(uint32_t));
  uint32_t *B2 = (uint32_t *)calloc((size_t)g->n + 1, sizeof(uint32_t));
  uint32_t *touched = (uint32_t *)malloc(sizeof(uint32_t) * ((size_t)g->n + 1));
  if (!B1 || !B2 || !touched) { t->rc = 4; free(B1); free(B2); free(touched); return NULL; }
  uint64_t total = t->starts ? t->n_starts : g->n;
  for (uint64_t i = 0, lim = 0;; ++i) {
    if (i == lim) {
      i = __atomic_fetch_add(t->cursor, ORACLE_CHUNK, __ATOMIC_RELAXED);
      lim = i + ORACLE_CHUNK < total ? i + ORACLE_CHUNK : total;
    }
    if (i >= total) break;
    uint32_t u = t->starts ? t->starts[i] : (uint32_t)i;
    uint64_t pu = g->prio[u];
    uint64_t nt = 0;
    for (uint64_t e = g->off[u]; e < g->off[u + 1]; ++e) {          /* v in Γ(u) */
      uint32_t v = g->nbr[e];
      if (!(g->prio[v] < pu)) break;                                  /* | p(v) < p(u) */
      int8_t s_uv = g->sgn[e];
      for (uint64_t f = g->off[v]; f < g->off[v + 1]; ++f) {        /* w in Γ(v) */
        uint32_t w = g->nbr[f];
        if (!(g->prio[w] < pu)) break;                                /* | p(w) < p(u) */
        if (B1[w] == 0 && B2[w] == 0) touched[nt++] = w;
        if (s_uv == g->sgn[f]) B1[w]++;                               /* σ(u,v) == σ(v,w) */
        else B2[w]++;
        t->W++;
      }
    }
    for (uint64_t k = 0; k < nt; ++k) {                               /* lines 15-18 */
      uint32_t w = touched[k];
      u128 b1 = B1[w], b2 = B2[w];
      t->B += b1 * (b1 - (b1 > 0)) / 2 + b2 * (b2 - (b2 > 0)) / 2;  /* C(B1,2) + C(B2,2) */
      t->N += b1 * b2;
      B1[w] = 0; B2[w] = 0;                                           /* per-u buckets (R5) */
    }
  }
  free(B1); free(B2); free(touched);
  return NULL;
}

/* out[0]=B, out[1]=N, out[2]=W_G, out[3]=wall ns of the counting loop (lines 7-19, after the
 * preprocessing of lines 2-3).  starts: optional list of global ids (NULL = all). */
int oracle_route_g(uint32_t n_u, uint32_t n_v, const uint64_t *row_ptr, const uint32_t *col,
                   const uint8_t *sign, const uint32_t *starts, uint64_t n_starts, int nthreads,
                   uint64_t *out) {
  graph_t g;
  int rc = graph_build(&g, n_u, n_v, row_ptr, col, sign);
  if (rc) return rc;
  if ((rc = sort_adjacency_by_priority(&g))) { graph_free(&g); return rc; }
  if (starts)
    for (uint64_t i = 0; i < n_starts; ++i)
      if (starts[i] >= g.n) { graph_free(&g); return 2; }
  if (nthreads < 1) nthreads = 1;
  rg_task *tasks = (rg_task *)calloc((size_t)nthreads, sizeof(rg_task));
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  uint64_t cursor = 0;
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (int i = 0; i < nthreads; ++i) {
    tasks[i].g = &g; tasks[i].starts = starts; tasks[i].n_starts = n_starts;
    tasks[i].tid = i; tasks[i].nthreads = nthreads; tasks[i].cursor = &cursor;
    pthread_create(&th[i], NULL, route_g_worker, &tasks[i]);
  }
  u128 B = 0, N = 0, W = 0;
  rc = 0;
  for (int i = 0; i < nthreads; ++i) {
    pthread_join(th[i], NULL);
    B += tasks[i].B; N += tasks[i].N; W += tasks[i].W;
    if (tasks[i].rc) rc = tasks[i].rc;
  }
  clock_gettime(CLOCK_MONOTONIC, &t1);
  free(tasks); free(th); graph_free(&g);
  if (rc) return rc;
  if (B >> 64 || N >> 64 || W >> 64) return 7;
  out[0] = (uint64_t)B; out[1] = (uint64_t)N; out[2] = (uint64_t)W;
  out[3] = (uint64_t)(t1.tv_sec - t0.tv_sec) * 1000000000ull + (uint64_t)(t1.tv_nsec - t0.tv_nsec);
  return 0;
}

/* ------------------------------------------------------------------------------------------
 * Alg. 2 with the 4-role scatter (reading R22): per-vertex
 * balanced / unbalanced counts from the same per-start buckets.  Alg. 2 counts every butterfly
 * once, at its maximum-priority vertex u, as a pair (u,w) of its two same-side vertices with
 * two middles v, v' among the l = B1[w] symmetric and m = B2[w] asymmetric wedges u-v-w
 * (Lemma 2: two wedges of the same class form a balanced butterfly, one of
 * each class an unbalanced one; Theorem proof).  So, per start u and end w:
 *   - u and w are in every butterfly of the pair:  C(l,2)+C(m,2) balanced, l*m unbalanced;
 *   - a middle v of a symmetric wedge is in the balanced butterflies it forms with the other
 *     l-1 symmetric middles and in the unbalanced ones it forms with the m asymmetric middles;
 *     a middle of an asymmetric wedge: m-1 balanced, l unbalanced.
 * Step by step: lines 7-14 of Alg. 2 fill B1/B2 (as route_g_worker); then a second sweep over
 * the same wedges hands each middle its share; then lines 15-18 hand u and w theirs.
 * bal / unb are indexed by global id (U: u, V: n_u + v).  Every per-vertex count is at most the
 * global count of its class (a butterfly containing z is counted once for z), so once the global
 * u128 sums are checked to fit uint64 every per-vertex uint64 sum is exact.
 * ---------------------------------------------------------------------------------------- */
typedef struct {
  const graph_t *g;
  const uint32_t *starts;  /* NULL: all vertices */
  uint64_t n_starts;
  int tid, nthreads;
  uint64_t *bal, *unb;
  uint64_t *cursor;
  uint32_t *B1, *B2, *touched;  /* per-thread buckets, zeroed, allocated before the clock starts */
  u128 B, N, W;
  int rc;
} rgpv_task;

static void *route_g_pv_worker(void *arg) {
  rgpv_task *t = (rgpv_task *)arg;
  const graph_t *g = t->g;
  uint32_t *B1 = t->B1, *B2 = t->B2, *touched = t->touched;
  uint64_t total = t->starts ? t->n_starts : g->n;
  for (uint64_t i = 0, lim = 0;; ++i) {
    if (i == lim) {
      i = __atomic_fetch_add(t->cursor, ORACLE_CHUNK, __ATOMIC_RELAXED);
      lim = i + ORACLE_CHUNK < total ? i + ORACLE_CHUNK : total;
    }
    if (i >= total) break;
    uint32_t u = t->starts ? t->starts[i] : (uint32_t)i;
    uint64_t pu = g->prio[u];
    uint64_t nt = 0;
    /* lines 7-14: buckets of the eligible wedges u-v-w */
    for (uint64_t e = g->off[u]; e < g->off[u + 1]; ++e) {
      uint32_t v = g->nbr[e];
      if (!(g->prio[v] < pu)) break;
      for (uint64_t f = g->off[v]; f < g->off[v + 1]; ++f) {
        uint32_t w = g->nbr[f];
        if (!(g->prio[w] < pu)) break;
        if (B1[w] == 0 && B2[w] == 0) touched[nt++] = w;
        if (g->sgn[e] == g->sgn[f]) B1[w]++;
        else B2[w]++;
        t->W++;
      }
    }
    /* middle role: the same wedges again, each middle v summing its shares over its ends */
    for (uint64_t e = g->off[u]; e < g->off[u + 1]; ++e) {
      uint32_t v = g->nbr[e];
      if (!(g->prio[v] < pu)) break;
      u128 bv = 0, nv = 0;
      for (uint64_t f = g->off[v]; f < g->off[v + 1]; ++f) {
        uint32_t w = g->nbr[f];
        if (!(g->prio[w] < pu)) break;
        if (g->sgn[e] == g->sgn[f]) { bv += B1[w] - 1; nv += B2[w]; }  /* symmetric wedge */
        else { bv += B2[w] - 1; nv += B1[w]; }                        /* asymmetric wedge */
      }
      __atomic_fetch_add(&t->bal[v], (uint64_t)bv, __ATOMIC_RELAXED);
      __atomic_fetch_add(&t->unb[v], (uint64_t)nv, __ATOMIC_RELAXED);
    }
    /* lines 15-18, plus the shares of the pair's two same-side vertices u and w */
    u128 bu = 0, nu = 0;
    for (uint64_t k = 0; k < nt; ++k) {
      uint32_t w = touched[k];
      u128 l = B1[w], m = B2[w];
      u128 fb = l * (l - (l > 0)) / 2 + m * (m - (m > 0)) / 2;   /* C(l,2) + C(m,2) */
      u128 fn = l * m;
      bu += fb; nu += fn;
      __atomic_fetch_add(&t->bal[w], (uint64_t)fb, __ATOMIC_RELAXED);
      __atomic_fetch_add(&t->unb[w], (uint64_t)fn, __ATOMIC_RELAXED);
      B1[w] = 0; B2[w] = 0;
    }
    t->B += bu; t->N += nu;
    __atomic_fetch_add(&t->bal[u], (uint64_t)bu, __ATOMIC_RELAXED);
    __atomic_fetch_add(&t->unb[u], (uint64_t)nu, __ATOMIC_RELAXED);
  }
  return NULL;
}

/* A prepared graph (lines 2-3 of Alg. 2 done once: adjacency built, validated and sorted by
 * priority), so repeated counts over start subsets (bench.py's reference arm) do not repeat the
 * preprocessing.  *rc receives the status; NULL on failure. */
void *oracle_prepare(uint32_t n_u, uint32_t n_v, const uint64_t *row_ptr, const uint32_t *col,
                     const uint8_t *sign, int *rc) {
  graph_t *g = (graph_t *)calloc(1, sizeof(graph_t));
  if (!g) { *rc = 4; return NULL; }
  *rc = graph_build(g, n_u, n_v, row_ptr, col, sign);
  if (!*rc) *rc = sort_adjacency_by_priority(g);
  if (*rc) { graph_free(g); free(g); return NULL; }
  return g;
}

void oracle_release(void *h) {
  if (h) { graph_free((graph_t *)h); free(h); }
}

/* out[0]=B, out[1]=N, out[2]=W_G, out[3]=wall ns of the counting loop; bal / unb: n_u + n_v
 * entries each (global ids), overwritten.  starts: optional list of global ids (NULL = all);
 * with a list, the counts are those of the butterflies counted at the listed starts. */
int oracle_route_g_pv_h(void *h, const uint32_t *starts, uint64_t n_starts, int nthreads,
                        uint64_t *out, uint64_t *bal, uint64_t *unb) {
  const graph_t *gp = (const graph_t *)h;
  if (!gp || !bal || !unb || !out) return 1;
  const graph_t g = *gp;
  if (starts)
    for (uint64_t i = 0; i < n_starts; ++i)
      if (starts[i] >= g.n) return 2;
  memset(bal, 0, sizeof(uint64_t) * (size_t)g.n);
  memset(unb, 0, sizeof(uint64_t) * (size_t)g.n);
  if (nthreads < 1) nthreads = 1;
  rgpv_task *tasks = (rgpv_task *)calloc((size_t)nthreads, sizeof(rgpv_task));
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  int oom = !tasks || !th;
  for (int i = 0; i < nthreads && !oom; ++i) {  /* buckets allocated (and zeroed) before the clock */
    tasks[i].B1 = (uint32_t *)calloc((size_t)g.n + 1, sizeof(uint32_t));
    tasks[i].B2 = (uint32_t *)calloc((size_t)g.n + 1, sizeof(uint32_t));
    tasks[i].touched = (uint32_t *)malloc(sizeof(uint32_t) * ((size_t)g.n + 1));
    oom = !tasks[i].B1 || !tasks[i].B2 || !tasks[i].touched;
  }
  if (oom) {
    for (int i = 0; tasks && i < nthreads; ++i) { free(tasks[i].B1); free(tasks[i].B2); free(tasks[i].touched); }
    free(tasks); free(th);
    return 4;
  }
  uint64_t cursor = 0;
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (int i = 0; i < nthreads; ++i) {
    tasks[i].g = &g; tasks[i].tid = i; tasks[i].nthreads = nthreads;
    tasks[i].starts = starts; tasks[i].n_starts = n_starts;
    tasks[i].bal = bal; tasks[i].unb = unb; tasks[i].cursor = &cursor;
    pthread_create(&th[i], NULL, route_g_pv_worker, &tasks[i]);
  }
  u128 B = 0, N = 0, W = 0;
  int rc = 0;
  for (int i = 0; i < nthreads; ++i) {
    pthread_join(th[i], NULL);
    B += tasks[i].B; N += tasks[i].N; W += tasks[i].W;
    if (tasks[i].rc) rc = tasks[i].rc;
  }
  clock_gettime(CLOCK_MONOTONIC, &t1);
  for (int i = 0; i < nthreads; ++i) { free(tasks[i].B1); free(tasks[i].B2); free(tasks[i].touched); }
  free(tasks); free(th);
  if (rc) return rc;
  if (B >> 64 || N >> 64 || W >> 64) return 7;
  out[0] = (uint64_t)B; out[1] = (uint64_t)N; out[2] = (uint64_t)W;
  out[3] = (uint64_t)(t1.tv_sec - t0.tv_sec) * 1000000000ull + (uint64_t)(t1.tv_nsec - t0.tv_nsec);
  return 0;
}

int oracle_route_g_pv(uint32_t n_u, uint32_t n_v, const uint64_t *row_ptr, const uint32_t *col,
                      const uint8_t *sign, const uint32_t *starts, uint64_t n_starts,
                      int nthreads, uint64_t *out, uint64_t *bal, uint64_t *unb) {
  if (!bal || !unb || !out) return 1;
  int rc = 0;
  void *h = oracle_prepare(n_u, n_v, row_ptr, col, sign, &rc);
  if (!h) return rc;
  rc = oracle_route_g_pv_h(h, starts, n_starts, nthreads, out, bal, unb);
  oracle_release(h);
  return rc;
}

/* ------------------------------------------------------------------------------------------
 * Alg. 1 BB-Base: the same priority-eligible wedges as Alg. 2, but each start
 * u stores the middles of every end w in a list H(w) (line 9: "H(w).add(v)") and then checks
 * every pair (v1, v2) of H(w) explicitly (lines 10-13: "if butterfly (u,v1,w,v2) is balanced,
 * count++").  Balanced = an even number of negative edges among the four (Def. Balanced
 * butterfly); the pairs that fail the check are the unbalanced butterflies.
 * Each unordered pair {v1, v2} is visited once.  Parallel over starts like route_g.
 * ---------------------------------------------------------------------------------------- */
typedef struct {
  const graph_t *g;
  int tid, nthreads;
  u128 B, N, W;
  int rc;
} bb_task;

static void *bb_base_worker(void *arg) {
  bb_task *t = (bb_task *)arg;
  const graph_t *g = t->g;
  uint64_t *cnt = (uint64_t *)calloc((size_t)g->n + 1, sizeof(uint64_t));   /* |H(w)| */
  uint64_t *pos = (uint64_t *)calloc((size_t)g->n + 1, sizeof(uint64_t));   /* H(w) start */
  uint32_t *touched = (uint32_t *)malloc(sizeof(uint32_t) * ((size_t)g->n + 1));
  uint64_t cap = 1024;
  int8_t *hs = (int8_t *)malloc(cap * 2);   /* H entries: (σ(u,v), σ(v,w)) of each stored v */
  if (!cnt || !pos || !touched || !hs) { t->rc = 4; goto done; }
  for (uint32_t u = (uint32_t)t->tid; u < g->n; u += (uint32_t)t->nthreads) {
    uint64_t pu = g->prio[u], nt = 0, tot = 0;
    /* lines 7-9, first sweep: |H(w)| (so every list can be stored contiguously) */
    for (uint64_t e = g->off[u]; e < g->off[u + 1]; ++e) {
      uint32_t v = g->nbr[e];
      if (!(g->prio[v] < pu)) break;                                  /* | p(v) < p(u) */
      for (uint64_t f = g->off[v]; f < g->off[v + 1]; ++f) {
        uint32_t w = g->nbr[f];
        if (!(g->prio[w] < pu)) break;                                /* | p(w) < p(u) */
        if (cnt[w] == 0) touched[nt++] = w;
        cnt[w]++;
        tot++;
      }
    }
    t->W += tot;
    if (tot > cap) {
      free(hs);
      cap = tot;
      hs = (int8_t *)malloc(cap * 2);
      if (!hs) { t->rc = 4; goto done; }
    }
    uint64_t acc = 0;
    for (uint64_t k = 0; k < nt; ++k) { pos[touched[k]] = acc; acc += cnt[touched[k]]; cnt[touched[k]] = 0; }
    /* second sweep: H(w).add(v), keeping the two signs the balance check needs */
    for (uint64_t e = g->off[u]; e < g->off[u + 1]; ++e) {
      uint32_t v = g->nbr[e];
      if (!(g->prio[v] < pu)) break;
      for (uint64_t f = g->off[v]; f < g->off[v + 1]; ++f) {
        uint32_t w = g->nbr[f];
        if (!(g->prio[w] < pu)) break;
        uint64_t i = pos[w] + cnt[w]++;
        hs[2 * i] = g->sgn[e];
        hs[2 * i + 1] = g->sgn[f];
      }
    }
    /* lines 10-13: every pair of H(w), |H(w)| > 1 */
    for (uint64_t k = 0; k < nt; ++k) {
      uint32_t w = touched[k];
      uint64_t o = pos[w], c = cnt[w];
      for (uint64_t i = 0; i + 1 < c; ++i)
        for (uint64_t j = i + 1; j < c; ++j) {
          int prod = hs[2 * (o + i)] * hs[2 * (o + i) + 1] * hs[2 * (o + j)] * hs[2 * (o + j) + 1];
          if (prod > 0) t->B++;                                       /* is_Balanced */
          else t->N++;
        }
      cnt[w] = 0;
    }
  }
done:
  free(cnt); free(pos); free(touched); free(hs);
  return NULL;
}

/* out[0]=B, out[1]=N, out[2]=W_G, out[3]=wall ns of the counting loop (after lines 2-3). */
int oracle_bb_base(uint32_t n_u, uint32_t n_v, const uint64_t *row_ptr, const uint32_t *col,
                   const uint8_t *sign, int nthreads, uint64_t *out) {
  graph_t g;
  int rc = graph_build(&g, n_u, n_v, row_ptr, col, sign);
  if (rc) return rc;
  if ((rc = sort_adjacency_by_priority(&g))) { graph_free(&g); return rc; }
  if (nthreads < 1) nthreads = 1;
  bb_task *tasks = (bb_task *)calloc((size_t)nthreads, sizeof(bb_task));
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (int i = 0; i < nthreads; ++i) {
    tasks[i].g = &g; tasks[i].tid = i; tasks[i].nthreads = nthreads;
    pthread_create(&th[i], NULL, bb_base_worker, &tasks[i]);
  }
  u128 B = 0, N = 0, W = 0;
  rc = 0;
  for (int i = 0; i < nthreads; ++i) {
    pthread_join(th[i], NULL);
    B += tasks[i].B; N += tasks[i].N; W += tasks[i].W;
    if (tasks[i].rc) rc = tasks[i].rc;
  }
  clock_gettime(CLOCK_MONOTONIC, &t1);
  free(tasks); free(th); graph_free(&g);
  if (rc) return rc;
  if (B >> 64 || N >> 64 || W >> 64) return 7;
  out[0] = (uint64_t)B; out[1] = (uint64_t)N; out[2] = (uint64_t)W;
  out[3] = (uint64_t)(t1.tv_sec - t0.tv_sec) * 1000000000ull + (uint64_t)(t1.tv_nsec - t0.tv_nsec);
  return 0;
}

/* ------------------------------------------------------------------------------------------
 * vBBFC for a list of vertices.  verts are global ids (NULL = all n).
 * bal[i], unb[i] receive the counts of verts[i].  pair mode (oracle_pairs) additionally
 * emits, for each listed z and each same-side y > z with C(H1,2)+C(H2,2) > 0, the record
 * (z, y, balanced, unbalanced).
 * ---------------------------------------------------------------------------------------- */
typedef struct {
  const graph_t *g;
  const uint32_t *verts;
  uint64_t n_verts;
  int tid, nthreads;
  uint64_t *bal, *unb;
  /* pair emission */
  int emit_pairs;
  uint32_t *pz, *py; uint64_t *pb, *pn;
  uint64_t cap, *cursor; pthread_mutex_t *mu;
  int rc;
} rs_task;

static void *route_s_worker(void *arg) {
  rs_task *t = (rs_task *)arg;
  const graph_t *g = t->g;
  uint32_t *H1 = (uint32_t *)calloc((size_t)g->n + 1, sizeof(uint32_t));
  uint32_t *H2 = (uint32_t *)calloc((size_t)g->n + 1, sizeof(uint32_t));
  uint32_t *touched = (uint32_t *)malloc(sizeof(uint32_t) * ((size_t)g->n + 1));
  if (!H1 || !H2 || !touched) { t->rc = 4; free(H1); free(H2); free(touched); return NULL; }
  uint64_t total = t->verts ? t->n_verts : g->n;
  for (uint64_t i = (uint64_t)t->tid; i < total; i += (uint64_t)t->nthreads) {
    uint32_t u = t->verts ? t->verts[i] : (uint32_t)i;
    uint64_t nt = 0;
    for (uint64_t e = g->off[u]; e < g->off[u + 1]; ++e) {      /* for v in Γ(u) */
      uint32_t v = g->nbr[e];
      for (uint64_t f = g->off[v]; f < g->off[v + 1]; ++f) {    /* for w in Γ(v) */
        uint32_t w = g->nbr[f];
        if (w == u) continue;                                   /* reading R9: w != u */
        if (H1[w] == 0 && H2[w] == 0) touched[nt++] = w;
        if (g->sgn[e] == g->sgn[f]) H1[w]++;                    /* σ(u,v) == σ(v,w) */
        else H2[w]++;
      }
    }
    u128 b = 0, nb = 0;
    for (uint64_t k = 0; k < nt; ++k) {
      uint32_t w = touched[k];
      u128 h1 = H1[w], h2 = H2[w];
      u128 pb = h1 * (h1 - (h1 > 0)) / 2 + h2 * (h2 - (h2 > 0)) / 2;
      u128 pn = h1 * h2;
      b += pb; nb += pn;
      if (t->emit_pairs && w > u && pb > 0) {
        pthread_mutex_lock(t->mu);
        uint64_t c = (*t->cursor)++;
        pthread_mutex_unlock(t->mu);
        if (c < t->cap) {
          t->pz[c] = u; t->py[c] = w;
          t->pb[c] = (uint64_t)pb; t->pn[c] = (uint64_t)pn;
        }
      }
      H1[w] = 0; H2[w] = 0;
    }
    if ((b >> 64) || (nb >> 64)) t->rc = 7;
    if (t->bal) t->bal[i] = (uint64_t)b;
    if (t->unb) t->unb[i] = (uint64_t)nb;
  }
  free(H1); free(H2); free(touched);
  return NULL;
}

static int run_route_s(const graph_t *g, const uint32_t *verts, uint64_t n_verts, int nthreads,
                       uint64_t *bal, uint64_t *unb, int emit, uint32_t *pz, uint32_t *py,
                       uint64_t *pb, uint64_t *pn, uint64_t cap, uint64_t *n_pairs) {
  if (nthreads < 1) nthreads = 1;
  rs_task *tasks = (rs_task *)calloc((size_t)nthreads, sizeof(rs_task));
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
  uint64_t cursor = 0;
  for (int i = 0; i < nthreads; ++i) {
    rs_task *t = &tasks[i];
    t->g = g; t->verts = verts; t->n_verts = n_verts; t->tid = i; t->nthreads = nthreads;
    t->bal = bal; t->unb = unb; t->emit_pairs = emit;
    t->pz = pz; t->py = py; t->pb = pb; t->pn = pn; t->cap = cap; t->cursor = &cursor; t->mu = &mu;
    pthread_create(&th[i], NULL, route_s_worker, t);
  }
  int rc = 0;
  for (int i = 0; i < nthreads; ++i) {
    pthread_join(th[i], NULL);
    if (tasks[i].rc) rc = tasks[i].rc;
  }
  free(tasks); free(th);
  if (n_pairs) *n_pairs = cursor;
  if (!rc && emit && cursor > cap) rc = 8;
  return rc;
}

int oracle_route_s(uint32_t n_u, uint32_t n_v, const uint64_t *row_ptr, const uint32_t *col,
                   const uint8_t *sign, const uint32_t *verts, uint64_t n_verts, int nthreads,
                   uint64_t *bal, uint64_t *unb) {
  graph_t g;
  int rc = graph_build(&g, n_u, n_v, row_ptr, col, sign);
  if (rc) return rc;
  if (verts)
    for (uint64_t i = 0; i < n_verts; ++i)
      if (verts[i] >= g.n) { graph_free(&g); return 2; }
  rc = run_route_s(&g, verts, n_verts, nthreads, bal, unb, 0, NULL, NULL, NULL, NULL, 0, NULL);
  graph_free(&g);
  return rc;
}

/* Per-pair Lemma 2 counts for side (0 = U, 1 = V): every unordered same-side pair {z, y} with a
 * positive balanced count, once (z < y in side-local ids).  Records are written in no
 * particular order; *n_pairs returns the number found (rc 8 if it exceeds cap). */
int oracle_pairs(uint32_t n_u, uint32_t n_v, const uint64_t *row_ptr, const uint32_t *col,
                 const uint8_t *sign, int side, int nthreads, uint32_t *pz, uint32_t *py,
                 uint64_t *pb, uint64_t *pn, uint64_t cap, uint64_t *n_pairs) {
  graph_t g;
  int rc = graph_build(&g, n_u, n_v, row_ptr, col, sign);
  if (rc) return rc;
  if (side != 0 && side != 1) { graph_free(&g); return 1; }
  uint32_t lo = side ? n_u : 0, cnt = side ? n_v : n_u;
  uint32_t *verts = (uint32_t *)malloc(sizeof(uint32_t) * ((size_t)cnt + 1));
  if (!verts) { graph_free(&g); return 4; }
  for (uint32_t i = 0; i < cnt; ++i) verts[i] = lo + i;
  rc = run_route_s(&g, verts, cnt, nthreads, NULL, NULL, 1, pz, py, pb, pn, cap, n_pairs);
  free(verts);
  uint64_t got = n_pairs ? (*n_pairs < cap ? *n_pairs : cap) : 0;
  for (uint64_t i = 0; i < got; ++i) { pz[i] -= lo; py[i] -= lo; }  /* side-local ids */
  graph_free(&g);
  return rc;
}

/* Def. Vertex Priority exposed for its own pin (SPEC.md:68 example): writes, for every global
 * id, its position in descending priority order (0 = highest). */
int oracle_priority_order(uint32_t n_u, uint32_t n_v, const uint64_t *row_ptr,
                          const uint32_t *col, const uint8_t *sign, uint32_t *pos) {
  graph_t g;
  int rc = graph_build(&g, n_u, n_v, row_ptr, col, sign);
  if (rc) return rc;
  for (uint32_t a = 0; a < g.n; ++a) {
    uint32_t higher = 0;
    for (uint32_t b = 0; b < g.n; ++b) higher += g.prio[b] > g.prio[a];  /* plain O(n^2) count */
    pos[a] = higher;
  }
  graph_free(&g);
  return 0;
}

/* ------------------------------------------------------------------------------------------
 * SBESPAR sparsification (§Approximation by Sparsification): "samples each
 * edge in the network independently with a fixed probability rho and constructs a network with
 * the sampled edges E' only".  The independent draws come from the counter-based generator the
 * library documents (include/bbf.h, bbf_estimate_global), written out here on its own:
 * SplitMix64 sm64(x) = mix(x + 0x9E3779B97F4A7C15); trial t uses key = sm64(seed + t); edge e of
 * the U-side CSR is kept iff rho >= 1 or sm64(key ^ e) < floor(rho * 2^64).
 * out_rp: n_u+1; out_col / out_sign: capacity nnz; *out_nnz receives the kept count.
 * ---------------------------------------------------------------------------------------- */
uint64_t oracle_sm64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int oracle_sparsify(uint32_t n_u, const uint64_t *row_ptr, const uint32_t *col, const uint8_t *sign,
                    double rho, uint64_t seed, uint32_t trial, uint64_t *out_rp, uint32_t *out_col,
                    uint8_t *out_sign, uint64_t *out_nnz) {
  if (!(rho > 0.0 && rho <= 1.0)) return 1;
  const uint64_t key = oracle_sm64(seed + trial);
  const int keep_all = rho >= 1.0;
  const uint64_t thr = keep_all ? ~0ull : (uint64_t)(rho * 18446744073709551616.0);
  uint64_t k = 0;
  out_rp[0] = 0;
  for (uint32_t u = 0; u < n_u; ++u) {
    for (uint64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
      if (keep_all || oracle_sm64(key ^ e) < thr) {
        out_col[k] = col[e];
        out_sign[k] = sign[e];
        ++k;
      }
    }
    out_rp[u + 1] = k;
  }
  *out_nnz = k;
  return 0;
}

/* ------------------------------------------------------------------------------------------
 * Per-edge counts.  Edge e of the input U-side CSR (u, col[e]); outputs in
 * input CSR order.  oracle_edge_brute: dense sign matrix, all 4-tuples (tiny graphs only).
 * ---------------------------------------------------------------------------------------- */
int oracle_edge_brute(uint32_t n_u, uint32_t n_v, const uint64_t *row_ptr, const uint32_t *col,
                      const uint8_t *sign, uint64_t *bal, uint64_t *unb) {
  graph_t g;
  int rc = graph_build(&g, n_u, n_v, row_ptr, col, sign);
  if (rc) return rc;
  graph_free(&g);
  const uint64_t nnz = row_ptr[n_u];
  int8_t *S = (int8_t *)calloc((size_t)n_u * n_v + 1, 1);
  int64_t *E = (int64_t *)malloc(sizeof(int64_t) * ((size_t)n_u * n_v + 1));  /* edge id or -1 */
  if (!S || !E) { free(S); free(E); return 4; }
  for (size_t i = 0; i < (size_t)n_u * n_v; ++i) E[i] = -1;
  for (uint32_t u = 0; u < n_u; ++u)
    for (uint64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
      S[(size_t)u * n_v + col[e]] = sign[e] ? 1 : -1;
      E[(size_t)u * n_v + col[e]] = (int64_t)e;
    }
  memset(bal, 0, sizeof(uint64_t) * nnz);
  memset(unb, 0, sizeof(uint64_t) * nnz);
  for (uint32_t ui = 0; ui < n_u; ++ui)
    for (uint32_t uj = ui + 1; uj < n_u; ++uj)
      for (uint32_t vi = 0; vi < n_v; ++vi) {
        if (!S[(size_t)ui * n_v + vi] || !S[(size_t)uj * n_v + vi]) continue;
        for (uint32_t vj = vi + 1; vj < n_v; ++vj) {
          if (!S[(size_t)ui * n_v + vj] || !S[(size_t)uj * n_v + vj]) continue;
          const int prod = S[(size_t)ui * n_v + vi] * S[(size_t)ui * n_v + vj] * S[(size_t)uj * n_v + vi] *
                           S[(size_t)uj * n_v + vj];
          uint64_t *t = prod > 0 ? bal : unb;   /* Def. Balanced butterfly: even # negatives */
          t[E[(size_t)ui * n_v + vi]]++; t[E[(size_t)ui * n_v + vj]]++;
          t[E[(size_t)uj * n_v + vi]]++; t[E[(size_t)uj * n_v + vj]]++;
        }
      }
  free(S); free(E);
  return 0;
}

static int8_t sign_of(const graph_t *g, uint32_t a, uint32_t b) {  /* 0 if (a, b) is no edge */
  for (uint64_t f = g->off[a]; f < g->off[a + 1]; ++f)
    if (g->nbr[f] == b) return g->sgn[f];
  return 0;
}

typedef struct {
  const graph_t *g;
  const uint64_t *row_ptr;
  const uint32_t *col;
  uint32_t n_u;
  uint64_t *bal, *unb, *cursor;
  int rc;
} edge_task;

static void *edge_worker(void *arg) {
  edge_task *t = (edge_task *)arg;
  const graph_t *g = t->g;
  const uint64_t nnz = t->row_ptr[t->n_u];
  for (uint64_t i = 0, lim = 0;; ++i) {
    if (i == lim) {
      i = __atomic_fetch_add(t->cursor, ORACLE_CHUNK, __ATOMIC_RELAXED);
      lim = i + ORACLE_CHUNK < nnz ? i + ORACLE_CHUNK : nnz;
    }
    if (i >= nnz) break;
    uint32_t lo = 0, hi = t->n_u;               /* u: the row holding edge i (row_ptr[u] <= i) */
    while (hi - lo > 1) {
      const uint32_t md = lo + (hi - lo) / 2;
      if (t->row_ptr[md] <= i) lo = md; else hi = md;
    }
    const uint32_t u = lo;
    const uint32_t v = t->n_u + t->col[i];
    const int8_t s_uv = sign_of(g, u, v);
    u128 b = 0, n = 0;
    for (uint64_t f = g->off[v]; f < g->off[v + 1]; ++f) {       /* w in Γ(v) \ {u} */
      const uint32_t w = g->nbr[f];
      if (w == u) continue;
      const int8_t s_vw = g->sgn[f];
      for (uint64_t h = g->off[w]; h < g->off[w + 1]; ++h) {     /* x in Γ(w) \ {v} */
        const uint32_t x = g->nbr[h];
        if (x == v) continue;
        const int8_t s_ux = sign_of(g, u, x);                  /* x in Γ(u)? */
        if (!s_ux) continue;
        if (s_uv * s_vw * g->sgn[h] * s_ux > 0) b++; else n++;  /* the 4-cycle u-v-w-x */
      }
    }
    if ((b >> 64) || (n >> 64)) t->rc = 7;
    t->bal[i] = (uint64_t)b;
    t->unb[i] = (uint64_t)n;
  }
  return NULL;
}

int oracle_edge(uint32_t n_u, uint32_t n_v, const uint64_t *row_ptr, const uint32_t *col,
                const uint8_t *sign, int nthreads, uint64_t *bal, uint64_t *unb) {
  graph_t g;
  int rc = graph_build(&g, n_u, n_v, row_ptr, col, sign);
  if (rc) return rc;
  if (nthreads < 1) nthreads = 1;
  edge_task *tasks = (edge_task *)calloc((size_t)nthreads, sizeof(edge_task));
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  uint64_t cursor = 0;
  for (int i = 0; i < nthreads; ++i) {
    tasks[i].g = &g; tasks[i].row_ptr = row_ptr; tasks[i].col = col; tasks[i].n_u = n_u;
    tasks[i].bal = bal; tasks[i].unb = unb; tasks[i].cursor = &cursor;
    pthread_create(&th[i], NULL, edge_worker, &tasks[i]);
  }
  rc = 0;
  for (int i = 0; i < nthreads; ++i) {
    pthread_join(th[i], NULL);
    if (tasks[i].rc) rc = tasks[i].rc;
  }
  free(tasks); free(th); graph_free(&g);
  return rc;
}
