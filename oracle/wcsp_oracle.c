/* wcsp_oracle.c — plain, slow, obviously-correct CPU oracle (see wcsp_oracle.h).
 *
 * TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench.py cpu_baseline leg).
 * Shares nothing with the CUDA path.  Integer arithmetic only (PAPER.md:3,
 * "The passage times over the edges are assumed to be positive integers").
 *
 * Four tiers, each an independent algorithm, pinned against each other and
 * against closed forms in tests/test_oracle.py:
 *   tier 1 orc_dense  — the definition as a shortest path on
 *                       the product graph (vertex, spent weight).
 *   tier 2 orc_pruned — label setting in time order on (vertex, remaining
 *                       quality), the "water quality" reading of PAPER.md:29.
 *   tier 3 orc_lex    — Dijkstra with lexicographic keys (the two M endpoints,
 *                       SURVEY §8(c) P4, and M = infinity).
 *   tier 4 orc_brute  — enumeration of simple paths (tiny graphs).
 *   tier 5 orc_model  — the paper's own cycle (§4) run sequentially,
 *                       one vertex and one edge at a time; it also counts the
 *                       method's work (the north_star metric's numerator).
 */
#include "wcsp_oracle.h"

#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* Graph access: the lattice neighbours of v over present edges.             */
/* ------------------------------------------------------------------------- */

typedef struct {
  int d;
  int64_t n[4], stride[4], N;
  const orc_problem* p;
} grid;

static void grid_init(grid* g, const orc_problem* p) {
  g->d = p->d;
  g->p = p;
  int64_t s = 1;
  for (int k = 0; k < p->d; ++k) {
    g->n[k] = p->shape[k];
    g->stride[k] = s;
    s *= p->shape[k];
  }
  g->N = s;
}

static int is_present(const grid* g, int64_t v) { return g->p->present == NULL || g->p->present[v] != 0; }

/* Fill u[], f1[], f2[] with the neighbours of v; returns their number (<= 8). */
static int neighbours(const grid* g, int64_t v, int64_t* u, int* f1, int* f2) {
  int c = 0;
  if (!is_present(g, v)) return 0;
  for (int k = 0; k < g->d; ++k) {
    int64_t xk = (v / g->stride[k]) % g->n[k];
    if (xk + 1 < g->n[k]) { /* edge (v, v+e_k) is stored at v */
      int64_t w = v + g->stride[k];
      int a = g->p->f1[k * g->N + v];
      if (a > 0 && is_present(g, w)) { u[c] = w; f1[c] = a; f2[c] = g->p->f2[k * g->N + v]; ++c; }
    }
    if (xk > 0) { /* edge (v-e_k, v) is stored at v-e_k */
      int64_t w = v - g->stride[k];
      int a = g->p->f1[k * g->N + w];
      if (a > 0 && is_present(g, w)) { u[c] = w; f1[c] = a; f2[c] = g->p->f2[k * g->N + w]; ++c; }
    }
  }
  return c;
}

static int inA(const grid* g, int64_t v) { return g->p->maskA[v] && is_present(g, v); }
static int inB(const grid* g, int64_t v) { return g->p->maskB[v] && is_present(g, v); }

static int check_problem(const orc_problem* p) {
  if (p->d < 1 || p->d > 4) return ORC_EINVAL;
  for (int k = 0; k < p->d; ++k) if (p->shape[k] < 1) return ORC_EINVAL;
  if (p->M != ORC_M_INF && p->M < 1) return ORC_EINVAL;
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Binary min-heap of (key1, key2, id), lazy deletion.                       */
/* ------------------------------------------------------------------------- */

typedef struct { int64_t k1, k2, id; } hitem;
typedef struct { hitem* a; int64_t n, cap; } heap;

static int hless(const hitem* x, const hitem* y) {
  return x->k1 < y->k1 || (x->k1 == y->k1 && (x->k2 < y->k2 || (x->k2 == y->k2 && x->id < y->id)));
}

static int heap_push(heap* h, int64_t k1, int64_t k2, int64_t id) {
  if (h->n == h->cap) {
    int64_t nc = h->cap ? 2 * h->cap : 1024;
    hitem* na = (hitem*)realloc(h->a, (size_t)nc * sizeof(hitem));
    if (!na) return -1;
    h->a = na;
    h->cap = nc;
  }
  int64_t i = h->n++;
  h->a[i].k1 = k1; h->a[i].k2 = k2; h->a[i].id = id;
  while (i > 0) {
    int64_t par = (i - 1) / 2;
    if (!hless(&h->a[i], &h->a[par])) break;
    hitem t = h->a[i]; h->a[i] = h->a[par]; h->a[par] = t;
    i = par;
  }
  return 0;
}

static hitem heap_pop(heap* h) {
  hitem top = h->a[0];
  h->a[0] = h->a[--h->n];
  int64_t i = 0;
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < h->n && hless(&h->a[l], &h->a[m])) m = l;
    if (r < h->n && hless(&h->a[r], &h->a[m])) m = r;
    if (m == i) break;
    hitem t = h->a[i]; h->a[i] = h->a[m]; h->a[m] = t;
    i = m;
  }
  return top;
}

/* ------------------------------------------------------------------------- */
/* Tier 1: product-graph Dijkstra.                                           */
/* State (v, s): at v having spent weight s = F2 so far, s in [0, M-1].      */
/* Arc (v, s) -> (u, s + f2) with cost f1 if s + f2 < M (PAPER.md:21 strict). */
/* Sources (a, 0), a in A.  B states are not expanded (a path reaching B     */
/* earlier is strictly faster, so optimal paths touch B only at the end).    */
/* ------------------------------------------------------------------------- */

#define INF64 INT64_MAX

int orc_dense(const orc_problem* p, orc_result* r) {
  memset(r, 0, sizeof(*r));
  if (check_problem(p) || p->M == ORC_M_INF) return (int)(r->status = ORC_EINVAL);
  grid g;
  grid_init(&g, p);
  const int64_t M = p->M, N = g.N;
  if (N * M > (int64_t)400000000) return (int)(r->status = ORC_ELIMIT);
  int64_t* dist = (int64_t*)malloc((size_t)(N * M) * sizeof(int64_t));
  if (!dist) return (int)(r->status = ORC_ENOMEM);
  for (int64_t i = 0; i < N * M; ++i) dist[i] = INF64;
  heap h = {0};
  for (int64_t a = 0; a < N; ++a)
    if (inA(&g, a)) { dist[a * M + 0] = 0; heap_push(&h, 0, 0, a * M + 0); }
  int64_t u[8];
  int f1[8], f2[8];
  while (h.n > 0) {
    hitem it = heap_pop(&h);
    if (it.k1 != dist[it.id]) continue;
    int64_t v = it.id / M, s = it.id % M;
    if (inB(&g, v)) continue;
    int c = neighbours(&g, v, u, f1, f2);
    for (int i = 0; i < c; ++i) {
      int64_t s2 = s + f2[i];
      if (s2 >= M) continue;
      int64_t id2 = u[i] * M + s2, d2 = it.k1 + f1[i];
      if (d2 < dist[id2]) { dist[id2] = d2; heap_push(&h, d2, 0, id2); }
    }
  }
  free(h.a);
  /* F1* = min over b in B, s; F2* = min s at F1*; X* = min b at (F1*, F2*). */
  int64_t F1 = INF64, F2 = INF64, X = -1;
  for (int64_t b = 0; b < N; ++b) {
    if (!inB(&g, b)) continue;
    for (int64_t s = 0; s < M; ++s) {
      int64_t dv = dist[b * M + s];
      if (dv == INF64) continue;
      if (dv < F1 || (dv == F1 && s < F2) || (dv == F1 && s == F2 && b < X)) { F1 = dv; F2 = s; X = b; }
    }
  }
  if (X < 0) {
    free(dist);
    r->status = ORC_INFEASIBLE;
    return ORC_INFEASIBLE;
  }
  /* Y* = min y ~ X*, y not in B, with dist(y, F2* - f2(y,X*)) = F1* - f1(y,X*). */
  int64_t Y = INF64;
  int c = neighbours(&g, X, u, f1, f2);
  for (int i = 0; i < c; ++i) {
    if (inB(&g, u[i])) continue;
    int64_t s = F2 - f2[i];
    if (s < 0) continue;
    if (dist[u[i] * M + s] == F1 - f1[i] && u[i] < Y) Y = u[i];
  }
  free(dist);
  r->status = ORC_REACHED;
  r->F1 = F1; r->F2 = F2; r->X = X; r->Y = Y;
  return ORC_REACHED;
}

/* ------------------------------------------------------------------------- */
/* Tier 2: label setting in time order on (vertex, remaining quality).       */
/* Water of quality q at v crossing e arrives at t + f1(e) with q - f2(e)    */
/* (PAPER.md:29); quality <= 0 cannot travel (reading R3); a    */
/* vertex keeps the best quality seen so far, best_q (labels start at M on A  */
/* and 0 elsewhere).  At each event time t: per vertex,    */
/* q* = max quality among arrivals at t that beat best_q; if a B vertex gets  */
/* one, stop (first drop at B gives F1); otherwise every   */
/* improved vertex sends its new water to each neighbour it could improve.    */
/* M = infinity is the first-arrival special case: q = 1 everywhere, f2 := 0  */
/* (reading R14).                                                            */
/* `work` = sum over processed event times of the flows in flight at that     */
/* time (created earlier, arriving now or later).                            */
/* ------------------------------------------------------------------------- */

typedef struct { uint32_t v; int32_t q; uint32_t src; } event;
typedef struct { event* a; int64_t n, cap; } evec;

static int evec_push(evec* e, uint32_t v, int32_t q, uint32_t src) {
  if (e->n == e->cap) {
    int64_t nc = e->cap ? 2 * e->cap : 256;
    event* na = (event*)realloc(e->a, (size_t)nc * sizeof(event));
    if (!na) return -1;
    e->a = na;
    e->cap = nc;
  }
  e->a[e->n].v = v; e->a[e->n].q = q; e->a[e->n].src = src;
  e->n++;
  return 0;
}

#define NBUCKET 256 /* f1 <= 255, so every event lies within 255 time units */

int orc_pruned(const orc_problem* p, int64_t t_limit, orc_result* r) {
  memset(r, 0, sizeof(*r));
  if (check_problem(p)) return (int)(r->status = ORC_EINVAL);
  grid g;
  grid_init(&g, p);
  const int64_t N = g.N;
  if (N > (int64_t)UINT32_MAX) return (int)(r->status = ORC_ELIMIT);
  const int minf = (p->M == ORC_M_INF);
  const int32_t M = minf ? 1 : (int32_t)p->M;
  int32_t* best_q = (int32_t*)calloc((size_t)N, sizeof(int32_t));
  int32_t* qstar = (int32_t*)calloc((size_t)N, sizeof(int32_t));
  uint32_t* touched = (uint32_t*)malloc((size_t)N * sizeof(uint32_t));
  evec bucket[NBUCKET];
  memset(bucket, 0, sizeof(bucket));
  if (!best_q || !qstar || !touched) { free(best_q); free(qstar); free(touched); return (int)(r->status = ORC_ENOMEM); }
  int64_t u[8];
  int f1[8], f2[8];
  int64_t pending = 0, work = 0, cycles = 0;
  int status = ORC_INFEASIBLE;

  /* t = 0: A holds water of quality M; it starts flowing. */
  for (int64_t a = 0; a < N; ++a) if (inA(&g, a)) best_q[a] = M;
  for (int64_t a = 0; a < N; ++a) {
    if (!inA(&g, a)) continue;
    int c = neighbours(&g, a, u, f1, f2);
    for (int i = 0; i < c; ++i) {
      int32_t nq = M - (minf ? 0 : f2[i]);
      if (nq > 0 && nq > best_q[u[i]]) { evec_push(&bucket[f1[i] % NBUCKET], (uint32_t)u[i], nq, (uint32_t)a); ++pending; }
    }
  }
  int64_t t = 0;
  while (pending > 0) {
    /* advance to the next event time */
    do { ++t; } while (bucket[t % NBUCKET].n == 0);
    if (t_limit > 0 && t > t_limit) { status = ORC_ELIMIT; break; }
    evec* E = &bucket[t % NBUCKET];
    work += pending;
    ++cycles;
    pending -= E->n;
    /* pass 1: q* per vertex over arrivals that beat the current label */
    int64_t nt = 0;
    for (int64_t i = 0; i < E->n; ++i) {
      event ev = E->a[i];
      if (ev.q > 0 && ev.q > best_q[ev.v]) {
        if (qstar[ev.v] == 0) touched[nt++] = ev.v;
        if (ev.q > qstar[ev.v]) qstar[ev.v] = ev.q;
      }
    }
    /* first drop at B: F1 = t, F2 = M - q, X = min index at max q, Y = min source */
    int64_t X = -1;
    int32_t qb = 0;
    for (int64_t i = 0; i < nt; ++i) {
      uint32_t v = touched[i];
      if (!inB(&g, v)) continue;
      if (qstar[v] > qb || (qstar[v] == qb && (int64_t)v < X)) { qb = qstar[v]; X = v; }
    }
    if (X >= 0) {
      int64_t Y = INT64_MAX;
      for (int64_t i = 0; i < E->n; ++i)
        if (E->a[i].v == (uint32_t)X && E->a[i].q == qb && (int64_t)E->a[i].src < Y) Y = E->a[i].src;
      r->F1 = t; r->F2 = minf ? -1 : (int64_t)(M - qb); r->X = X; r->Y = Y;
      status = ORC_REACHED;
      break;
    }
    /* pass 2: relabel */
    for (int64_t i = 0; i < nt; ++i) best_q[touched[i]] = qstar[touched[i]];
    /* pass 3: send the new water to every neighbour it can improve */
    for (int64_t i = 0; i < nt; ++i) {
      uint32_t v = touched[i];
      int32_t q = best_q[v];
      qstar[v] = 0;
      int c = neighbours(&g, v, u, f1, f2);
      for (int j = 0; j < c; ++j) {
        int32_t nq = q - (minf ? 0 : f2[j]);
        if (nq > 0 && nq > best_q[u[j]]) {
          if (evec_push(&bucket[(t + f1[j]) % NBUCKET], (uint32_t)u[j], nq, v)) { status = ORC_ENOMEM; goto done; }
          ++pending;
        }
      }
    }
    E->n = 0;
  }
done:
  r->status = status;
  r->work = work;
  r->cycles = cycles;
  r->t_reached = t;
  for (int i = 0; i < NBUCKET; ++i) free(bucket[i].a);
  free(best_q); free(qstar); free(touched);
  return status;
}

/* ------------------------------------------------------------------------- */
/* Tier 3: Dijkstra with lexicographic edge keys.                            */
/* mode 0: (f1, f2) — the constrained optimum when M >= F2_lex + 1 (P4);     */
/* mode 1: (f2, f1) — the constrained optimum when M = F2_min + 1 (P4);      */
/* mode 2: f1 only — M = infinity, first passage.           */
/* ------------------------------------------------------------------------- */

int orc_lex(const orc_problem* p, int mode, orc_result* r) {
  memset(r, 0, sizeof(*r));
  if (check_problem(p) || mode < 0 || mode > 2) return (int)(r->status = ORC_EINVAL);
  grid g;
  grid_init(&g, p);
  const int64_t N = g.N;
  int64_t* d1 = (int64_t*)malloc((size_t)N * sizeof(int64_t));
  int64_t* d2 = (int64_t*)malloc((size_t)N * sizeof(int64_t));
  if (!d1 || !d2) { free(d1); free(d2); return (int)(r->status = ORC_ENOMEM); }
  for (int64_t i = 0; i < N; ++i) { d1[i] = INF64; d2[i] = INF64; }
  heap h = {0};
  for (int64_t a = 0; a < N; ++a)
    if (inA(&g, a)) { d1[a] = 0; d2[a] = 0; heap_push(&h, 0, 0, a); }
  int64_t u[8];
  int f1[8], f2[8];
  while (h.n > 0) {
    hitem it = heap_pop(&h);
    if (it.k1 != d1[it.id] || it.k2 != d2[it.id]) continue;
    int64_t v = it.id;
    if (inB(&g, v)) continue;
    int c = neighbours(&g, v, u, f1, f2);
    for (int i = 0; i < c; ++i) {
      int64_t w1 = mode == 1 ? f2[i] : f1[i];
      int64_t w2 = mode == 0 ? f2[i] : (mode == 1 ? f1[i] : 0);
      int64_t a1 = it.k1 + w1, a2 = it.k2 + w2;
      if (a1 < d1[u[i]] || (a1 == d1[u[i]] && a2 < d2[u[i]])) {
        d1[u[i]] = a1; d2[u[i]] = a2;
        heap_push(&h, a1, a2, u[i]);
      }
    }
  }
  free(h.a);
  int64_t X = -1;
  for (int64_t b = 0; b < N; ++b) {
    if (!inB(&g, b) || d1[b] == INF64) continue;
    if (X < 0 || d1[b] < d1[X] || (d1[b] == d1[X] && d2[b] < d2[X])) X = b;
  }
  if (X < 0) {
    free(d1); free(d2);
    r->status = ORC_INFEASIBLE;
    return ORC_INFEASIBLE;
  }
  int64_t Y = INF64;
  int c = neighbours(&g, X, u, f1, f2);
  for (int i = 0; i < c; ++i) {
    if (inB(&g, u[i]) || d1[u[i]] == INF64) continue;
    int64_t w1 = mode == 1 ? f2[i] : f1[i];
    int64_t w2 = mode == 0 ? f2[i] : (mode == 1 ? f1[i] : 0);
    if (d1[u[i]] + w1 == d1[X] && d2[u[i]] + w2 == d2[X] && u[i] < Y) Y = u[i];
  }
  r->status = ORC_REACHED;
  r->X = X; r->Y = Y;
  if (mode == 0) { r->F1 = d1[X]; r->F2 = d2[X]; }
  else if (mode == 1) { r->F1 = d2[X]; r->F2 = d1[X]; }
  else { r->F1 = d1[X]; r->F2 = -1; }
  free(d1); free(d2);
  return ORC_REACHED;
}

/* ------------------------------------------------------------------------- */
/* Tier 4: every simple path from every a in A; each time the path reaches a */
/* B vertex it is a candidate A->B path.  Keep the         */
/* lexicographic minimum of (F1, F2, X, Y) among those with F2 < M.          */
/* ------------------------------------------------------------------------- */

typedef struct {
  const grid* g;
  int64_t M;
  uint8_t* on_path;
  int64_t best[4];
  int found;
} brute_ctx;

static void brute_dfs(brute_ctx* c, int64_t v, int64_t prev, int64_t F1, int64_t F2) {
  if (c->M != ORC_M_INF && F2 >= c->M) return;
  if (prev >= 0 && inB(c->g, v)) {
    int64_t cand[4] = {F1, c->M == ORC_M_INF ? -1 : F2, v, prev};
    int better = !c->found;
    for (int i = 0; i < 4 && !better; ++i) {
      if (cand[i] < c->best[i]) { better = 1; break; }
      if (cand[i] > c->best[i]) break;
    }
    if (better) { memcpy(c->best, cand, sizeof(cand)); c->found = 1; }
  }
  int64_t u[8];
  int f1[8], f2[8];
  int n = neighbours(c->g, v, u, f1, f2);
  c->on_path[v] = 1;
  for (int i = 0; i < n; ++i)
    if (!c->on_path[u[i]]) brute_dfs(c, u[i], v, F1 + f1[i], F2 + f2[i]);
  c->on_path[v] = 0;
}

int orc_brute(const orc_problem* p, orc_result* r) {
  memset(r, 0, sizeof(*r));
  if (check_problem(p)) return (int)(r->status = ORC_EINVAL);
  grid g;
  grid_init(&g, p);
  if (g.N > 24) return (int)(r->status = ORC_ELIMIT);
  brute_ctx c = {&g, p->M, (uint8_t*)calloc((size_t)g.N, 1), {0, 0, 0, 0}, 0};
  for (int64_t a = 0; a < g.N; ++a)
    if (inA(&g, a)) brute_dfs(&c, a, -1, 0, 0);
  free(c.on_path);
  if (!c.found) return (int)(r->status = ORC_INFEASIBLE);
  r->status = ORC_REACHED;
  r->F1 = c.best[0]; r->F2 = c.best[1]; r->X = c.best[2]; r->Y = c.best[3];
  return ORC_REACHED;
}

/* ------------------------------------------------------------------------- */

int orc_validate_path(const orc_problem* p, const int64_t* path, int64_t len, int64_t* F1, int64_t* F2) {
  if (check_problem(p) || len < 2) return ORC_EINVAL;
  grid g;
  grid_init(&g, p);
  for (int64_t i = 0; i < len; ++i)
    if (path[i] < 0 || path[i] >= g.N || !is_present(&g, path[i])) return ORC_EINVAL;
  if (!inA(&g, path[0]) || !inB(&g, path[len - 1])) return ORC_EINVAL;
  int64_t s1 = 0, s2 = 0, u[8];
  int f1[8], f2[8];
  for (int64_t i = 0; i + 1 < len; ++i) {
    int n = neighbours(&g, path[i], u, f1, f2), hit = -1;
    for (int j = 0; j < n; ++j) if (u[j] == path[i + 1]) hit = j;
    if (hit < 0) return ORC_EINVAL;
    s1 += f1[hit];
    s2 += f2[hit];
  }
  *F1 = s1;
  *F2 = s2;
  if (p->M != ORC_M_INF && s2 >= p->M) return ORC_INFEASIBLE;
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Tier 5: the nine-step cycle of PAPER.md §4, one vertex / edge at a time.  */
/* State: label L(v), the residual time of each half-edge     */
/* (v, j) that carries v's water (the active edges; 0 = idle),  */
/* the phantom edges (src, lane, quality, residual), the  */
/* temporary labels of this cycle and the triggered set.      */
/* ------------------------------------------------------------------------- */

typedef struct { int64_t src; int lane; int32_t cand; int32_t res; } phantom;

static void log_event(orc_event* ev, int64_t cap, int64_t* n, int64_t t, int64_t kind, int64_t v,
                      int64_t u, int64_t label) {
  if (ev && *n < cap) { ev[*n].t = t; ev[*n].kind = kind; ev[*n].v = v; ev[*n].u = u; ev[*n].label = label; }
  if (ev) ++*n;
}

int orc_model(const orc_problem* p, int unit, orc_result* r, orc_counters* cnt,
              orc_event* ev, int64_t ev_cap, int64_t* n_ev) {
  int64_t nev_ = 0;
  if (!n_ev) n_ev = &nev_;
  *n_ev = 0;
  memset(r, 0, sizeof(*r));
  memset(cnt, 0, sizeof(*cnt));
  if (check_problem(p)) return (int)(r->status = ORC_EINVAL);
  grid g;
  grid_init(&g, p);
  const int64_t N = g.N;
  const int NL = 2 * p->d;
  const int minf = p->M == ORC_M_INF;
  const int32_t M = minf ? 1 : (int32_t)p->M;
  int32_t* L = (int32_t*)calloc((size_t)N, sizeof(int32_t));
  int32_t* temp = (int32_t*)calloc((size_t)N, sizeof(int32_t));
  uint8_t* trig = (uint8_t*)calloc((size_t)N, 1);
  int32_t* res = (int32_t*)calloc((size_t)N * NL, sizeof(int32_t));
  int64_t* tlist = (int64_t*)malloc((size_t)N * sizeof(int64_t));
  phantom* ph = NULL;
  int64_t nph = 0, cph = 0, t = 0;
  if (!L || !temp || !trig || !res || !tlist) { r->status = ORC_ENOMEM; goto out; }

  /* lane j of v: 2k -> v + e_k, 2k+1 -> v - e_k; its (f1, f2), or f1 = 0 if absent */
#define LANE(v, j, U, F1, F2)                                                              \
  do {                                                                                     \
    const int k_ = (j) / 2;                                                                \
    const int64_t xk_ = ((v) / g.stride[k_]) % g.n[k_];                                    \
    F1 = 0; F2 = 0; U = -1;                                                                \
    if (((j) & 1) == 0 && xk_ + 1 < g.n[k_]) {                                             \
      U = (v) + g.stride[k_]; F1 = p->f1[k_ * N + (v)]; F2 = p->f2[k_ * N + (v)];          \
    } else if (((j) & 1) == 1 && xk_ > 0) {                                                \
      U = (v) - g.stride[k_]; F1 = p->f1[k_ * N + U]; F2 = p->f2[k_ * N + U];              \
    }                                                                                      \
    if (U >= 0 && (!is_present(&g, (v)) || !is_present(&g, U))) F1 = 0;                   \
    if (minf) F2 = 0;                                                                      \
  } while (0)

  /* Steps 4, 5 and 8.1 for the triggered vertices in tlist[0..nt) */
  int64_t nt = 0;
  /* initial state: A triggered with temporary label M (reading R20) */
  for (int64_t a = 0; a < N; ++a)
    if (inA(&g, a) && !inB(&g, a)) { temp[a] = M; trig[a] = 1; tlist[nt++] = a; }
  for (;;) {
    /* ---- treat the triggered vertices (skipped in the terminating cycle) ---- */
    for (int64_t i = 0; i < nt; ++i) {
      const int64_t q = tlist[i];
      const int32_t lstar = temp[q];
      if (!(lstar > L[q])) continue;
      cnt->triggered++;
      int inactive = 1;                                   /* no live edge left (reading R6) */
      for (int j = 0; j < NL; ++j) if (res[q * NL + j] > 0) inactive = 0;
      for (int j = 0; j < NL; ++j) {
        int64_t u; int a1, a2;
        LANE(q, j, u, a1, a2);
        if (a1 == 0) continue;
        const int32_t c = lstar - a2;
        const int32_t tu = trig[u] ? temp[u] : 0;        /* this cycle's temporary label only */
        const int32_t lu = L[u] > tu ? L[u] : tu;
        if (!(c > 0 && c > lu)) continue;                /* edge j triggered */
        if (inactive) {                                  /* restart with time f1 */
          res[q * NL + j] = a1;
          cnt->started++;
        } else {                                         /* phantom */
          if (nph == cph) {
            cph = cph ? 2 * cph : 1024;
            phantom* np = (phantom*)realloc(ph, (size_t)cph * sizeof(phantom));
            if (!np) { r->status = ORC_ENOMEM; goto out; }
            ph = np;
          }
          ph[nph].src = q; ph[nph].lane = j; ph[nph].cand = c; ph[nph].res = a1;
          ++nph;
          cnt->created++;
          log_event(ev, ev_cap, n_ev, t, 1, q, u, lstar);
        }
      }
      if (inactive) {                                    /* Step 8.1: relabel */
        L[q] = lstar;
        cnt->relabels++;
        log_event(ev, ev_cap, n_ev, t, 0, q, -1, lstar);
      }
    }
    for (int64_t i = 0; i < nt; ++i) { trig[tlist[i]] = 0; temp[tlist[i]] = 0; }
    nt = 0;
    /* ---- Step 6, 2°: nothing live -> infeasible ---- */
    int64_t live_e = 0, active_v = 0;
    int32_t dmin = INT32_MAX;
    for (int64_t v = 0; v < N; ++v) {
      int act = 0;
      for (int j = 0; j < NL; ++j) {
        const int32_t rr = res[v * NL + j];
        if (rr > 0) { ++live_e; act = 1; if (rr < dmin) dmin = rr; }
      }
      active_v += act;                                   /* active vertex */
    }
    for (int64_t i = 0; i < nph; ++i) if (ph[i].res < dmin) dmin = ph[i].res;
    if (live_e + nph == 0) { r->status = ORC_INFEASIBLE; break; }
    /* ---- Step 1: advance time (jump by the min residual) ---- */
    const int32_t delta = unit ? 1 : dmin;
    t += delta;
    cnt->cycles++;
    cnt->work += live_e + nph;
    log_event(ev, ev_cap, n_ev, t, 2, active_v, live_e, nph);
    /* ---- Steps 1-3: edges and phantoms reaching 0 deliver their water ---- */
    int32_t bq = 0;
    int64_t bx = -1, by = -1;
    /* at B: keep the lexicographic best (quality desc, X asc, source asc), reading R5 */
#define ARRIVE(D, CAND, SRC)                                                             \
    do {                                                                                 \
      const int64_t d_ = (D); const int32_t c_ = (CAND); const int64_t s_ = (SRC);       \
      if (c_ > 0) {                                                                      \
        if (inB(&g, d_)) {                         /* 1°: a vertex of B */ \
          if (c_ > bq || (c_ == bq && d_ < bx)) { bq = c_; bx = d_; by = s_; }           \
          else if (c_ == bq && d_ == bx && s_ < by) by = s_;                             \
        } else if (c_ > L[d_]) {                   /* PAPER.md:32 */                     \
          if (!trig[d_]) { trig[d_] = 1; tlist[nt++] = d_; temp[d_] = c_; }              \
          else if (c_ > temp[d_]) temp[d_] = c_;                                         \
        }                                                                                \
      }                                                                                  \
    } while (0)
    for (int64_t v = 0; v < N; ++v) {
      for (int j = 0; j < NL; ++j) {
        int32_t* rr = &res[v * NL + j];
        if (*rr <= 0) continue;
        *rr -= delta;
        if (*rr == 0) {
          int64_t u; int a1, a2;
          LANE(v, j, u, a1, a2);
          (void)a1;
          cnt->arrivals++;
          ARRIVE(u, L[v] - a2, v);
        }
      }
    }
    int64_t keep = 0;
    for (int64_t i = 0; i < nph; ++i) {
      ph[i].res -= delta;
      if (ph[i].res == 0) {
        int64_t u; int a1, a2;
        LANE(ph[i].src, ph[i].lane, u, a1, a2);
        (void)a1; (void)a2;
        cnt->arrivals++;
        ARRIVE(u, ph[i].cand, ph[i].src);
      } else {
        ph[keep++] = ph[i];                             /* Step 7 */
      }
    }
    if (bx >= 0) {                                       /* terminate in this cycle (R17) */
      r->status = ORC_REACHED;
      r->F1 = t; r->F2 = minf ? -1 : M - bq; r->X = bx; r->Y = by;
      break;
    }
    nph = keep;
  }
#undef ARRIVE
#undef LANE
out:
  r->work = cnt->work;
  r->cycles = cnt->cycles;
  r->t_reached = t;
  free(L); free(temp); free(trig); free(res); free(tlist); free(ph);
  return (int)r->status;
}
