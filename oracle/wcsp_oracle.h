/* wcsp_oracle.h — CPU oracle for the weight-constrained shortest path on Z^d.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_1511_06441_b200/csrc/), and the CUDA path never calls it.
 *
 * Problem (§1): G = subgraph of Z^d, f = (f1, f2) : E -> Z_+^2,
 * A, B disjoint vertex sets, budget M.  Among all A->B paths pi with
 * F2(pi) < M (strict) find the one minimising F1(pi).
 * Tie-break (reading R5): the result is the lexicographic
 * minimum of (F1, F2, X, Y) over all such paths, X = endpoint in B, Y = the
 * vertex before X.
 *
 * Encoding: N = prod(shape), v = x0 + n0*(x1 + n1*(...)); f1[k*N + v],
 * f2[k*N + v] are the values of edge (v, v+e_k); f1 == 0 means absent.
 * present == NULL means every vertex is present.  M == ORC_M_INF (-1) is the
 * unconstrained first-passage case.
 */
#ifndef WCSP_ORACLE_H
#define WCSP_ORACLE_H
#include <stdint.h>

#define ORC_M_INF (-1)

enum { ORC_REACHED = 0, ORC_INFEASIBLE = 1, ORC_EINVAL = 2, ORC_ELIMIT = 3, ORC_ENOMEM = 4 };

typedef struct {
  int32_t d;
  int64_t shape[4];
  const uint8_t *f1, *f2;          /* [d][N] */
  const uint8_t *maskA, *maskB;    /* [N] */
  const uint8_t *present;          /* [N] or NULL */
  int64_t M;
} orc_problem;

typedef struct {
  int64_t status;                  /* ORC_* */
  int64_t F1, F2, X, Y;            /* F2 = -1 when M = ORC_M_INF */
  int64_t work;                    /* tier 2 only: sum over event times of flows in flight */
  int64_t cycles;                  /* tier 2 only: number of event times processed */
  int64_t t_reached;               /* tier 2 only: last time processed */
} orc_result;

/* Tier 1: Dijkstra on the product graph (vertex, spent weight s in [0, M-1]). */
int orc_dense(const orc_problem* p, orc_result* r);
/* Tier 2: time-ordered label setting on (vertex, remaining quality); t_limit > 0
 * stops after that simulated time with status ORC_ELIMIT (bounded CPU sample). */
int orc_pruned(const orc_problem* p, int64_t t_limit, orc_result* r);
/* Tier 3: Dijkstra with lexicographic keys.  mode 0: (f1, f2); mode 1: (f2, f1);
 * mode 2: f1 only (M = infinity).  Ignores p->M. */
int orc_lex(const orc_problem* p, int mode, orc_result* r);
/* Tier 4: exhaustive simple-path enumeration (tiny graphs only, N <= 24). */
int orc_brute(const orc_problem* p, orc_result* r);
/* Tier 5: the paper's cycle simulated step by step, sequentially (§4,
 * :155-227, in the SURVEY §8(a) canonical form: 'post' activeness R6, no twin
 * demotion R8, no eager kill R7, jump or unit time R4).  Outputs as tier 1; it
 * also counts the method's work: cycles, sum over cycles of live edges + live
 * phantoms (work), arrivals (edges/phantoms whose time reached 0), triggered
 * vertices (accepted first arrivals), phantoms created, lanes started,
 * relabels.  unit = 1: advance by 1; 0: by the min residual. */
typedef struct {
  int64_t cycles, work, arrivals, triggered, created, started, relabels;
} orc_counters;
/* Optional event log (ev may be NULL): kind 0 = relabel of v to `label` at t
 * (Step 8.1), kind 1 = phantom created at t by v toward u carrying the label
 * `label` = L* of v (Step 5; the water it delivers is label - f2),
 * kind 2 = a cycle advancing to t: v = active vertices (>= 1 live edge) and
 * u = live edges at its top, label = live phantoms. */
typedef struct { int64_t t, kind, v, u, label; } orc_event;
int orc_model(const orc_problem* p, int unit, orc_result* r, orc_counters* cnt,
              orc_event* ev, int64_t ev_cap, int64_t* n_ev);
/* Path check (PAPER.md:13-18 definitions of path, F1, F2). Returns 0 if path is
 * an A->B path over present edges with F2 < M; writes F1, F2. */
int orc_validate_path(const orc_problem* p, const int64_t* path, int64_t len, int64_t* F1, int64_t* F2);

#endif
