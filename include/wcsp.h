/* wcsp.h — C-ABI of the B200 (sm_100a) active-vertex label-correcting sweep
 * for the weight-constrained shortest path on subgraphs of Z^d (d = 1..4).
 *
 * The problem (§1): G(V, E) a subgraph of Z^d, f : E -> Z_+^2
 * with f1(e) the passage time and f2(e) the weight of e; A, B disjoint vertex
 * sets; a budget M.  Among all A->B paths pi with F2(pi) < M (strict,
 * PAPER.md:21; reading R1 in DESIGN.md) find pi^ minimising F1(pi).  The
 * output is F1(pi^) plus "the vertex X in B that is the endpoint of pi^, the
 * last edge x on the path pi^, and the value F2(pi^)", with
 * ties broken lexicographically on (F1, F2, X, Y), X and Y linear indices
 * (reading R5).  The path itself is recovered by repeated solves on
 * G'(V', E') (corrected as reading R12), see wcsp_reconstruct.
 *
 * The solve is the paper's per-unit-time cycle (§4, :155-227): water
 * of quality M leaves A; every cycle advances the clock by the
 * minimum live residual, counts down the active and phantom
 * edges, triggers the destinations of the edges that reach 0, corrects labels
 * (relabel + activate inactive vertices, phantom edges out of active ones,
 * PAPER.md:32), retires vertices with no live edge, and stops at the first
 * arrival at B (termination 1°) or when nothing is live (2°,
 * PAPER.md:126).  Every step runs in the library's CUDA kernels; there is no
 * CPU fallback (a missing or failing device returns WCSP_ECUDA).
 *
 * Encoding.  N = prod(shape) <= 2^30; vertex v = x0 + n0*(x1 + n1*(x2 + ...))
 * (x0 fastest).  f1[k*N + v], f2[k*N + v] (uint8) are f1, f2 of the edge
 * (v, v + e_k); f1 == 0 means "edge absent" (the subgraph of Z^d), values at
 * x_k = n_k - 1 are ignored.  maskA, maskB: uint8 [N], nonzero = member.
 * present: uint8 [N] or NULL; a vertex with present[v] == 0 is removed from
 * G with all its edges (G' of PAPER.md:25).
 *
 * Ownership.  The caller owns every input array; inputs are read-only and may
 * be freed once the call that takes them returns.  The handle owns all device
 * state until wcsp_destroy.  `path`/`trace` outputs are caller-allocated.
 *
 * Errors.  Every call returns a wcsp_status; no exception crosses the ABI; on
 * error the output structs are left untouched and wcsp_last_error() returns a
 * thread-local message naming the offending input.
 */
#ifndef WCSP_H
#define WCSP_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  WCSP_REACHED = 0,     /* termination 1°: a vertex of B was reached */
  WCSP_INFEASIBLE = 1,  /* termination 2°: no live edge left, no path with F2 < M */
  WCSP_EINVAL = 2,      /* invalid input (validation rules below) */
  WCSP_EMISMATCH = 3,   /* reconstruction: a re-solve on G' disagreed with the first solve */
  WCSP_EBUDGET = 4,     /* options.cycle_budget exceeded */
  WCSP_ENOMEM = 5,      /* device allocation failed */
  WCSP_ECUDA = 6,       /* CUDA error (message in wcsp_last_error) */
  WCSP_ENCCL = 7,       /* reserved: multi-GPU slab exchange */
  WCSP_EOVERFLOW = 8    /* phantom pool overflow after the automatic retries */
} wcsp_status;

#define WCSP_M_INF (-1)           /* M = +infinity: first passage */
#define WCSP_M_MAX 65533          /* largest M of the 16-bit label layout, the fast default */
#define WCSP_M_MAX_WIDE 2147483646LL   /* largest finite M: budgets in (WCSP_M_MAX, WCSP_M_MAX_WIDE] are not
                                     an error ("M in R+"; integer f2 makes ceil(M) equivalent) —
                                     they switch the solve to 32-bit labels and 64-bit stamped temporary
                                     labels, on the sweep engine (WCSP_ENGINE_PERSISTENT / _STEPPED; a
                                     wheel-engine handle runs its sweep form for that solve), single device
                                     only (slab handles and wcsp_staircase return WCSP_EINVAL) */

enum { WCSP_MEM_HOST = 0, WCSP_MEM_DEVICE = 1 };
enum { WCSP_JUMP = 0,             /* advance t by the min live residual */
       WCSP_UNIT = 1 };           /* advance t by 1 — identical outputs */
enum { WCSP_ENGINE_PERSISTENT = 0,   /* sweep engine: residual countdown on the active list + phantom pool
                                        (PAPER.md:157, :173), one cooperative kernel runs every cycle */
       WCSP_ENGINE_STEPPED = 1,      /* sweep engine, one kernel per phase, host polls termination */
       WCSP_ENGINE_WHEEL = 2,        /* timing-wheel engine: live edges stored by arrival time, written
                                        once and read once (same outputs and counters), persistent */
       WCSP_ENGINE_WHEEL_STEPPED = 3 };
enum { WCSP_HALO_COPY = 0,          /* slab boundary: ghost planes exchanged by copies / NCCL per cycle */
       WCSP_HALO_PEER = 1 };        /* slab boundary: fused into the cycle kernel over peer memory (f2) */

/* Problem statement.  Validation (wcsp_create / wcsp_load):
 *  d in 1..4, every shape[k] >= 1, N <= 2^30;  A and B non-empty among the
 *  present vertices and disjoint;  M == WCSP_M_INF or
 *  1 <= M <= WCSP_M_MAX_WIDE;  every present edge (f1 > 0) has f2 >= 1
 *  (f : E -> Z_+^2).  Violations return WCSP_EINVAL. */
typedef struct {
  int32_t d;
  int64_t shape[4];
  const uint8_t* f1;        /* [d][N] passage times, 0 = absent edge */
  const uint8_t* f2;        /* [d][N] weights */
  const uint8_t* maskA;     /* [N] sources: "vertices in A have label M" */
  const uint8_t* maskB;     /* [N] targets */
  const uint8_t* present;   /* [N] or NULL (all present) */
  int64_t M;                /* budget, strict F2 < M, or WCSP_M_INF */
  int32_t mem;              /* WCSP_MEM_HOST: host arrays (copied); WCSP_MEM_DEVICE: device
                               pointers, read on options.stream during the call */
} wcsp_problem;

typedef struct {
  int32_t time_mode;        /* WCSP_JUMP (default) | WCSP_UNIT */
  int32_t engine;           /* WCSP_ENGINE_* (default 0 = sweep, persistent) */
  int32_t demote_twin;      /* reserved (twin re-sourcing): must be 0 in this version */
  int32_t device;           /* CUDA device ordinal */
  int64_t cycle_budget;     /* 0 = unlimited; else WCSP_EBUDGET after that many cycles */
  int64_t phantom_capacity; /* sweep: phantom records per pool buffer; wheel: event-ring slots;
                               0 = auto (4N, min 2^20); grown automatically on overflow */
  int64_t trace_cap;        /* per-cycle trace records kept (0 = off) */
  void* stream;             /* cudaStream_t or NULL (the library creates one) */
  int32_t slabs;            /* > 1: slab engine on this device — the grid is cut along its last axis
                               into `slabs` slabs with ghost planes that exchange the water crossing
                               a slab boundary every cycle (the multi-GPU layout run
                               on one GPU); requires engine WHEEL and host arrays.  0/1 = off. */
  int32_t halo;             /* how slabs exchange their boundary (slabs > 1 or nranks > 1):
                               WCSP_HALO_COPY (0, default): ghost planes, one copy / ncclSend-Recv
                               of boundary water and labels per cycle, host-driven per-phase
                               kernels; WCSP_HALO_PEER (1): SURVEY §8(f) f2 — one persistent
                               cooperative kernel per device in which water crossing a slab
                               boundary is a system-scope atomicMax into the neighbour's state
                               word and the Step-4 test reads the neighbour's label
                               in place (NVLink peer memory via CUDA IPC across GPUs; with
                               nranks > 1 every rank's GPU must have peer access to its
                               neighbours').  Outputs and work counters equal the single-device
                               run's.  At most 8 virtual slabs. */
  int32_t nranks;           /* > 1: multi-GPU slab engine — this process owns slab `rank` of `nranks`
                               (one process per GPU); the slabs exchange boundary water and labels
                               with ncclSend/ncclRecv and combine the cycle decision with one
                               ncclAllReduce(max) per cycle.  Every rank passes the whole problem
                               (host arrays) and the same nccl_id. */
  int32_t rank;
  const uint8_t* nccl_id;   /* 128 bytes from wcsp_nccl_unique_id() on one rank, shared with all;
                               non-NULL with nranks = 1 runs the NCCL path on one GPU */
  int32_t local_slab;       /* multi-GPU only (nccl_id set): 1 = the problem's arrays hold ONLY this
                               rank's planes [p0, p1) of the last axis (wcsp_slab_planes: its slab
                               plus one ghost plane per neighbour), laid out as the whole-grid arrays
                               with N replaced by (p1 - p0) * plane; problem.shape stays the global
                               shape; host or device memory.  Each rank validates its own planes and
                               the counts are combined over NCCL, so no rank ever holds (or scans)
                               the whole grid — a 1024^3 cube over 8 GPUs.  0 = every
                               rank passes the whole problem (host arrays). */
} wcsp_options;

typedef struct {
  int64_t F1;               /* t at termination 1° = F1(pi^) */
  int64_t F2;               /* M - L(X); -1 when M = WCSP_M_INF */
  int64_t X;                /* endpoint of pi^ in B (smallest index among ties) */
  int64_t Y;                /* second-to-last vertex of pi^: the other endpoint of x, or the
                               origin of the phantom that delivered it (the copy set C) */
  int32_t x_lane;           /* lane of X toward Y: 2k = +e_k, 2k+1 = -e_k */
  int32_t via_phantom;      /* 1 if the arrival at X was carried only by a phantom edge */
  int64_t cycles;           /* cycles executed (time jumps) */
  int64_t edge_updates;     /* sum over cycles of (live active edges + live phantom edges) */
  int64_t arrivals;         /* edges/phantoms whose residual reached 0 */
  int64_t triggered;        /* sum over cycles of triggered vertices */
  int64_t phantoms_created;
  int64_t relabels;
  int64_t lanes_started;    /* active edges (re)started by inactive triggered vertices */
  int64_t peak_active;      /* max active-vertex list size (sweep engines) */
  int64_t peak_phantoms;    /* sweep: max live phantoms; wheel: max live edges + phantoms */
  int64_t phantom_capacity; /* pool capacity used by the successful run */
  int64_t kernel_launches;  /* CUDA kernels this solve launched */
  double device_ms;         /* device time of the solve (init + cycles), CUDA events */
  double cycle_ms;          /* device time of the cycle kernels alone (excludes the init kernel) */
  int64_t retries;          /* grow-and-rerun attempts after a device-side storage overflow (phantom
                               pool, event ring, run-descriptor table) */
  int64_t staging_appended; /* wheel treat: events past the shared-memory staging appended to the
                               block's open ring regions ... */
  int64_t staging_spilled;  /* ... past those, written to the block's spill buffer ... */
  int64_t staging_singles;  /* ... past the spill buffer, filed as runs of one (all exact; counted so
                               tests can show every path ran) */
} wcsp_result;

/* One record per cycle when options.trace_cap > 0 (after the cycle ran). */
typedef struct {
  int64_t t, delta;
  int64_t active_vertices;  /* entries of the active-vertex list swept this cycle */
  int64_t live_lanes;       /* E: live active edges at the top of the cycle */
  int64_t phantoms;         /* P: live phantoms at the top of the cycle */
  int64_t triggered;        /* T: vertices triggered this cycle */
  int64_t arrivals;         /* R */
  int64_t created;          /* phantoms created */
  int64_t relabels;
  int64_t tested;           /* triggered-bitmap entries examined by the treat phase */
  int64_t ns_arrive;        /* device ns of the arrival phase (sweep / fire) incl. its grid barrier */
  int64_t ns_treat;         /* device ns of the treat phase incl. its grid barrier */
  int64_t ns_arrive_spread; /* wheel persistent: last minus first block to finish the arrival phase */
  int64_t ns_treat_spread;  /* ... the treat phase (load imbalance) */
} wcsp_trace_rec;

typedef struct wcsp_handle wcsp_handle;

/* Allocate device state for the problem's shape and load it (validates). */
wcsp_status wcsp_create(const wcsp_problem* problem, const wcsp_options* options, wcsp_handle** out);
/* Re-load f1, f2, A, B, present, M into an existing handle of the same d/shape. */
wcsp_status wcsp_load(wcsp_handle* h, const wcsp_problem* problem);
/* Run the sweep on the loaded problem. Returns WCSP_REACHED / WCSP_INFEASIBLE or an error. */
wcsp_status wcsp_solve(wcsp_handle* h, wcsp_result* result);
/* Replace B (maskB != NULL), the present set (present != NULL; all present if
 * present_all) and M for subsequent solves.  Arrays follow `mem`. */
wcsp_status wcsp_set_targets(wcsp_handle* h, const uint8_t* maskB, const uint8_t* present,
                             int32_t present_all, int64_t M, int32_t mem);
/* Full path pi^ = (v_1 in A, ..., v_k = X in B) by repeated solves on G'
 * (reading R12: B' = {Y}, V' = V \ (B u earlier targets),
 * M' = F2 - f2(x) + 1).  Each re-solve must return (F1 - f1(x), F2 - f2(x)),
 * else WCSP_EMISMATCH.  path has room for cap vertices; if cap is too small
 * returns WCSP_EINVAL with *len = the required length.  Restores the loaded
 * problem's B/present/M afterwards.  result = the first solve's result. */
wcsp_status wcsp_reconstruct(wcsp_handle* h, int64_t* path, int64_t cap, int64_t* len, wcsp_result* result);
/* Copy the last solve's trace (host memory). */
wcsp_status wcsp_trace(wcsp_handle* h, wcsp_trace_rec* out, int64_t cap, int64_t* n);
/* Host-side path check: path over present edges from A to B;
 * writes F1, F2.  Returns 0 if valid with F2 < M, WCSP_INFEASIBLE if F2 >= M,
 * WCSP_EINVAL otherwise.  Host arrays only. */
wcsp_status wcsp_validate_path(const wcsp_problem* problem, const int64_t* path, int64_t len,
                               int64_t* F1, int64_t* F2);
/* The whole F1*(M) staircase in one run (PAPER.md:21 for every
 * budget at once): run with M = M_max past the first arrival at B and record every
 * arrival that beats all earlier ones — step i = (F1_i, F2_i, X_i, Y_i), F1 increasing,
 * F2 decreasing.  The constrained optimum for any budget M <= M_max is the first step
 * with F2_i < M (infeasible if none).  The run ends when nothing is live or a step
 * reaches F2 <= f2_stop.  steps: caller-allocated [cap][4]; *n = number of steps (may
 * exceed cap).  Wheel engine, single device.  Returns WCSP_REACHED if a step exists,
 * else WCSP_INFEASIBLE; result = the last step's solve record. */
wcsp_status wcsp_staircase(wcsp_handle* h, int64_t M_max, int64_t f2_stop, int64_t* steps, int64_t cap,
                           int64_t* n, wcsp_result* result);
/* Seeded synthetic instances generated in device memory (DESIGN.md §4 recipe; the same pure
 * function as the host generator paper_1511_06441_b200/instances.py, so a rank can build only
 * its own slab of a large cube in HBM).  Not part of the method: input preparation only.
 * wcsp_generate_grid: f1, f2 of the planes [z0, z1) of the LAST axis of `shape` (z1 < 0: to the
 * end), written as f1[k * Nl + i] (Nl = (z1 - z0) * plane, i = global index - z0 * plane):
 * value = lo + ((h >> 32) mod (hi - lo + 1)), h = sm(sm(seed) ^ (8v + 2k + c)), c = 0 for f1 and
 * 1 for f2, sm = the splitmix64 finaliser of x + 0x9E3779B97F4A7C15; 0 where x_k = n_k - 1.
 * 1 <= lo <= hi <= 255.  f1, f2: device buffers of d * Nl bytes, written on `stream` (asynchronous).
 * wcsp_generate_mask: out[i] = 1 if the vertex belongs to the set `rule` (below), else 0.
 * Errors: WCSP_EINVAL for a bad shape / range / rule / NULL pointer, WCSP_ECUDA on a launch error. */
enum { WCSP_SET_FACE0 = 0,        /* x0 = 0 (A of the face-to-face configs) */
       WCSP_SET_FACE1 = 1,        /* x0 = n0 - 1 (their B) */
       WCSP_SET_BOUNDARY = 2,     /* any x_k in {0, n_k - 1}: water on the boundary */
       WCSP_SET_CENTRE = 3,       /* floor(n_k / 2) on every axis (reading R18) */
       WCSP_SET_CORNER0 = 4,      /* v = 0 */
       WCSP_SET_CORNER1 = 5 };    /* v = N - 1 */
wcsp_status wcsp_generate_grid(int32_t d, const int64_t* shape, uint64_t seed, int32_t lo, int32_t hi, int64_t z0,
                               int64_t z1, uint8_t* f1, uint8_t* f2, void* stream);
wcsp_status wcsp_generate_mask(int32_t d, const int64_t* shape, int32_t rule, int64_t z0, int64_t z1, uint8_t* out,
                               void* stream);
/* The planes of the last axis a rank holds in the slab partition: slab `rank` of
 * `nranks` owns z in [out[0], out[1]) = [rank * n_last / nranks, (rank + 1) * n_last / nranks) and
 * its local arrays (options.local_slab) cover [out[2], out[3]) = the slab plus one ghost plane on
 * each side that has a neighbour.  Host-only arithmetic; WCSP_EINVAL for a bad argument. */
wcsp_status wcsp_slab_planes(int64_t n_last, int32_t nranks, int32_t rank, int64_t* out4);
/* NCCL unique id (128 bytes) for options.nccl_id; call on one rank and share it
 * (e.g. through torch.distributed).  Returns WCSP_ENCCL if NCCL cannot be loaded. */
wcsp_status wcsp_nccl_unique_id(uint8_t* out128);
void wcsp_destroy(wcsp_handle* h);
const char* wcsp_last_error(void);
/* Version string, and the number of SMs / cooperative blocks the persistent engine uses. */
const char* wcsp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* WCSP_H */
