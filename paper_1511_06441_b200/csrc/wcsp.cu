// wcsp.cu — host side of the C-ABI (include/wcsp.h): handle, validation,
// engines (sweep / timing wheel, each persistent or stepped), reconstruction.
#include "wcsp.h"
#include "wcsp_device.cuh"
#include "wcsp_wheel.cuh"
#include "wcsp_gen.cuh"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#ifndef HYB_LAG_DEFAULT
#define HYB_LAG_DEFAULT 1   // lagged-decision wheel kernel where the hybrid applies
#endif

using namespace wcspk;

namespace {

thread_local std::string g_err;

wcsp_status fail(wcsp_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CK(call)                                                                                \
  do {                                                                                          \
    cudaError_t e_ = (call);                                                                    \
    if (e_ != cudaSuccess)                                                                      \
      return fail(e_ == cudaErrorMemoryAllocation ? WCSP_ENOMEM : WCSP_ECUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                           \
  } while (0)

bool is_wheel(int engine) { return engine == WCSP_ENGINE_WHEEL || engine == WCSP_ENGINE_WHEEL_STEPPED; }
bool is_stepped(int engine) { return engine == WCSP_ENGINE_STEPPED || engine == WCSP_ENGINE_WHEEL_STEPPED; }

}  // namespace

struct wcsp_handle {
  int dev = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int d = 0;
  long long shape[4] = {1, 1, 1, 1};
  unsigned long long N = 0;
  wcsp_options opt{};
  // device buffers
  uint8_t *d_f1 = nullptr, *d_f2 = nullptr;          // staging of host inputs [d][N]
  uint8_t *d_maskA = nullptr, *d_maskB = nullptr, *d_present = nullptr;
  bool present_all = true;
  void* wt = nullptr;
  void* res = nullptr;                               // sweep engines only
  unsigned long long* sw = nullptr;                  // vertex state words (label | temp)
  unsigned* tbits = nullptr;                         // triggered bitmap
  unsigned nwords = 0;
  BArr* barr = nullptr;                              // arrivals at targets (terminating cycle)
  unsigned barr_cap = 0;
  unsigned* act[2] = {nullptr, nullptr};             // sweep engines only
  unsigned long long* pool[2] = {nullptr, nullptr};  // sweep engines only
  unsigned long long pool_cap = 0;
  unsigned long long* ev = nullptr;                  // wheel engines only
  unsigned long long ev_cap = 0;
  unsigned long long* bdesc = nullptr;
  unsigned long long* spill = nullptr;               // [grid][spill_cap] staging overflow of the treat
  unsigned* tlist = nullptr;                         // [grid * QA_CAP] triggered list of a sparse fire phase
  unsigned spill_cap = 0;
  unsigned* bcounts = nullptr;                       // bnev [256] | bnlane [256] | bndesc [256][grid]
  unsigned dcap = 0;
  int f1max = 255;
  Ctl* ctl = nullptr;
  Ctl* h_ctl = nullptr;                              // pinned
  TraceRec* trace = nullptr;
  unsigned long long* d_cnt = nullptr;               // validation counters
  long long M = 0;
  int nsm = 0, grid = 0;
  long long l2_bytes = 0;
  int grid_main = 0;                                 // grid of opt.engine's cycle kernel (grid = this solve's)
  bool big = false;                                  // wheel: the 4-blocks-per-SM cycle kernel
  // wide labels (M > WCSP_M_MAX): this solve runs the sweep engine on u32 labels + u64 temps
  int eng = 0;                                       // engine of this solve (opt.engine, or its sweep form)
  bool wide = false;
  unsigned* lab = nullptr;                           // [N] u32 labels (allocated on the first wide solve)
  int pool_rec = 8;                                  // bytes per phantom record in pool[] (16: wide)
  int grid_wide = 0;
  // one-barrier hybrid wheel kernel (k_wheel_hybrid): per-block treat progress, neighbourhood radius
  bool hyb = false;
  unsigned long long* prog = nullptr;
  int hyb_R = 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr, em = nullptr;
  long long last_cycles = 0;
  long long launches = 0;
  // slab engine: a child owns planes [z0, z1) of the last axis plus ghost planes
  int slab_index = -1;
  long long z0 = 0, z1 = 0;
  int glo = 0, ghi = 0;
  unsigned goff = 0, plane = 0, ghost_hi_start = 0;
  uint8_t* d_ghost = nullptr;                        // 1 = ghost, 2 = ghost target
  unsigned long long *g_out_lo = nullptr, *g_out_hi = nullptr, *g_in_lo = nullptr, *g_in_hi = nullptr;
  unsigned *l_out_lo = nullptr, *l_out_hi = nullptr, *l_in_lo = nullptr, *l_in_hi = nullptr;
  unsigned long long preset_nB = 0;                  // child: |B| of the whole problem (B-arrival list)
  std::vector<wcsp_handle*> children;                // parent of a virtual slab group
  Ctl** d_ctls = nullptr;                            // children's control blocks (device array)
  void* comm = nullptr;                              // ncclComm_t (multi-GPU slab engine)
  int rank = 0, nranks = 1;
  int staircase = 0;                                 // wcsp_staircase in progress
  long long f2stop = 0;
  long long* stair = nullptr;
  unsigned stair_cap = 0;
  // peer halo: one cooperative kernel, boundary fused over peer memory
  int halo = WCSP_HALO_COPY;
  unsigned peer_per = 0;                             // blocks per slab in the peer kernel
  unsigned long long* xbar = nullptr;                // [0] cross-slab barrier, [1] watchdog flag
  unsigned long long* xbar_ptr = nullptr;            // multi-GPU: rank 0's counter, mapped
  Ctl** d_pctl = nullptr;                            // multi-GPU: every rank's control block (mapped)
  std::vector<void*> ipc_opened;                     // peer allocations mapped with CUDA IPC
  unsigned long long* peer_sw[2] = {nullptr, nullptr};
  unsigned* peer_tb[2] = {nullptr, nullptr};
  unsigned peer_shift[2] = {0, 0}, peer_goff[2] = {0, 0};
};

namespace {

size_t lane_bytes(int d) { return d <= 2 ? 4 : 8; }

template <int D>
void* cycle_fn(int engine, bool big, bool wide = false) {
  if (wide) return engine == WCSP_ENGINE_STEPPED ? reinterpret_cast<void*>(&k_sweep<D, true>)
                                                 : reinterpret_cast<void*>(&k_persistent<D, true>);
  switch (engine) {
    case WCSP_ENGINE_PERSISTENT: return reinterpret_cast<void*>(&k_persistent<D>);
    case WCSP_ENGINE_STEPPED: return reinterpret_cast<void*>(&k_sweep<D>);
    case WCSP_ENGINE_WHEEL: return big ? reinterpret_cast<void*>(&k_wheel_persistent<D, 4>)
                                       : reinterpret_cast<void*>(&k_wheel_persistent<D, 3>);
    default: return reinterpret_cast<void*>(&k_wheel_treat<D>);
  }
}
void* cycle_fn_d(int d, int engine, bool big, bool wide = false) {
  return d == 1 ? cycle_fn<1>(engine, big, wide) : d == 2 ? cycle_fn<2>(engine, big, wide)
         : d == 3 ? cycle_fn<3>(engine, big, wide) : cycle_fn<4>(engine, big, wide);
}

template <int D>
cudaError_t set_smem_attrs() {
  const int bytes = (int)sizeof(Smem);
  void* fns[] = {reinterpret_cast<void*>(&k_persistent<D>), reinterpret_cast<void*>(&k_sweep<D>),
                 reinterpret_cast<void*>(&k_treat<D>), reinterpret_cast<void*>(&k_wheel_persistent<D, 3>),
                 reinterpret_cast<void*>(&k_wheel_persistent<D, 4>),
                 reinterpret_cast<void*>(&k_wheel_fire<D>), reinterpret_cast<void*>(&k_wheel_treat<D>),
                 reinterpret_cast<void*>(&k_wheel_peer<D, 3>), reinterpret_cast<void*>(&k_wheel_peer<D, 4>),
                 reinterpret_cast<void*>(&k_persistent<D, true>), reinterpret_cast<void*>(&k_sweep<D, true>),
                 reinterpret_cast<void*>(&k_treat<D, true>), reinterpret_cast<void*>(&k_wheel_hybrid<D, 3>),
                 reinterpret_cast<void*>(&k_wheel_hybrid<D, 4>), reinterpret_cast<void*>(&k_wheel_lag<D, 3>),
                 reinterpret_cast<void*>(&k_wheel_lag<D, 4>)};
  const char* co = getenv("WCSP_CARVEOUT");       // A/B runs: shared-memory carveout in percent of L1
  for (void* f : fns) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    if (co && (e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(co))) != cudaSuccess)
      return e;
  }
  return cudaSuccess;
}

// Treat window size (bitmap words per warp window).  Blocks own contiguous ranges of windows,
// so a round count just above an integer leaves most warps idle in the last round: take 16
// words when that gives at most one round or at least four (C2, C3), else 8 (C3s, P6 cubes).
// WCSP_WIN_WORDS overrides (A/B runs).
// Interleaved treat rounds (phase_treat, build option for A/B runs, WCSP_ILEAVE=1): every block's
// round r lies in one chunk of the grid so that the whole device treats and fires one L2-sized
// chunk of the front at a time.  Measured slower than contiguous block slabs on C3 and C5.
bool ileave_for(const wcsp_handle* h);

unsigned win_words_for(unsigned nwords, unsigned nblocks) {
  if (const char* e = getenv("WCSP_WIN_WORDS")) return atoi(e) >= WIN_WORDS ? (unsigned)WIN_WORDS : atoi(e) >= 16 ? 16u : 8u;
  if (nblocks == 0) return 8u;
  const double rounds16 = (double)nwords / (16.0 * nblocks * WARPS);
  return std::min<unsigned>(rounds16 <= 1.0 || rounds16 >= 4.0 ? 16u : 8u, (unsigned)WIN_WORDS);
}

bool ileave_for(const wcsp_handle* h) {
  (void)h;
  // measured slower on C3 (134 -> 161 ms: no block-local bitmap, scattered fire) and on C5 (80.5 ->
  // 80.0 / 83.5 s): off unless requested (profiles/r02/ab_ileave_*.txt)
  if (const char* e = getenv("WCSP_ILEAVE")) return atoi(e) != 0;
  return false;
}

// Fire chunk order (wheel_fire): strided = every block walks its run lists in filing order.
// WCSP_FIRE_STRIDE=0/1 overrides (A/B runs).
bool fstride_for(const wcsp_handle* h) {
  if (const char* e = getenv("WCSP_FIRE_STRIDE")) return atoi(e) != 0;
  return ileave_for(h);
}

Dev make_dev(const wcsp_handle* h) {
  Dev s{};
  s.N = (unsigned)h->N;
  s.NL = 2 * h->d;
  unsigned long long st = 1;
  for (int k = 0; k < 4; ++k) {
    if (k < h->d) {
      s.off[2 * k] = (unsigned)st;
      s.off[2 * k + 1] = (unsigned)(0ull - st);
      st *= (unsigned long long)h->shape[k];
    } else {
      s.off[2 * k] = s.off[2 * k + 1] = 0;
    }
  }
  s.wt = h->wt;
  s.res = h->res;
  s.sw = h->sw;
  s.lab = h->lab;
  s.wide = h->wide ? 1 : 0;
  s.tbits = h->tbits;
  s.nwords = h->nwords;
  s.act[0] = h->act[0]; s.act[1] = h->act[1];
  s.pool[0] = h->pool[0]; s.pool[1] = h->pool[1];
  s.pool_cap = h->pool_cap;
  s.barr = h->barr;
  s.barr_cap = h->barr_cap;
  s.ctl = h->ctl;
  s.trace = h->trace;
  s.trace_cap = h->opt.trace_cap;
  s.budget = h->opt.cycle_budget;
  s.unit = h->opt.time_mode == WCSP_UNIT;
  s.minf = h->M == WCSP_M_INF;
  s.M = (int)(h->M == WCSP_M_INF ? 1 : h->M);
  s.ev = h->ev;
  s.ev_mask = h->ev_cap ? h->ev_cap - 1 : 0;
  s.bdesc = h->bdesc;
  s.bnev = h->bcounts;
  s.bnlane = h->bcounts ? h->bcounts + WHEEL : nullptr;
  s.bndesc = h->bcounts ? h->bcounts + 2 * WHEEL : nullptr;
  s.dcap = h->dcap;
  s.f1max = h->f1max;
  s.spill = h->spill;
  s.spill_cap = h->spill_cap;
  s.tlist = h->tlist;
  s.prog = h->prog;
  s.hyb_R = h->hyb_R;
  s.hyb_prep = getenv("WCSP_HYB_PREP") ? atoi(getenv("WCSP_HYB_PREP")) != 0 : 1;   // A/B switch
  // k_wheel_lag: decision c - 1 before treat(c) while the state words fit in a few L2s (C3 124.5 ->
  // 122.5 ms, C2 90.4 -> 85.4 ms), after it on DRAM-resident grids, whose fires are too uneven to
  // make treat(c) wait for the slowest block's fire(c - 1) (C5z8 6.98 -> 6.66 s;
  // profiles/r02/ab_lag_pre.txt)
  // k_wheel_lag A/B: warp 1 waits for the neighbourhood beside warp 0's decision (C3 122.6 -> 122.9,
  // C2 85.3 -> 87.5, C3s 14.3 -> 14.1 ms; profiles/r02/ab_lag_par.txt): off
  s.lag_par = getenv("WCSP_LAG_PAR") ? atoi(getenv("WCSP_LAG_PAR")) != 0 : 0;
  // WCSP_LAG_PRE=2: before treat(c) only if every block's fire(c - 1) is already counted, else after
  s.lag_pre = getenv("WCSP_LAG_PRE") ? atoi(getenv("WCSP_LAG_PRE"))
                                     : 8.0 * (double)h->N <= 4.0 * (double)std::max<long long>(h->l2_bytes, 1);
  // sparse cycles: about 64 triggered vertices per block (WCSP_LIST_MAX overrides, A/B runs)
  s.list_max = getenv("WCSP_LIST_MAX") ? strtoull(getenv("WCSP_LIST_MAX"), nullptr, 10)
                                       : (unsigned long long)h->grid * 64ull;
  s.nblocks = (unsigned)h->grid;
  s.win_words = win_words_for(s.nwords, s.nblocks);
  s.ileave = ileave_for(h);
  s.fstride = fstride_for(h);
  s.wbal = getenv("WCSP_WBAL") ? atoi(getenv("WCSP_WBAL")) != 0 : false;   // A/B: neutral on C3, slower on C2
  s.goff = h->goff;
  s.plane = h->plane;
  s.ghost_hi_start = h->ghi ? h->ghost_hi_start : (unsigned)h->N;
  s.ghost_out_lo = h->g_out_lo;
  s.ghost_out_hi = h->g_out_hi;
  s.slab = h->slab_index >= 0;
  s.staircase = h->staircase;
  s.f2stop = h->f2stop;
  s.stair = h->stair;
  s.stair_cap = h->stair_cap;
  return s;
}

wcsp_status alloc_pool(wcsp_handle* h, unsigned long long cap, int rec = 0) {
  if (rec == 0) rec = h->pool_rec;
  if (h->pool[0]) cudaFree(h->pool[0]);
  if (h->pool[1]) cudaFree(h->pool[1]);
  h->pool[0] = h->pool[1] = nullptr;
  h->pool_cap = 0;
  CK(cudaMalloc(&h->pool[0], cap * rec));
  CK(cudaMalloc(&h->pool[1], cap * rec));
  h->pool_cap = cap;
  h->pool_rec = rec;
  return WCSP_REACHED;
}

unsigned long long pow2_at_least(unsigned long long x) {
  unsigned long long p = 1;
  while (p < x) p <<= 1;
  return p;
}

wcsp_status alloc_ring(wcsp_handle* h, unsigned long long cap) {
  if (h->ev) cudaFree(h->ev);
  h->ev = nullptr;
  h->ev_cap = 0;
  cap = pow2_at_least(cap);
#if WCSP_WARP_FLUSH
  cap = std::min(cap, 1ull << 32);                  // ring slot indices are 32-bit in the warp-level filing
#endif
  CK(cudaMalloc(&h->ev, cap * sizeof(unsigned long long)));
  h->ev_cap = cap;
  return WCSP_REACHED;
}

wcsp_status alloc_desc(wcsp_handle* h, unsigned dcap) {
  if (h->bdesc) cudaFree(h->bdesc);
  h->bdesc = nullptr;
  h->dcap = 0;
  CK(cudaMalloc(&h->bdesc, (size_t)WHEEL * h->grid * dcap * sizeof(unsigned long long)));
  h->dcap = dcap;
  return WCSP_REACHED;
}

int grid_for(const wcsp_handle* h, unsigned long long n) {
  unsigned long long b = (n + THREADS - 1) / THREADS;
  return (int)std::max<unsigned long long>(1, std::min<unsigned long long>(b, (unsigned long long)h->nsm * 8));
}

wcsp_status check_M(long long M) {
  if (M == WCSP_M_INF) return WCSP_REACHED;
  if (M < 1 || M > WCSP_M_MAX_WIDE)
    return fail(WCSP_EINVAL, "M = %lld outside [1, %lld] (and not WCSP_M_INF)", M, (long long)WCSP_M_MAX_WIDE);
  return WCSP_REACHED;
}
bool wide_M(long long M) { return M != WCSP_M_INF && M > WCSP_M_MAX; }

wcsp_status validate_device(wcsp_handle* h, const uint8_t* f1, const uint8_t* f2) {
  CK(cudaMemsetAsync(h->d_cnt, 0, 5 * sizeof(unsigned long long), h->stream));
  k_validate<<<grid_for(h, h->N), THREADS, 0, h->stream>>>(h->N, h->d, h->shape[0], h->shape[1], h->shape[2],
                                                          h->shape[3], f1, f2, h->d_maskA, h->d_maskB,
                                                          h->present_all ? nullptr : h->d_present, h->d_cnt);
  CK(cudaGetLastError());
  unsigned long long c[5];
  CK(cudaMemcpyAsync(c, h->d_cnt, sizeof(c), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  if (c[0] == 0) return fail(WCSP_EINVAL, "A is empty (among present vertices)");
  if (c[1] == 0) return fail(WCSP_EINVAL, "B is empty (among present vertices)");
  if (c[2] != 0) return fail(WCSP_EINVAL, "A and B intersect in %llu vertices", c[2]);
  if (c[3] != 0) return fail(WCSP_EINVAL, "%llu present edges have f1 > 0 and f2 = 0", c[3]);
  h->f1max = std::max<int>(1, (int)c[4]);
  // per cycle a target receives at most one lane and one phantom per half-edge: 2 * 2d arrivals
  const unsigned long long need = std::max<unsigned long long>(64, 4ull * h->d * c[1]);
  if (need > h->barr_cap) {
    if (h->barr) cudaFree(h->barr);
    h->barr = nullptr;
    h->barr_cap = 0;
    CK(cudaMalloc(&h->barr, 2 * need * sizeof(BArr)));   // one list per cycle parity
    h->barr_cap = (unsigned)need;
  }
  return WCSP_REACHED;
}

wcsp_status build_weights(wcsp_handle* h, const uint8_t* f1, const uint8_t* f2) {
  Dev s = make_dev(h);
  const int g = grid_for(h, h->N);
  switch (h->d) {
    case 1: k_weights<1><<<g, THREADS, 0, h->stream>>>(s, f1, f2, h->shape[0], 1, 1, 1); break;
    case 2: k_weights<2><<<g, THREADS, 0, h->stream>>>(s, f1, f2, h->shape[0], h->shape[1], 1, 1); break;
    case 3: k_weights<3><<<g, THREADS, 0, h->stream>>>(s, f1, f2, h->shape[0], h->shape[1], h->shape[2], 1); break;
    default: k_weights<4><<<g, THREADS, 0, h->stream>>>(s, f1, f2, h->shape[0], h->shape[1], h->shape[2], h->shape[3]); break;
  }
  CK(cudaGetLastError());
  return WCSP_REACHED;
}

wcsp_status copy_mask(wcsp_handle* h, uint8_t* dst, const uint8_t* src, int mem) {
  CK(cudaMemcpyAsync(dst, src, h->N, mem == WCSP_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                     h->stream));
  return WCSP_REACHED;
}

wcsp_status load_problem(wcsp_handle* h, const wcsp_problem* p) {
  wcsp_status st;
  if ((st = check_M(p->M)) != WCSP_REACHED) return st;
  if (!p->f1 || !p->f2 || !p->maskA || !p->maskB) return fail(WCSP_EINVAL, "f1, f2, maskA, maskB must be non-NULL");
  const size_t fb = (size_t)h->d * h->N;
  const uint8_t *f1 = p->f1, *f2 = p->f2;
  if (p->mem == WCSP_MEM_HOST) {
    CK(cudaMemcpyAsync(h->d_f1, p->f1, fb, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->d_f2, p->f2, fb, cudaMemcpyHostToDevice, h->stream));
    f1 = h->d_f1;
    f2 = h->d_f2;
  } else if (p->mem != WCSP_MEM_DEVICE) {
    return fail(WCSP_EINVAL, "mem must be WCSP_MEM_HOST or WCSP_MEM_DEVICE");
  }
  if ((st = copy_mask(h, h->d_maskA, p->maskA, p->mem)) != WCSP_REACHED) return st;
  if ((st = copy_mask(h, h->d_maskB, p->maskB, p->mem)) != WCSP_REACHED) return st;
  h->present_all = p->present == nullptr;
  if (!h->present_all && (st = copy_mask(h, h->d_present, p->present, p->mem)) != WCSP_REACHED) return st;
  if (h->slab_index < 0) {
    if ((st = validate_device(h, f1, f2)) != WCSP_REACHED) return st;
  } else {                         // slab child: the group validated the whole problem on the host
    const unsigned long long need = std::max<unsigned long long>(64, 4ull * h->d * h->preset_nB);
    if (need > h->barr_cap) {
      if (h->barr) cudaFree(h->barr);
      h->barr = nullptr;
      CK(cudaMalloc(&h->barr, 2 * need * sizeof(BArr)));
      h->barr_cap = (unsigned)need;
    }
  }
  if ((st = build_weights(h, f1, f2)) != WCSP_REACHED) return st;
  h->M = p->M;
  return WCSP_REACHED;
}

void destroy_comm(void* comm);

void release(wcsp_handle* h) {
  if (h->comm) destroy_comm(h->comm);
  h->comm = nullptr;
  for (void* p : h->ipc_opened) cudaIpcCloseMemHandle(p);
  h->ipc_opened.clear();
  for (wcsp_handle* c : h->children) {
    release(c);
    delete c;
  }
  h->children.clear();
  void* bufs[] = {h->d_f1, h->d_f2, h->d_maskA, h->d_maskB, h->d_present, h->wt, h->res, h->sw, h->lab, h->tbits, h->barr,
                  h->act[0], h->act[1], h->pool[0], h->pool[1], h->ev, h->bdesc, h->bcounts, h->ctl, h->trace,
                  h->d_cnt, h->d_ghost, h->g_out_lo, h->g_out_hi, h->g_in_lo, h->g_in_hi, h->l_out_lo,
                  h->l_out_hi, h->l_in_lo, h->l_in_hi, h->d_ctls, h->stair, h->xbar, h->d_pctl, h->spill, h->tlist, h->prog};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (h->h_ctl) cudaFreeHost(h->h_ctl);
  if (h->e0) cudaEventDestroy(h->e0);
  if (h->e1) cudaEventDestroy(h->e1);
  if (h->em) cudaEventDestroy(h->em);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
}

// Optional (WCSP_L2_PERSIST=1): an access-policy window on the solver's stream marking up to the
// device's persisting set-aside of the vertex state words as persisting.  Off by default: the
// per-access cache-policy hints of the kernels (evict-last on state words, evict-first on events
// and weight records) already keep the state words resident, and the set-aside only shrinks the
// L2 the rest competes for — C3 133.8 -> 131.6 ms, C3s 15.08 -> 14.48 ms, C2 96.2 -> 95.4 ms,
// C5z8 8.75 -> 8.60 s without it (profiles/r02/ab_persist.txt, ab_c5z8_l2.txt).
void set_l2_window(wcsp_handle* h) {
  const char* env = getenv("WCSP_L2_PERSIST");
  if (!env || env[0] != '1') return;
  int max_persist = 0, max_window = 0;
  if (cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, h->dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, h->dev) != cudaSuccess ||
      max_persist <= 0 || max_window <= 0) {
    cudaGetLastError();
    return;
  }
  if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)max_persist) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  const size_t bytes = std::min<size_t>((size_t)h->N * sizeof(unsigned long long), (size_t)max_window);
  cudaStreamAttrValue attr{};
  attr.accessPolicyWindow.base_ptr = h->sw;
  attr.accessPolicyWindow.num_bytes = bytes;
  attr.accessPolicyWindow.hitRatio = std::min(1.0f, (float)max_persist / (float)bytes);
  attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  if (cudaStreamSetAttribute(h->stream, cudaStreamAttributeAccessPolicyWindow, &attr) != cudaSuccess)
    cudaGetLastError();
}

wcsp_status reset_ctl(wcsp_handle* h) {
  memset(h->h_ctl, 0, sizeof(Ctl));
  Ctl& c = *h->h_ctl;
  c.view.stamp = stamp_of(0);
  c.view.status = ST_RUNNING;
  c.view.region = 256;
  for (int i = 0; i < NACC; ++i) c.acc[i].dmin = 0xFFFFFFFFu;
  c.acc[0].tl_over = 1;            // cycle 0 treats A from the bitmap (k_init)
  c.ovf_t = 0x7FFFFFFFFFFFFFFFll;
  CK(cudaMemcpyAsync(h->ctl, h->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, h->stream));
  if (is_wheel(h->eng)) {
    CK(cudaMemsetAsync(h->bcounts, 0, (size_t)WHEEL * (2 + h->grid) * sizeof(unsigned), h->stream));
    if (h->prog) CK(cudaMemsetAsync(h->prog, 0, (size_t)h->grid * sizeof(unsigned long long), h->stream));
  }
  return WCSP_REACHED;
}

wcsp_status launch_init(wcsp_handle* h) {
  Dev s = make_dev(h);
  k_init<<<grid_for(h, h->N), THREADS, 0, h->stream>>>(s, h->d_maskA, h->d_maskB,
                                                      h->present_all ? nullptr : h->d_present, h->d_ghost,
                                                      h->M == WCSP_M_INF ? 1 : (int)h->M, h->d);
  CK(cudaGetLastError());
  h->launches += 1;
  return WCSP_REACHED;
}

template <int D>
void* hybrid_fn(bool big) {
  return big ? reinterpret_cast<void*>(&k_wheel_hybrid<D, 4>) : reinterpret_cast<void*>(&k_wheel_hybrid<D, 3>);
}
void* hybrid_fn_d(int d, bool big) {
  return d == 1 ? hybrid_fn<1>(big) : d == 2 ? hybrid_fn<2>(big) : d == 3 ? hybrid_fn<3>(big) : hybrid_fn<4>(big);
}
template <int D>
void* lag_fn(bool big) {
  return big ? reinterpret_cast<void*>(&k_wheel_lag<D, 4>) : reinterpret_cast<void*>(&k_wheel_lag<D, 3>);
}
void* lag_fn_d(int d, bool big) {
  return d == 1 ? lag_fn<1>(big) : d == 2 ? lag_fn<2>(big) : d == 3 ? lag_fn<3>(big) : lag_fn<4>(big);
}
// The lagged-decision kernel (k_wheel_lag) wherever the hybrid applies, unless tracing (its cycle
// records come from the hybrid's per-cycle decision) or WCSP_HYB_LAG=0 (A/B).
bool lag_for(const wcsp_handle* h) {
  const char* e = getenv("WCSP_HYB_LAG");
  return h->hyb && h->opt.trace_cap == 0 && (e ? atoi(e) != 0 : HYB_LAG_DEFAULT);
}

wcsp_status run_persistent(wcsp_handle* h) {
  Dev s = make_dev(h);
  void* args[] = {&s};
  void* fn = h->hyb ? (lag_for(h) ? lag_fn_d(h->d, h->big) : hybrid_fn_d(h->d, h->big))
                    : cycle_fn_d(h->d, h->eng, h->big, h->wide);
  CK(cudaLaunchCooperativeKernel(fn, dim3(h->grid), dim3(THREADS), args, sizeof(Smem),
                                 h->stream));
  h->launches += 1;
  return WCSP_REACHED;
}

template <int D>
void launch_cycle(wcsp_handle* h, const Dev& s) {
  const size_t sm = sizeof(Smem);
  if (is_wheel(h->eng)) {
    k_wheel_fire<D><<<h->grid, THREADS, sm, h->stream>>>(s);
    k_wheel_treat<D><<<h->grid, THREADS, sm, h->stream>>>(s);
    k_wheel_decide<<<1, 32, 0, h->stream>>>(s);
  } else if (h->wide) {
    k_sweep<D, true><<<h->grid, THREADS, sm, h->stream>>>(s);
    k_treat<D, true><<<h->grid, THREADS, sm, h->stream>>>(s);
    k_decide<<<1, 32, 0, h->stream>>>(s);
  } else {
    k_sweep<D><<<h->grid, THREADS, sm, h->stream>>>(s);
    k_treat<D><<<h->grid, THREADS, sm, h->stream>>>(s);
    k_decide<<<1, 32, 0, h->stream>>>(s);
  }
}

wcsp_status run_stepped(wcsp_handle* h) {
  Dev s = make_dev(h);
  int batch = 4;
  for (;;) {
    for (int i = 0; i < batch; ++i) {
      switch (h->d) {
        case 1: launch_cycle<1>(h, s); break;
        case 2: launch_cycle<2>(h, s); break;
        case 3: launch_cycle<3>(h, s); break;
        default: launch_cycle<4>(h, s); break;
      }
      h->launches += 3;
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&h->h_ctl->view, &h->ctl->view, sizeof(View), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    const int st = h->h_ctl->view.status;
    if (st == ST_WRAP) {               // maintenance pass (stamp wrap / texp refresh), then continue
      if (is_wheel(h->eng)) k_wheel_maintain<<<h->grid, THREADS, 0, h->stream>>>(s);
      else if (h->wide) k_clear_temps<true><<<h->grid, THREADS, 0, h->stream>>>(s);
      else k_clear_temps<<<h->grid, THREADS, 0, h->stream>>>(s);
      h->launches += 1;
      CK(cudaGetLastError());
      const int run = ST_RUNNING;
      CK(cudaMemcpyAsync(&h->ctl->view.status, &run, sizeof(int), cudaMemcpyHostToDevice, h->stream));
      CK(cudaStreamSynchronize(h->stream));
      continue;
    }
    if (st != ST_RUNNING) break;
    batch = std::min(batch * 2, 64);
  }
  return WCSP_REACHED;
}

int x_lane_of(const wcsp_handle* h, long long X, long long Y) {
  long long st = 1;
  for (int k = 0; k < h->d; ++k) {
    if (Y == X + st) return 2 * k;
    if (Y == X - st) return 2 * k + 1;
    st *= h->shape[k];
  }
  return -1;
}

wcsp_status solve_once(wcsp_handle* h, wcsp_result* r, int* status) {
  wcsp_status st;
  h->launches = 0;
#if WCSP_CHECKS
  // checked build: poison the event ring (src 0x3F7F7F7F), so an event read before it was written
  // in this solve traps in the fire's bounds check
  if (is_wheel(h->eng) && h->ev) CK(cudaMemsetAsync(h->ev, 0x7F, h->ev_cap * sizeof(unsigned long long), h->stream));
#endif
  CK(cudaEventRecord(h->e0, h->stream));
  if ((st = reset_ctl(h)) != WCSP_REACHED) return st;
  if ((st = launch_init(h)) != WCSP_REACHED) return st;
  CK(cudaEventRecord(h->em, h->stream));
  st = is_stepped(h->eng) ? run_stepped(h) : run_persistent(h);
  if (st != WCSP_REACHED) return st;
  CK(cudaEventRecord(h->e1, h->stream));
  CK(cudaMemcpyAsync(h->h_ctl, h->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  float ms = 0, cms = 0;
  CK(cudaEventElapsedTime(&ms, h->e0, h->e1));
  CK(cudaEventElapsedTime(&cms, h->em, h->e1));
  const Ctl& c = *h->h_ctl;
  if (c.abort) return fail(WCSP_ECUDA, "persistent kernel: grid barrier watchdog fired (blocks not co-resident?)");
  *status = c.view.status;
  memset(r, 0, sizeof(*r));
  r->F1 = c.F1;
  r->F2 = c.F2;
  r->X = c.X;
  r->Y = c.Y;
  r->via_phantom = (int)c.via;
  r->x_lane = *status == WCSP_REACHED ? x_lane_of(h, c.X, c.Y) : -1;
  if (*status != WCSP_REACHED) r->F1 = r->F2 = r->X = r->Y = -1;
  r->cycles = c.cycles;
  r->edge_updates = c.edge_updates;
  r->arrivals = c.arrivals;
  r->triggered = c.triggered;
  r->phantoms_created = c.created;
  r->relabels = c.relabels;
  r->lanes_started = c.started;
  r->peak_active = c.peak_active;
  r->peak_phantoms = c.peak_phantoms;
  r->phantom_capacity = (long long)(is_wheel(h->eng) ? h->ev_cap : h->pool_cap);
  r->kernel_launches = h->launches;
  r->device_ms = ms;
  r->cycle_ms = cms;
  r->staging_appended = (long long)c.n_appended;
  r->staging_spilled = (long long)c.n_spilled;
  r->staging_singles = (long long)c.n_single;
  h->last_cycles = c.cycles;
  if (*status == WCSP_EOVERFLOW) r->phantom_capacity = c.need_pool;
  return WCSP_REACHED;
}

// Device-side overflow path ("difficulties with dynamic memory locations"): a
// storage overflow ends the run with a flag and the needed size; the host grows exactly the
// structure that overflowed and re-runs.  The size a run reports is only what its failing cycle
// needed (the front keeps growing), so a retry takes twice that and at least 4x the old size
// (2x once the structure is past 2^26 entries, where memory matters).
constexpr int MAX_ATTEMPTS = 12;
#ifndef HYBRID_DEFAULT
#define HYBRID_DEFAULT true
#endif
unsigned long long grown(unsigned long long cap, long long need) {
  const unsigned long long f = cap < (1ull << 26) ? 4 : 2;
  return std::max<unsigned long long>(2ull * (unsigned long long)std::max(need, 0ll), f * cap);
}

// The one-barrier hybrid kernel (k_wheel_hybrid) for single-device persistent wheel solves; its
// neighbourhood radius in blocks covers twice the largest lane offset (a fire's destinations are one
// offset from its sources, a treat's neighbour reads one offset from its vertices).  WCSP_HYBRID=0/1.
bool hybrid_for(wcsp_handle* h) {
  // default on (profiles/r02/ab_hybrid.txt, warp-parallel neighbourhood wait): C3 132.8 -> 131.0 ms,
  // C2 99.6 -> 95.2 ms, C5z8 8.62 -> 7.74 s; C3s 14.65 -> 15.29 ms is the one measured loss
  const char* e = getenv("WCSP_HYBRID");
  const bool want = e ? atoi(e) != 0 : HYBRID_DEFAULT;
  if (!want || h->eng != WCSP_ENGINE_WHEEL || h->slab_index >= 0 || h->staircase || h->f1max >= 64 || !h->prog)
    return false;
  const Dev s = make_dev(h);
  if (s.ileave || s.wbal) return false;
  const unsigned long long ww = s.win_words, nwin = (s.nwords + ww - 1) / ww;
  const unsigned long long r0 = (nwin + (unsigned long long)h->grid * WARPS - 1) / ((unsigned long long)h->grid * WARPS);
  const unsigned long long span = std::max<unsigned long long>(1, r0 * WARPS * ww * 32ull);
  unsigned long long maxoff = 1;
  for (int k = 0; k + 1 < h->d; ++k) maxoff *= (unsigned long long)h->shape[k];
  h->hyb_R = (int)std::min<unsigned long long>((2 * maxoff + span - 1) / span + 1, (unsigned long long)h->grid);
  if (const char* r = getenv("WCSP_HYB_R")) h->hyb_R = std::max(h->hyb_R, atoi(r));   // A/B: a wider wait
  return true;
}

// Budgets above WCSP_M_MAX run the sweep engine with u32 labels and u64 stamped temps
// (include/wcsp.h; the 16-bit layout stays the default): allocate its state on first use.
wcsp_status prepare_engine(wcsp_handle* h) {
  h->wide = wide_M(h->M);
  h->hyb = false;
  if (!h->wide) {
    h->eng = h->opt.engine;
    h->grid = h->grid_main;
    h->hyb = hybrid_for(h);
    return WCSP_REACHED;
  }
  h->eng = is_stepped(h->opt.engine) ? WCSP_ENGINE_STEPPED : WCSP_ENGINE_PERSISTENT;
  const unsigned long long N = h->N;
  if (!h->lab) CK(cudaMalloc(&h->lab, N * sizeof(unsigned)));
  if (!h->res) CK(cudaMalloc(&h->res, N * lane_bytes(h->d)));
  if (!h->act[0]) CK(cudaMalloc(&h->act[0], N * sizeof(unsigned)));
  if (!h->act[1]) CK(cudaMalloc(&h->act[1], N * sizeof(unsigned)));
  if (!h->pool[0] || h->pool_rec != (int)sizeof(PhW)) {
    const unsigned long long cap = h->opt.phantom_capacity > 0 ? (unsigned long long)h->opt.phantom_capacity
                                                               : std::max<unsigned long long>(4 * N, 1ull << 20);
    wcsp_status st = alloc_pool(h, cap, (int)sizeof(PhW));
    if (st != WCSP_REACHED) return st;
  }
  if (!h->grid_wide) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cycle_fn_d(h->d, h->eng, false, true), THREADS,
                                                     sizeof(Smem)));
    if (per_sm < 1) return fail(WCSP_ECUDA, "wide cycle kernel cannot be resident");
    h->grid_wide = std::min(per_sm * h->nsm, h->grid_main);
  }
  h->grid = h->grid_wide;
  return WCSP_REACHED;
}

wcsp_status solve_impl(wcsp_handle* h, wcsp_result* out) {
  {
    wcsp_status st = prepare_engine(h);
    if (st != WCSP_REACHED) return st;
  }
  wcsp_result r;
  int status = ST_RUNNING;
  int attempt = 0;
  for (; attempt < MAX_ATTEMPTS; ++attempt) {
    wcsp_status st = solve_once(h, &r, &status);
    if (st != WCSP_REACHED) return st;
    r.retries = attempt;
    if (status != WCSP_EOVERFLOW) break;
    // overflow of a device structure: grow it and re-run (device flag -> host retry)
    const long long need = r.phantom_capacity;
    if (is_wheel(h->eng)) {
      if (need == -2) st = alloc_desc(h, h->dcap * 2);
      else st = alloc_ring(h, grown(h->ev_cap, need));
    } else {
      st = alloc_pool(h, grown(h->pool_cap, need));
    }
    if (st != WCSP_REACHED) return st;
  }
  if (status == WCSP_EOVERFLOW) return fail(WCSP_EOVERFLOW, "phantom/event storage overflow after retries");
  if (status == WCSP_EBUDGET) { *out = r; return fail(WCSP_EBUDGET, "cycle budget %lld exceeded", h->opt.cycle_budget); }
  if (status != WCSP_REACHED && status != WCSP_INFEASIBLE) return fail(WCSP_ECUDA, "solver ended in state %d", status);
  *out = r;
  return (wcsp_status)status;
}

struct SlabSpec {
  int index;
  long long z0, z1;
  int glo, ghi;
  unsigned goff, plane;
  const uint8_t* ghost;            // host [N_local]
  unsigned long long nB;
  int f1max;
  int per_sm;                      // > 0: blocks per SM of the slab's grid (peer halo, 4-block build)
};

wcsp_status create_impl(const wcsp_problem* p, const wcsp_options& opt, const SlabSpec* spec, wcsp_handle** out) {
  unsigned long long N = 1;
  for (int k = 0; k < p->d; ++k) N *= (unsigned long long)p->shape[k];
  wcsp_handle* h = new wcsp_handle();
  h->opt = opt;
  h->d = p->d;
  for (int k = 0; k < 4; ++k) h->shape[k] = k < p->d ? p->shape[k] : 1;
  h->N = N;
  h->nwords = (unsigned)((N + 31) / 32);
  h->dev = opt.device;
#define CKH(call)                       \
  do {                                  \
    wcsp_status s_ = (call);            \
    if (s_ != WCSP_REACHED) {           \
      release(h);                       \
      delete h;                         \
      return s_;                        \
    }                                   \
  } while (0)
#define CKC(call) CKH([&]() -> wcsp_status { CK(call); return WCSP_REACHED; }())
  CKC(cudaSetDevice(h->dev));
  if (opt.stream) {
    h->stream = (cudaStream_t)opt.stream;
  } else {
    CKC(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    h->own_stream = true;
  }
  CKC(cudaDeviceGetAttribute(&h->nsm, cudaDevAttrMultiProcessorCount, h->dev));
  {
    int l2 = 0;
    CKC(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, h->dev));
    h->l2_bytes = l2;
  }
  switch (p->d) {
    case 1: CKC(set_smem_attrs<1>()); break;
    case 2: CKC(set_smem_attrs<2>()); break;
    case 3: CKC(set_smem_attrs<3>()); break;
    default: CKC(set_smem_attrs<4>()); break;
  }
  // Persistent wheel engine: the build for 4 resident blocks per SM (64 registers) on 3-D and
  // higher grids of at least 1.5 * 2^20 vertices (thick fronts: C3 157.8 -> 137.3 ms), the one for 3 (80
  // registers) otherwise, where cycles are short or fronts thin and the grid barriers dominate
  // (C2 1024^2, C4 fractal: 24.6 vs 31 ms).
  const char* bps = getenv("WCSP_BLOCKS_PER_SM");                   // A/B runs
  // (lagged kernel, profiles/r02/ab_bps_lag.txt: 3-D from 1.5 * 2^20 vertices — P6-125, 1.95M: 13.0 ->
  // 10.7 ms; P6-100, 1.0M: 7.07 vs 7.31 ms, P6-75 and P6-50 also faster with 3)
  h->big = opt.engine == WCSP_ENGINE_WHEEL && (bps ? atoi(bps) >= 4 : p->d >= 3 && N >= (3ull << 19));
  int per_sm = 0;
  CKC(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cycle_fn_d(p->d, opt.engine, h->big), THREADS,
                                                    sizeof(Smem)));
  if (per_sm < 1) CKH(fail(WCSP_ECUDA, "cycle kernel cannot be resident"));
  if (bps) per_sm = std::max(1, std::min(per_sm, atoi(bps)));
  // 2-D grids up to 2^22 vertices: short cycles whose fixed costs (barriers, waits, decisions) grow
  // with the block count — 2 resident blocks per SM (C2 94.0 -> 89.1 ms, C4 15.9 -> 15.1 ms;
  // profiles/r02/ab_bps.txt); 3-D grids keep the occupancy their treat gathers need
  else if (p->d <= 2 && N <= (1ull << 22) && !spec) per_sm = std::min(per_sm, 2);
  if (spec && spec->per_sm > 0) per_sm = spec->per_sm;     // peer-halo slab: sized for the peer kernel
  h->grid = h->grid_main = per_sm * h->nsm;
  h->eng = opt.engine;
  const size_t fb = (size_t)h->d * N;
  CKC(cudaMalloc(&h->d_f1, fb));
  CKC(cudaMalloc(&h->d_f2, fb));
  CKC(cudaMalloc(&h->d_maskA, N));
  CKC(cudaMalloc(&h->d_maskB, N));
  CKC(cudaMalloc(&h->d_present, N));
  CKC(cudaMalloc(&h->wt, N * 2 * lane_bytes(h->d)));
  CKC(cudaMalloc(&h->sw, N * sizeof(unsigned long long)));
  CKC(cudaMalloc(&h->tbits, (size_t)h->nwords * sizeof(unsigned)));
  CKC(cudaMalloc(&h->ctl, sizeof(Ctl)));
  CKC(cudaMallocHost(&h->h_ctl, sizeof(Ctl)));
  CKC(cudaMalloc(&h->d_cnt, 5 * sizeof(unsigned long long)));
  CKC(cudaMalloc(&h->trace, std::max<long long>(1, opt.trace_cap) * sizeof(TraceRec)));
  CKC(cudaEventCreate(&h->e0));
  CKC(cudaEventCreate(&h->e1));
  CKC(cudaEventCreate(&h->em));
  const unsigned long long cap = opt.phantom_capacity > 0 ? (unsigned long long)opt.phantom_capacity
                                                          : std::max<unsigned long long>(4 * N, 1ull << 20);
  if (is_wheel(opt.engine)) {
    // auto: twice the sweep pool's default plus the slack of every block's open regions (grid x 10
    // delays x 4096-slot regions) over the cycles the ring guard keeps them live — eight: the
    // lagged-decision kernel counts a cycle's slots live until every block has fired two cycles
    // past their last use (with two, C3's first solve on a fresh handle overflowed the 2^28-slot
    // ring and re-ran: profiles/r02/first_solve_lag_r02aj.log) — unless the power-of-two rounding
    // would then double a ring of more than 2^31 slots (C5: 8N alone suffices).  An explicit
    // capacity is taken as given (the overflow path grows it).
    unsigned long long ring = std::max<unsigned long long>(2 * cap, (unsigned long long)h->grid * 2 * 4096);
    const unsigned long long slack = std::min<unsigned long long>((unsigned long long)h->grid * 8ull * 10ull * 4096ull,
                                                                  4 * cap);   // small grids: small rings
    if (pow2_at_least(ring + slack) <= (1ull << 31)) ring += slack;
    CKH(alloc_ring(h, opt.phantom_capacity > 0 ? cap : ring));
    const char* dc = getenv("WCSP_DCAP");          // tests: a tiny run-descriptor table forces its overflow path
    // runs per (bucket, block): one per source cycle and region; big grids file more (C5z8: up to 40
    // on block 0, which made every fresh handle's first solve overflow 32 and re-run)
    CKH(alloc_desc(h, dc ? (unsigned)std::max(1, atoi(dc)) : (N >= (1ull << 22) ? 64u : 32u)));
    CKC(cudaMalloc(&h->bcounts, (size_t)WHEEL * (2 + h->grid) * sizeof(unsigned)));
    // spill room per block and flush period: a dense window round (e.g. the initial treatment
    // of a whole boundary) can stage several times the shared-memory staging
    h->spill_cap = (unsigned)std::min<unsigned long long>(WCSP_FLUSH_LAZY < 0 ? 65536 : 16384,
                                                          std::max<unsigned long long>(2048, pow2_at_least(8 * N / h->grid)));
    CKC(cudaMalloc(&h->spill, (size_t)h->grid * h->spill_cap * sizeof(unsigned long long)));
    CKC(cudaMalloc(&h->tlist, (size_t)h->grid * QA_CAP * sizeof(unsigned)));
    CKC(cudaMalloc(&h->prog, (size_t)h->grid * sizeof(unsigned long long)));
  } else {
    CKC(cudaMalloc(&h->res, N * lane_bytes(h->d)));
    CKC(cudaMalloc(&h->act[0], N * sizeof(unsigned)));
    CKC(cudaMalloc(&h->act[1], N * sizeof(unsigned)));
    CKH(alloc_pool(h, cap));
  }
  set_l2_window(h);
  if (spec) {                      // slab child: geometry, ghost flags and exchange planes
    h->slab_index = spec->index;
    h->z0 = spec->z0; h->z1 = spec->z1; h->glo = spec->glo; h->ghi = spec->ghi;
    h->goff = spec->goff; h->plane = spec->plane;
    h->ghost_hi_start = (unsigned)((spec->glo + spec->z1 - spec->z0) * spec->plane);
    h->preset_nB = spec->nB;
    h->f1max = spec->f1max;
    CKC(cudaMalloc(&h->d_ghost, N));
    CKC(cudaMemcpy(h->d_ghost, spec->ghost, N, cudaMemcpyHostToDevice));
    const size_t pb = (size_t)spec->plane;
    CKC(cudaMalloc(&h->g_out_lo, pb * 8)); CKC(cudaMalloc(&h->g_out_hi, pb * 8));
    CKC(cudaMalloc(&h->g_in_lo, pb * 8)); CKC(cudaMalloc(&h->g_in_hi, pb * 8));
    CKC(cudaMalloc(&h->l_out_lo, pb * 4)); CKC(cudaMalloc(&h->l_out_hi, pb * 4));
    CKC(cudaMalloc(&h->l_in_lo, pb * 4)); CKC(cudaMalloc(&h->l_in_hi, pb * 4));
    CKC(cudaMemset(h->g_out_lo, 0, pb * 8)); CKC(cudaMemset(h->g_out_hi, 0, pb * 8));
    CKC(cudaMemset(h->g_in_lo, 0, pb * 8)); CKC(cudaMemset(h->g_in_hi, 0, pb * 8));
  }
  CKH(load_problem(h, p));
  if (spec) h->f1max = spec->f1max;
#undef CKC
#undef CKH
  *out = h;
  return WCSP_REACHED;
}


// ---------------------------------------------------------------------------
// Slab engine, virtual slabs on one device: the grid is cut
// along its last axis into opt.slabs children, each a complete wheel solver
// over its slab plus ghost planes; per cycle the children exchange the water
// that crossed a slab boundary and their boundary labels, and combine their
// proposals for the cycle decision.  The multi-GPU form replaces the
// device-to-device copies and k_slab_reduce by NCCL send/recv and an
// allreduce(max); the kernels are the same.
// ---------------------------------------------------------------------------
struct NcclApi {
  bool ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
};

NcclApi& nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  const char* path = getenv("WCSP_NCCL_LIB");
  void* lib = dlopen(path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) return api;
  api.getUniqueId = (decltype(api.getUniqueId))dlsym(lib, "ncclGetUniqueId");
  api.commInitRank = (decltype(api.commInitRank))dlsym(lib, "ncclCommInitRank");
  api.commDestroy = (decltype(api.commDestroy))dlsym(lib, "ncclCommDestroy");
  api.send = (decltype(api.send))dlsym(lib, "ncclSend");
  api.recv = (decltype(api.recv))dlsym(lib, "ncclRecv");
  api.allReduce = (decltype(api.allReduce))dlsym(lib, "ncclAllReduce");
  api.allGather = (decltype(api.allGather))dlsym(lib, "ncclAllGather");
  api.groupStart = (decltype(api.groupStart))dlsym(lib, "ncclGroupStart");
  api.groupEnd = (decltype(api.groupEnd))dlsym(lib, "ncclGroupEnd");
  api.errStr = (decltype(api.errStr))dlsym(lib, "ncclGetErrorString");
  api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.send && api.recv && api.allReduce &&
           api.allGather &&
           api.groupStart && api.groupEnd && api.errStr;
  return api;
}

wcsp_status host_validate(const wcsp_problem* p, unsigned long long* nB, int* f1max) {
  long long N = 1, st[4] = {1, 1, 1, 1};
  for (int k = 0; k < p->d; ++k) { st[k] = N; N *= p->shape[k]; }
  unsigned long long na = 0, nb = 0, nab = 0, bad = 0;
  int fmax = 1;
  for (long long v = 0; v < N; ++v) {
    const bool pr = p->present == nullptr || p->present[v] != 0;
    const bool a = pr && p->maskA[v], b = pr && p->maskB[v];
    na += a; nb += b; nab += a && b;
    for (int k = 0; k < p->d; ++k) {
      if ((v / st[k]) % p->shape[k] + 1 < p->shape[k]) {
        const uint8_t f1 = p->f1[(size_t)k * N + v], f2 = p->f2[(size_t)k * N + v];
        bad += f1 != 0 && f2 == 0;
        fmax = std::max<int>(fmax, f1);
      }
    }
  }
  if (na == 0) return fail(WCSP_EINVAL, "A is empty (among present vertices)");
  if (nb == 0) return fail(WCSP_EINVAL, "B is empty (among present vertices)");
  if (nab) return fail(WCSP_EINVAL, "A and B intersect in %llu vertices", nab);
  if (bad) return fail(WCSP_EINVAL, "%llu present edges have f1 > 0 and f2 = 0", bad);
  *nB = nb;
  *f1max = fmax;
  return WCSP_REACHED;
}

void* peer_fn_d(int d, bool big);
wcsp_status peer_connect(wcsp_handle* g);

// options.local_slab: counts of the validation rules (include/wcsp.h) over the planes [z0, z1) a
// rank owns, from its local arrays that start at plane p0 ([0] |A|, [1] |B|, [2] |A n B|, [3]
// present edges with f2 = 0, [4] max f1); every edge (v, v + e_k) is stored at v, so summing the
// owners' counts checks each vertex and edge of the grid exactly once.
void local_counts(const wcsp_problem* p, long long Nl, long long plane, long long p0, long long z0, long long z1,
                  unsigned long long c[5]) {
  long long st[4] = {1, 1, 1, 1}, N = 1;
  for (int k = 0; k < p->d; ++k) { st[k] = N; N *= p->shape[k]; }
  for (int i = 0; i < 5; ++i) c[i] = 0;
  for (long long vl = (z0 - p0) * plane; vl < (z1 - p0) * plane; ++vl) {
    const long long v = p0 * plane + vl;
    const bool pr = p->present == nullptr || p->present[vl] != 0;
    const bool a = pr && p->maskA[vl], b = pr && p->maskB[vl];
    c[0] += a; c[1] += b; c[2] += a && b;
    for (int k = 0; k < p->d; ++k) {
      if ((v / st[k]) % p->shape[k] + 1 < p->shape[k]) {
        const uint8_t f1 = p->f1[(size_t)k * Nl + vl], f2 = p->f2[(size_t)k * Nl + vl];
        c[3] += f1 != 0 && f2 == 0;
        c[4] = std::max<unsigned long long>(c[4], f1);
      }
    }
  }
}

wcsp_status create_group(const wcsp_problem* p, const wcsp_options& opt, wcsp_handle** out) {
  const bool local = opt.local_slab != 0;
  if (local && !opt.nccl_id) return fail(WCSP_EINVAL, "local_slab needs the multi-GPU slab engine (nccl_id)");
  if (p->mem != WCSP_MEM_HOST && !local) return fail(WCSP_EINVAL, "the slab engine takes host arrays");
  if (!is_wheel(opt.engine)) return fail(WCSP_EINVAL, "the slab engine runs the wheel engine (engine = WHEEL)");
  if (wide_M(p->M)) return fail(WCSP_EINVAL, "slab engine: M > %d (wide labels) is single-device only", WCSP_M_MAX);
  const bool dist = opt.nccl_id != nullptr && opt.nranks >= 1;   // nranks = 1: NCCL path on one GPU (tests)
  if (dist && (opt.rank < 0 || opt.rank >= opt.nranks || !opt.nccl_id))
    return fail(WCSP_EINVAL, "multi-GPU slab engine needs 0 <= rank < nranks and nccl_id");
  if (dist && !nccl_api().ok) return fail(WCSP_ENCCL, "cannot load libnccl.so.2 (set WCSP_NCCL_LIB)");
  const int R = dist ? opt.nranks : opt.slabs, d = p->d;
  const long long nL = p->shape[d - 1];
  if (nL < R) return fail(WCSP_EINVAL, "last axis (%lld) shorter than the number of slabs (%d)", nL, R);
  long long N = 1;
  for (int k = 0; k < d; ++k) N *= p->shape[k];
  const long long plane = N / nL;
  // peer halo on 3-D grids >= 2^21 vertices: the 4-blocks-per-SM build of the fused kernel (as
  // k_wheel_persistent); every slab handle is then sized for it
  const char* bps = getenv("WCSP_BLOCKS_PER_SM");
  const bool peer_big = opt.halo == WCSP_HALO_PEER && (bps ? atoi(bps) >= 4 : d >= 3 && N >= (1ll << 21));
  unsigned long long nB = 0;
  int f1max = 1;
  wcsp_status st = WCSP_REACHED;
  if (!local && (st = host_validate(p, &nB, &f1max)) != WCSP_REACHED) return st;
  wcsp_handle* g = new wcsp_handle();
  g->opt = opt;
  g->d = d;
  for (int k = 0; k < 4; ++k) g->shape[k] = k < d ? p->shape[k] : 1;
  g->N = (unsigned long long)N;
  g->dev = opt.device;
  g->M = p->M;
  g->plane = (unsigned)plane;
  auto bail = [&](wcsp_status s) { release(g); delete g; return s; };
  if (cudaSetDevice(g->dev) != cudaSuccess) return bail(fail(WCSP_ECUDA, "cudaSetDevice failed"));
  if (opt.stream) {
    g->stream = (cudaStream_t)opt.stream;
  } else {
    if (cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking) != cudaSuccess)
      return bail(fail(WCSP_ECUDA, "stream creation failed"));
    g->own_stream = true;
  }
  if (cudaEventCreate(&g->e0) != cudaSuccess || cudaEventCreate(&g->e1) != cudaSuccess ||
      cudaEventCreate(&g->em) != cudaSuccess)
    return bail(fail(WCSP_ECUDA, "event creation failed"));
  g->rank = dist ? opt.rank : 0;
  g->nranks = dist ? opt.nranks : 1;
  if (dist) {                      // the communicator first: local slabs combine their validation over it
    ncclUniqueId id;
    memcpy(&id, opt.nccl_id, sizeof(id));
    ncclComm_t comm = nullptr;
    const ncclResult_t nr = nccl_api().commInitRank(&comm, opt.nranks, id, opt.rank);
    if (nr != ncclSuccess) return bail(fail(WCSP_ENCCL, "ncclCommInitRank: %s", nccl_api().errStr(nr)));
    g->comm = comm;
  }
  // local_slab: this rank's arrays cover planes [lp0, lp1) only (device arrays are brought to the
  // host once, slab-sized); validate the owned planes and combine the counts over NCCL
  wcsp_problem lpb = *p;
  std::vector<uint8_t> hf1, hf2, hA, hB, hP;
  long long lp0 = 0;
  if (local) {
    long long zz[4];
    if ((st = wcsp_slab_planes(nL, R, opt.rank, (int64_t*)zz)) != WCSP_REACHED) return bail(st);
    lp0 = zz[2];
    const long long Nl = (zz[3] - zz[2]) * plane;
    if (p->mem == WCSP_MEM_DEVICE) {
      hf1.resize((size_t)d * Nl); hf2.resize((size_t)d * Nl); hA.resize(Nl); hB.resize(Nl);
      if (cudaMemcpy(hf1.data(), p->f1, hf1.size(), cudaMemcpyDeviceToHost) != cudaSuccess ||
          cudaMemcpy(hf2.data(), p->f2, hf2.size(), cudaMemcpyDeviceToHost) != cudaSuccess ||
          cudaMemcpy(hA.data(), p->maskA, Nl, cudaMemcpyDeviceToHost) != cudaSuccess ||
          cudaMemcpy(hB.data(), p->maskB, Nl, cudaMemcpyDeviceToHost) != cudaSuccess)
        return bail(fail(WCSP_ECUDA, "local slab: reading the device arrays failed"));
      if (p->present) {
        hP.resize(Nl);
        if (cudaMemcpy(hP.data(), p->present, Nl, cudaMemcpyDeviceToHost) != cudaSuccess)
          return bail(fail(WCSP_ECUDA, "local slab: reading present failed"));
      }
      lpb.f1 = hf1.data(); lpb.f2 = hf2.data(); lpb.maskA = hA.data(); lpb.maskB = hB.data();
      lpb.present = p->present ? hP.data() : nullptr;
      lpb.mem = WCSP_MEM_HOST;
    }
    unsigned long long c[5];
    local_counts(&lpb, Nl, plane, zz[2], zz[0], zz[1], c);
    NcclApi& nc = nccl_api();
    unsigned long long* dc = nullptr;
    unsigned long long h4[4] = {c[0], c[1], c[2], c[3]}, hm = c[4];
    if (cudaMalloc(&dc, 5 * sizeof(unsigned long long)) != cudaSuccess) return bail(fail(WCSP_ENOMEM, "counts"));
    cudaMemcpy(dc, h4, sizeof(h4), cudaMemcpyHostToDevice);
    cudaMemcpy(dc + 4, &hm, sizeof(hm), cudaMemcpyHostToDevice);
    ncclResult_t r1 = nc.allReduce(dc, dc, 4, ncclUint64, ncclSum, (ncclComm_t)g->comm, g->stream);
    ncclResult_t r2 = nc.allReduce(dc + 4, dc + 4, 1, ncclUint64, ncclMax, (ncclComm_t)g->comm, g->stream);
    cudaStreamSynchronize(g->stream);
    cudaMemcpy(h4, dc, sizeof(h4), cudaMemcpyDeviceToHost);
    cudaMemcpy(&hm, dc + 4, sizeof(hm), cudaMemcpyDeviceToHost);
    cudaFree(dc);
    if (r1 != ncclSuccess || r2 != ncclSuccess) return bail(fail(WCSP_ENCCL, "validation allreduce failed"));
    if (h4[0] == 0) return bail(fail(WCSP_EINVAL, "A is empty (among present vertices)"));
    if (h4[1] == 0) return bail(fail(WCSP_EINVAL, "B is empty (among present vertices)"));
    if (h4[2]) return bail(fail(WCSP_EINVAL, "A and B intersect in %llu vertices", h4[2]));
    if (h4[3]) return bail(fail(WCSP_EINVAL, "%llu present edges have f1 > 0 and f2 = 0", h4[3]));
    nB = h4[1];
    f1max = std::max<int>(1, (int)hm);
  }
  const wcsp_problem* src = local ? &lpb : p;
  for (int i = 0; i < R; ++i) {
    if (dist && i != opt.rank) continue;          // one slab per process
    SlabSpec sp{};
    sp.index = i;
    sp.z0 = (long long)i * nL / R;
    sp.z1 = (long long)(i + 1) * nL / R;
    sp.glo = i > 0;
    sp.ghi = i < R - 1;
    const long long lo = (sp.z0 - sp.glo) * plane, hi = (sp.z1 + sp.ghi) * plane, Nl = hi - lo;
    sp.goff = (unsigned)lo;
    sp.plane = (unsigned)plane;
    sp.nB = nB;
    sp.f1max = f1max;
    sp.per_sm = peer_big ? 4 : 0;
    // the slab's planes in the source arrays: the whole grid's (offset lo) or the local ones (offset
    // lo - lp0 * plane within arrays of SN vertices)
    const long long SN = local ? (long long)(((lo / plane) - lp0) * plane + Nl) : N;
    const long long so = local ? lo - lp0 * plane : lo;
    std::vector<uint8_t> f1((size_t)d * Nl), f2((size_t)d * Nl), A(Nl), B(Nl), ghost(Nl, 0), pres;
    for (int k = 0; k < d; ++k) {
      memcpy(&f1[(size_t)k * Nl], src->f1 + (size_t)k * SN + so, Nl);
      memcpy(&f2[(size_t)k * Nl], src->f2 + (size_t)k * SN + so, Nl);
    }
    memcpy(A.data(), src->maskA + so, Nl);
    memcpy(B.data(), src->maskB + so, Nl);
    if (src->present) { pres.resize(Nl); memcpy(pres.data(), src->present + so, Nl); }
    auto mark_ghost = [&](long long first) {
      for (long long j = first; j < first + plane; ++j) {
        const bool pr = src->present == nullptr || pres[j] != 0;
        ghost[j] = pr ? (B[j] ? 2 : 1) : 0;
        A[j] = 0;
        B[j] = 0;
      }
    };
    if (sp.glo) mark_ghost(0);
    if (sp.ghi) mark_ghost(Nl - plane);
    sp.ghost = ghost.data();
    wcsp_problem lp = *p;
    lp.shape[d - 1] = sp.z1 - sp.z0 + sp.glo + sp.ghi;
    lp.f1 = f1.data(); lp.f2 = f2.data(); lp.maskA = A.data(); lp.maskB = B.data();
    lp.present = src->present ? pres.data() : nullptr;
    lp.mem = WCSP_MEM_HOST;
    wcsp_options co = opt;
    co.slabs = 0;
    co.engine = WCSP_ENGINE_WHEEL_STEPPED;
    co.stream = g->stream;
    wcsp_handle* ch = nullptr;
    if ((st = create_impl(&lp, co, &sp, &ch)) != WCSP_REACHED) return bail(st);
    g->children.push_back(ch);
  }
  std::vector<Ctl*> ctls;
  for (auto* ch : g->children) ctls.push_back(ch->ctl);
  if (cudaMalloc(&g->d_ctls, R * sizeof(Ctl*)) != cudaSuccess ||
      cudaMemcpy(g->d_ctls, ctls.data(), R * sizeof(Ctl*), cudaMemcpyHostToDevice) != cudaSuccess)
    return bail(fail(WCSP_ENOMEM, "slab control array"));
  if (cudaMallocHost(&g->h_ctl, sizeof(Ctl)) != cudaSuccess) return bail(fail(WCSP_ENOMEM, "pinned control block"));
  g->grid = g->children[0]->grid;
  if (opt.halo == WCSP_HALO_PEER) {
    if (!dist && R > MAX_VSLABS) return bail(fail(WCSP_EINVAL, "at most %d virtual slabs with the peer halo", MAX_VSLABS));
    int per_sm = 0, nsm = 0;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, g->dev) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, peer_fn_d(d, peer_big), THREADS, sizeof(Smem)) != cudaSuccess ||
        per_sm < 1)
      return bail(fail(WCSP_ECUDA, "peer-halo kernel cannot be resident"));
    const int per = std::min(g->grid, per_sm * nsm / (dist ? 1 : R));
    if (per < 1) return bail(fail(WCSP_EINVAL, "too many slabs for one device"));
    g->halo = WCSP_HALO_PEER;
    g->big = peer_big;
    g->peer_per = (unsigned)per;
    if (cudaMalloc(&g->xbar, 4 * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMemset(g->xbar, 0, 4 * sizeof(unsigned long long)) != cudaSuccess)
      return bail(fail(WCSP_ENOMEM, "peer barrier"));
    if (dist && (st = peer_connect(g)) != WCSP_REACHED) return bail(st);
  }
  *out = g;
  return WCSP_REACHED;
}

wcsp_status group_collect(wcsp_handle* g, wcsp_result* r, int* status);

// The ghost-plane exchange buffers carry cycle stamps, which restart at every solve (and every
// overflow retry): clear them so no water of an earlier run is applied.
wcsp_status clear_halo(wcsp_handle* c) {
  const size_t pb = (size_t)c->plane;
  for (unsigned long long* b : {c->g_out_lo, c->g_out_hi, c->g_in_lo, c->g_in_hi})
    if (b) CK(cudaMemsetAsync(b, 0, pb * 8, c->stream));
  return WCSP_REACHED;
}
wcsp_status dist_collect(wcsp_handle* g, wcsp_result* r, int* status);

template <int D>
void group_cycle(wcsp_handle* g, const std::vector<Dev>& devs) {
  auto& ch = g->children;
  const int R = (int)ch.size();
  const size_t sm = sizeof(Smem), pl = g->plane;
  const int pg = (int)std::min<unsigned long long>((pl + THREADS - 1) / THREADS, (unsigned long long)g->grid);
  cudaStream_t s = g->stream;
  for (int i = 0; i < R; ++i) k_wheel_fire<D><<<ch[i]->grid, THREADS, sm, s>>>(devs[i]);
  for (int i = 0; i < R; ++i) {   // water that crossed a slab boundary goes to its owner
    if (ch[i]->glo) cudaMemcpyAsync(ch[i - 1]->g_in_hi, ch[i]->g_out_lo, pl * 8, cudaMemcpyDeviceToDevice, s);
    if (ch[i]->ghi) cudaMemcpyAsync(ch[i + 1]->g_in_lo, ch[i]->g_out_hi, pl * 8, cudaMemcpyDeviceToDevice, s);
  }
  for (int i = 0; i < R; ++i) {
    if (ch[i]->glo) k_slab_apply<<<pg, THREADS, 0, s>>>(devs[i], ch[i]->g_in_lo, ch[i]->plane);
    if (ch[i]->ghi) k_slab_apply<<<pg, THREADS, 0, s>>>(devs[i], ch[i]->g_in_hi, ch[i]->ghost_hi_start - ch[i]->plane);
  }
  for (int i = 0; i < R; ++i) k_wheel_treat<D><<<ch[i]->grid, THREADS, sm, s>>>(devs[i]);
  for (int i = 0; i < R; ++i) {   // boundary labels refresh the neighbours' ghost planes
    if (ch[i]->glo) k_slab_gather_labels<<<pg, THREADS, 0, s>>>(devs[i], ch[i]->plane, ch[i]->l_out_lo);
    if (ch[i]->ghi) k_slab_gather_labels<<<pg, THREADS, 0, s>>>(devs[i], ch[i]->ghost_hi_start - ch[i]->plane, ch[i]->l_out_hi);
  }
  for (int i = 0; i < R; ++i) {
    if (ch[i]->glo) cudaMemcpyAsync(ch[i - 1]->l_in_hi, ch[i]->l_out_lo, pl * 4, cudaMemcpyDeviceToDevice, s);
    if (ch[i]->ghi) cudaMemcpyAsync(ch[i + 1]->l_in_lo, ch[i]->l_out_hi, pl * 4, cudaMemcpyDeviceToDevice, s);
  }
  for (int i = 0; i < R; ++i) {
    if (ch[i]->glo) k_slab_scatter_labels<<<pg, THREADS, 0, s>>>(devs[i], ch[i]->l_in_lo, 0u);
    if (ch[i]->ghi) k_slab_scatter_labels<<<pg, THREADS, 0, s>>>(devs[i], ch[i]->l_in_hi, ch[i]->ghost_hi_start);
  }
  for (int i = 0; i < R; ++i) k_slab_propose<<<1, 32, 0, s>>>(devs[i]);
  k_slab_reduce<<<1, 32, 0, s>>>(g->d_ctls, R);
  for (int i = 0; i < R; ++i) k_wheel_decide<<<1, 32, 0, s>>>(devs[i]);
  g->launches += 5 * R + 1 + 4 * (R - 1);
}

wcsp_status group_solve_once(wcsp_handle* g, wcsp_result* r, int* status) {
  wcsp_status st;
  auto& ch = g->children;
  const int R = (int)ch.size();
  g->launches = 0;
  CK(cudaEventRecord(g->e0, g->stream));
  for (auto* c : ch) {
    c->M = g->M;
    if ((st = reset_ctl(c)) != WCSP_REACHED) return st;
    if ((st = clear_halo(c)) != WCSP_REACHED) return st;
    if ((st = launch_init(c)) != WCSP_REACHED) return st;
    g->launches += 1;
  }
  CK(cudaEventRecord(g->em, g->stream));
  std::vector<Dev> devs;
  for (auto* c : ch) devs.push_back(make_dev(c));
  int batch = 4;
  for (;;) {
    for (int i = 0; i < batch; ++i) {
      switch (g->d) {
        case 1: group_cycle<1>(g, devs); break;
        case 2: group_cycle<2>(g, devs); break;
        case 3: group_cycle<3>(g, devs); break;
        default: group_cycle<4>(g, devs); break;
      }
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&g->h_ctl->view, &ch[0]->ctl->view, sizeof(View), cudaMemcpyDeviceToHost, g->stream));
    CK(cudaStreamSynchronize(g->stream));
    const int s0 = g->h_ctl->view.status;
    if (s0 == ST_WRAP) {
      const int run = ST_RUNNING;
      for (int i = 0; i < R; ++i) {
        k_wheel_maintain<<<ch[i]->grid, THREADS, 0, g->stream>>>(devs[i]);
        CK(cudaMemcpyAsync(&ch[i]->ctl->view.status, &run, sizeof(int), cudaMemcpyHostToDevice, g->stream));
      }
      CK(cudaStreamSynchronize(g->stream));
      continue;
    }
    if (s0 != ST_RUNNING) break;
    batch = std::min(batch * 2, 64);
  }
  return group_collect(g, r, status);
}

// Results of a virtual slab group: counters summed over the slabs, Y = min over the slabs.
wcsp_status group_collect(wcsp_handle* g, wcsp_result* r, int* status) {
  auto& ch = g->children;
  const int R = (int)ch.size();
  CK(cudaEventRecord(g->e1, g->stream));
  std::vector<Ctl> cs(R);
  for (int i = 0; i < R; ++i) CK(cudaMemcpyAsync(&cs[i], ch[i]->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, g->stream));
  CK(cudaStreamSynchronize(g->stream));
  float ms = 0, cms = 0;
  CK(cudaEventElapsedTime(&ms, g->e0, g->e1));
  CK(cudaEventElapsedTime(&cms, g->em, g->e1));
  *status = cs[0].view.status;
  memset(r, 0, sizeof(*r));
  unsigned long long ybest = ~0ull;
  long long need = 0;
  for (int i = 0; i < R; ++i) {
    ybest = std::min(ybest, cs[i].ybest);
    r->edge_updates += cs[i].edge_updates;
    r->arrivals += cs[i].arrivals;
    r->triggered += cs[i].triggered;
    r->phantoms_created += cs[i].created;
    r->relabels += cs[i].relabels;
    r->lanes_started += cs[i].started;
    r->peak_phantoms += cs[i].peak_phantoms;
    r->staging_appended += (long long)cs[i].n_appended;
    r->staging_spilled += (long long)cs[i].n_spilled;
    r->staging_singles += (long long)cs[i].n_single;
    ch[i]->last_cycles = cs[i].cycles;
    if (cs[i].need_pool) need = cs[i].need_pool == -2 ? -2 : std::max(need, cs[i].need_pool);
    if (cs[i].abort) return fail(WCSP_ECUDA, "slab %d: barrier watchdog fired", i);
  }
  r->cycles = cs[0].cycles;
  g->last_cycles = cs[0].cycles;
  if (*status == WCSP_REACHED) {
    r->F1 = cs[0].F1;
    r->F2 = cs[0].F2;
    r->X = cs[0].X;
    r->Y = ybest == ~0ull ? -1 : (long long)(ybest >> 1);
    r->via_phantom = (int)(ybest & 1);
    r->x_lane = x_lane_of(g, r->X, r->Y);
  } else {
    r->F1 = r->F2 = r->X = r->Y = -1;
    r->x_lane = -1;
  }
  r->phantom_capacity = *status == WCSP_EOVERFLOW ? need : (long long)ch[0]->ev_cap;
  r->kernel_launches = g->launches;
  r->device_ms = ms;
  r->cycle_ms = cms;
  return WCSP_REACHED;
}

// ---------------------------------------------------------------------------
// NCCL transport of the slab engine (one process per GPU).  NCCL is loaded
// with dlopen on first use (the process normally already holds torch's
// libnccl.so.2), so the library itself does not depend on it.
// ---------------------------------------------------------------------------
void destroy_comm(void* comm) {
  if (comm && nccl_api().ok) nccl_api().commDestroy((ncclComm_t)comm);
}

#define NCK(call)                                                                                       \
  do {                                                                                                  \
    ncclResult_t r_ = (call);                                                                           \
    if (r_ != ncclSuccess) return fail(WCSP_ENCCL, "%s: %s (%s:%d)", #call, nccl_api().errStr(r_), __FILE__, \
                                       __LINE__);                                                       \
  } while (0)

// One cycle of the distributed slab engine (this rank's slab = children[0]).
template <int D>
wcsp_status dist_cycle(wcsp_handle* g, const Dev& dv) {
  NcclApi& nc = nccl_api();
  wcsp_handle* c = g->children[0];
  const size_t sm = sizeof(Smem), pl = g->plane;
  const int pg = (int)std::min<unsigned long long>((pl + THREADS - 1) / THREADS, (unsigned long long)g->grid);
  cudaStream_t s = g->stream;
  ncclComm_t comm = (ncclComm_t)g->comm;
  const int lo = g->rank - 1, hi = g->rank + 1;
  k_wheel_fire<D><<<c->grid, THREADS, sm, s>>>(dv);
  NCK(nc.groupStart());             // water that crossed a slab boundary goes to its owner
  if (c->glo) { NCK(nc.send(c->g_out_lo, pl, ncclUint64, lo, comm, s)); NCK(nc.recv(c->g_in_lo, pl, ncclUint64, lo, comm, s)); }
  if (c->ghi) { NCK(nc.send(c->g_out_hi, pl, ncclUint64, hi, comm, s)); NCK(nc.recv(c->g_in_hi, pl, ncclUint64, hi, comm, s)); }
  NCK(nc.groupEnd());
  if (c->glo) k_slab_apply<<<pg, THREADS, 0, s>>>(dv, c->g_in_lo, c->plane);
  if (c->ghi) k_slab_apply<<<pg, THREADS, 0, s>>>(dv, c->g_in_hi, c->ghost_hi_start - c->plane);
  k_wheel_treat<D><<<c->grid, THREADS, sm, s>>>(dv);
  if (c->glo) k_slab_gather_labels<<<pg, THREADS, 0, s>>>(dv, c->plane, c->l_out_lo);
  if (c->ghi) k_slab_gather_labels<<<pg, THREADS, 0, s>>>(dv, c->ghost_hi_start - c->plane, c->l_out_hi);
  NCK(nc.groupStart());             // boundary labels refresh the neighbours' ghost planes
  if (c->glo) { NCK(nc.send(c->l_out_lo, pl, ncclUint32, lo, comm, s)); NCK(nc.recv(c->l_in_lo, pl, ncclUint32, lo, comm, s)); }
  if (c->ghi) { NCK(nc.send(c->l_out_hi, pl, ncclUint32, hi, comm, s)); NCK(nc.recv(c->l_in_hi, pl, ncclUint32, hi, comm, s)); }
  NCK(nc.groupEnd());
  if (c->glo) k_slab_scatter_labels<<<pg, THREADS, 0, s>>>(dv, c->l_in_lo, 0u);
  if (c->ghi) k_slab_scatter_labels<<<pg, THREADS, 0, s>>>(dv, c->l_in_hi, c->ghost_hi_start);
  k_slab_propose<<<1, 32, 0, s>>>(dv);
  NCK(nc.allReduce(&c->ctl->prop, &c->ctl->gprop, 4, ncclInt64, ncclMax, comm, s));
  k_wheel_decide<<<1, 32, 0, s>>>(dv);
  g->launches += 5 + (c->glo + c->ghi) * 3;
  return WCSP_REACHED;
}

wcsp_status dist_solve_once(wcsp_handle* g, wcsp_result* r, int* status) {
  wcsp_status st;
  wcsp_handle* c = g->children[0];
  g->launches = 0;
  CK(cudaEventRecord(g->e0, g->stream));
  c->M = g->M;
  if ((st = reset_ctl(c)) != WCSP_REACHED) return st;
  if ((st = clear_halo(c)) != WCSP_REACHED) return st;
  if ((st = launch_init(c)) != WCSP_REACHED) return st;
  g->launches += 1;
  CK(cudaEventRecord(g->em, g->stream));
  const Dev dv = make_dev(c);
  int batch = 4;
  for (;;) {
    for (int i = 0; i < batch; ++i) {
      switch (g->d) {
        case 1: st = dist_cycle<1>(g, dv); break;
        case 2: st = dist_cycle<2>(g, dv); break;
        case 3: st = dist_cycle<3>(g, dv); break;
        default: st = dist_cycle<4>(g, dv); break;
      }
      if (st != WCSP_REACHED) return st;
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&g->h_ctl->view, &c->ctl->view, sizeof(View), cudaMemcpyDeviceToHost, g->stream));
    CK(cudaStreamSynchronize(g->stream));
    const int s0 = g->h_ctl->view.status;   // identical on every rank (decisions use the reduced proposal)
    if (s0 == ST_WRAP) {
      k_wheel_maintain<<<c->grid, THREADS, 0, g->stream>>>(dv);
      const int run = ST_RUNNING;
      CK(cudaMemcpyAsync(&c->ctl->view.status, &run, sizeof(int), cudaMemcpyHostToDevice, g->stream));
      CK(cudaStreamSynchronize(g->stream));
      continue;
    }
    if (s0 != ST_RUNNING) break;
    batch = std::min(batch * 2, 64);
  }
  return dist_collect(g, r, status);
}

// Results of the multi-GPU slab engine: totals over the ranks — counters (sum), Y (min),
// overflow need (max) — with three small allreduces.
wcsp_status dist_collect(wcsp_handle* g, wcsp_result* r, int* status) {
  NcclApi& nc = nccl_api();
  wcsp_handle* c = g->children[0];
  ncclComm_t comm = (ncclComm_t)g->comm;
  CK(cudaEventRecord(g->e1, g->stream));
  Ctl cs;
  CK(cudaMemcpyAsync(&cs, c->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, g->stream));
  CK(cudaStreamSynchronize(g->stream));
  long long sums[10] = {cs.edge_updates, cs.arrivals, cs.triggered, cs.created, cs.relabels, cs.started,
                        cs.peak_phantoms, (long long)cs.n_appended, (long long)cs.n_spilled, (long long)cs.n_single};
  unsigned long long mins[2] = {cs.ybest, 0}, maxs[2] = {(unsigned long long)std::max(0ll, cs.need_pool),
                                                         cs.need_pool == -2 ? 1ull : 0ull};
  long long* dsum = nullptr;
  unsigned long long *dmin = nullptr, *dmax = nullptr;
  CK(cudaMalloc(&dsum, sizeof(sums)));
  CK(cudaMalloc(&dmin, sizeof(mins)));
  CK(cudaMalloc(&dmax, sizeof(maxs)));
  CK(cudaMemcpyAsync(dsum, sums, sizeof(sums), cudaMemcpyHostToDevice, g->stream));
  CK(cudaMemcpyAsync(dmin, mins, sizeof(mins), cudaMemcpyHostToDevice, g->stream));
  CK(cudaMemcpyAsync(dmax, maxs, sizeof(maxs), cudaMemcpyHostToDevice, g->stream));
  NCK(nc.allReduce(dsum, dsum, 10, ncclInt64, ncclSum, comm, g->stream));
  NCK(nc.allReduce(dmin, dmin, 2, ncclUint64, ncclMin, comm, g->stream));
  NCK(nc.allReduce(dmax, dmax, 2, ncclUint64, ncclMax, comm, g->stream));
  CK(cudaMemcpyAsync(sums, dsum, sizeof(sums), cudaMemcpyDeviceToHost, g->stream));
  CK(cudaMemcpyAsync(mins, dmin, sizeof(mins), cudaMemcpyDeviceToHost, g->stream));
  CK(cudaMemcpyAsync(maxs, dmax, sizeof(maxs), cudaMemcpyDeviceToHost, g->stream));
  CK(cudaStreamSynchronize(g->stream));
  cudaFree(dsum); cudaFree(dmin); cudaFree(dmax);
  float ms = 0, cms = 0;
  CK(cudaEventElapsedTime(&ms, g->e0, g->e1));
  CK(cudaEventElapsedTime(&cms, g->em, g->e1));
  *status = cs.view.status;
  memset(r, 0, sizeof(*r));
  r->edge_updates = sums[0]; r->arrivals = sums[1]; r->triggered = sums[2]; r->phantoms_created = sums[3];
  r->relabels = sums[4]; r->lanes_started = sums[5]; r->peak_phantoms = sums[6];
  r->staging_appended = sums[7]; r->staging_spilled = sums[8]; r->staging_singles = sums[9];
  r->cycles = cs.cycles;
  c->last_cycles = g->last_cycles = cs.cycles;
  if (*status == WCSP_REACHED) {
    r->F1 = cs.F1; r->F2 = cs.F2; r->X = cs.X;
    r->Y = mins[0] == ~0ull ? -1 : (long long)(mins[0] >> 1);
    r->via_phantom = (int)(mins[0] & 1);
    r->x_lane = x_lane_of(g, r->X, r->Y);
  } else {
    r->F1 = r->F2 = r->X = r->Y = -1;
    r->x_lane = -1;
  }
  r->phantom_capacity = *status == WCSP_EOVERFLOW ? (maxs[1] ? -2 : (long long)maxs[0]) : (long long)c->ev_cap;
  r->kernel_launches = g->launches;
  r->device_ms = ms;
  r->cycle_ms = cms;
  return WCSP_REACHED;
}

// ---------------------------------------------------------------------------
// Peer halo (k_wheel_peer in wcsp_wheel.cuh).
// ---------------------------------------------------------------------------
Dev make_peer_dev(wcsp_handle* g, int i) {
  wcsp_handle* c = g->children[i];
  Dev s = make_dev(c);
  const bool dist = g->comm != nullptr;
  s.peer = 1;
  s.slab = 1;
  s.nblocks = g->peer_per;
  s.win_words = win_words_for(s.nwords, s.nblocks);
  s.ileave = ileave_for(c);
  s.fstride = fstride_for(c);
  s.wbal = getenv("WCSP_WBAL") ? atoi(getenv("WCSP_WBAL")) != 0 : false;   // A/B: neutral on C3, slower on C2
  s.blk0 = dist ? 0u : (unsigned)i * g->peer_per;
  s.plo_end = c->glo ? c->plane : 0u;
  if (dist) {
    for (int k = 0; k < 2; ++k) {
      s.psw[k] = g->peer_sw[k]; s.ptb[k] = g->peer_tb[k];
      s.pshift[k] = g->peer_shift[k]; s.pgoff[k] = g->peer_goff[k];
    }
    s.pctl = g->d_pctl;
    s.nslab = g->nranks;
    s.islab = g->rank;
  } else {
    if (c->glo) {                  // our lower ghost plane = the lower slab's last owned plane
      wcsp_handle* lo = g->children[i - 1];
      s.psw[0] = lo->sw; s.ptb[0] = lo->tbits;
      s.pshift[0] = (unsigned)(lo->N - 2ull * c->plane); s.pgoff[0] = lo->goff;
    }
    if (c->ghi) {                  // our upper ghost plane = the upper slab's first owned plane
      wcsp_handle* hi = g->children[i + 1];
      s.psw[1] = hi->sw; s.ptb[1] = hi->tbits;
      s.pshift[1] = c->plane - c->ghost_hi_start; s.pgoff[1] = hi->goff;
    }
    s.pctl = g->d_ctls;
    s.nslab = (int)g->children.size();
    s.islab = i;
  }
  unsigned long long* xb = g->xbar_ptr ? g->xbar_ptr : g->xbar;
  s.xbar = xb;
  s.xabort = reinterpret_cast<unsigned*>(xb + 1);
  return s;
}

template <int D>
void* peer_fn(bool big) {
  return big ? reinterpret_cast<void*>(&k_wheel_peer<D, 4>) : reinterpret_cast<void*>(&k_wheel_peer<D, 3>);
}
void* peer_fn_d(int d, bool big) {
  return d == 1 ? peer_fn<1>(big) : d == 2 ? peer_fn<2>(big) : d == 3 ? peer_fn<3>(big) : peer_fn<4>(big);
}

wcsp_status peer_solve_once(wcsp_handle* g, wcsp_result* r, int* status) {
  wcsp_status st;
  auto& ch = g->children;
  const int n = (int)ch.size();
  const bool dist = g->comm != nullptr;
  g->launches = 0;
  CK(cudaEventRecord(g->e0, g->stream));
  for (auto* c : ch) {
    c->M = g->M;
    if ((st = reset_ctl(c)) != WCSP_REACHED) return st;
    if ((st = launch_init(c)) != WCSP_REACHED) return st;
    g->launches += 1;
  }
  if (!dist || g->rank == 0) CK(cudaMemsetAsync(g->xbar, 0, 4 * sizeof(unsigned long long), g->stream));
  if (dist) {                      // every rank has reset its state before any rank's kernel starts
    NcclApi& nc = nccl_api();
    NCK(nc.allReduce(g->xbar + 2, g->xbar + 3, 1, ncclUint64, ncclMax, (ncclComm_t)g->comm, g->stream));
  }
  CK(cudaEventRecord(g->em, g->stream));
  DevSet set{};
  set.per = g->peer_per;
  set.n = n;
  for (int i = 0; i < n; ++i) set.d[i] = make_peer_dev(g, i);
  void* args[] = {&set};
  CK(cudaLaunchCooperativeKernel(peer_fn_d(g->d, g->big), dim3(n * g->peer_per), dim3(THREADS), args, sizeof(Smem),
                                 g->stream));
  g->launches += 1;
  return dist ? dist_collect(g, r, status) : group_collect(g, r, status);
}

// Multi-GPU peer halo: map the neighbours' state words and bitmaps, every rank's
// control block and rank 0's barrier counter with CUDA IPC (handles all-gathered
// over NCCL).
struct PeerBlob {
  cudaIpcMemHandle_t sw, tb, ctl, xbar;
  unsigned long long nloc, goff;
};

wcsp_status peer_connect(wcsp_handle* g) {
  NcclApi& nc = nccl_api();
  wcsp_handle* c = g->children[0];
  const int R = g->nranks, me = g->rank;
  PeerBlob mine{};
  CK(cudaIpcGetMemHandle(&mine.sw, c->sw));
  CK(cudaIpcGetMemHandle(&mine.tb, c->tbits));
  CK(cudaIpcGetMemHandle(&mine.ctl, c->ctl));
  CK(cudaIpcGetMemHandle(&mine.xbar, g->xbar));
  mine.nloc = c->N;
  mine.goff = c->goff;
  uint8_t* dbuf = nullptr;
  CK(cudaMalloc(&dbuf, (size_t)(R + 1) * sizeof(PeerBlob)));
  CK(cudaMemcpy(dbuf + (size_t)R * sizeof(PeerBlob), &mine, sizeof(PeerBlob), cudaMemcpyHostToDevice));
  std::vector<PeerBlob> all(R);
  const ncclResult_t nr = nc.allGather(dbuf + (size_t)R * sizeof(PeerBlob), dbuf, sizeof(PeerBlob), ncclUint8,
                                       (ncclComm_t)g->comm, g->stream);
  if (nr != ncclSuccess) { cudaFree(dbuf); return fail(WCSP_ENCCL, "ncclAllGather: %s", nc.errStr(nr)); }
  cudaError_t e = cudaMemcpyAsync(all.data(), dbuf, (size_t)R * sizeof(PeerBlob), cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  cudaFree(dbuf);
  if (e != cudaSuccess) return fail(WCSP_ECUDA, "peer handle exchange: %s", cudaGetErrorString(e));
  auto open = [&](const cudaIpcMemHandle_t& hd, void** p) -> wcsp_status {
    const cudaError_t oe = cudaIpcOpenMemHandle(p, hd, cudaIpcMemLazyEnablePeerAccess);
    if (oe != cudaSuccess)
      return fail(WCSP_ECUDA, "cudaIpcOpenMemHandle: %s (peer access between the GPUs required)",
                  cudaGetErrorString(oe));
    g->ipc_opened.push_back(*p);
    return WCSP_REACHED;
  };
  wcsp_status st;
  std::vector<Ctl*> ctls(R, nullptr);
  for (int r = 0; r < R; ++r) {
    if (r == me) { ctls[r] = c->ctl; continue; }
    void* p = nullptr;
    if ((st = open(all[r].ctl, &p)) != WCSP_REACHED) return st;
    ctls[r] = (Ctl*)p;
  }
  if (me > 0) {
    void *sw = nullptr, *tb = nullptr, *xb = nullptr;
    if ((st = open(all[me - 1].sw, &sw)) != WCSP_REACHED) return st;
    if ((st = open(all[me - 1].tb, &tb)) != WCSP_REACHED) return st;
    if ((st = open(all[0].xbar, &xb)) != WCSP_REACHED) return st;
    g->peer_sw[0] = (unsigned long long*)sw; g->peer_tb[0] = (unsigned*)tb;
    g->peer_shift[0] = (unsigned)(all[me - 1].nloc - 2ull * c->plane);
    g->peer_goff[0] = (unsigned)all[me - 1].goff;
    g->xbar_ptr = (unsigned long long*)xb;
  }
  if (me < R - 1) {
    void *sw = nullptr, *tb = nullptr;
    if ((st = open(all[me + 1].sw, &sw)) != WCSP_REACHED) return st;
    if ((st = open(all[me + 1].tb, &tb)) != WCSP_REACHED) return st;
    g->peer_sw[1] = (unsigned long long*)sw; g->peer_tb[1] = (unsigned*)tb;
    g->peer_shift[1] = c->plane - c->ghost_hi_start;
    g->peer_goff[1] = (unsigned)all[me + 1].goff;
  }
  CK(cudaMalloc(&g->d_pctl, R * sizeof(Ctl*)));
  CK(cudaMemcpy(g->d_pctl, ctls.data(), R * sizeof(Ctl*), cudaMemcpyHostToDevice));
  return WCSP_REACHED;
}

wcsp_status group_solve(wcsp_handle* g, wcsp_result* out) {
  wcsp_result r;
  int status = ST_RUNNING;
  for (int attempt = 0; attempt < MAX_ATTEMPTS; ++attempt) {
    wcsp_status st = g->halo == WCSP_HALO_PEER ? peer_solve_once(g, &r, &status)
                   : g->comm ? dist_solve_once(g, &r, &status) : group_solve_once(g, &r, &status);
    if (st != WCSP_REACHED) return st;
    r.retries = attempt;
    if (status != WCSP_EOVERFLOW) break;
    // grow what overflowed in every slab (same sizes everywhere: the peer kernel's slabs and
    // the ranks share one layout) and re-run: -2 = the run-descriptor table, else the ring
    // slots the largest slab needed
    const long long need = r.phantom_capacity;
    for (auto* c : g->children) {
      if (need == -2) st = alloc_desc(c, c->dcap * 2);
      else st = alloc_ring(c, grown(c->ev_cap, need));
      if (st != WCSP_REACHED) return st;
    }
  }
  if (status == WCSP_EOVERFLOW) return fail(WCSP_EOVERFLOW, "event storage overflow after retries");
  if (status == WCSP_EBUDGET) { *out = r; return fail(WCSP_EBUDGET, "cycle budget %lld exceeded", g->opt.cycle_budget); }
  if (status != WCSP_REACHED && status != WCSP_INFEASIBLE) return fail(WCSP_ECUDA, "solver ended in state %d", status);
  *out = r;
  return (wcsp_status)status;
}
}  // namespace

extern "C" {

const char* wcsp_last_error(void) { return g_err.c_str(); }

const char* wcsp_version(void) {
  return "wcsp-b200 0.4 (sm_100a; engines: sweep/wheel x persistent/stepped, one-barrier hybrid wheel; wide labels; slab partition)";
}

wcsp_status wcsp_create(const wcsp_problem* p, const wcsp_options* o, wcsp_handle** out) {
  if (!p || !out) return fail(WCSP_EINVAL, "problem and out must be non-NULL");
  if (p->d < 1 || p->d > 4) return fail(WCSP_EINVAL, "d = %d outside 1..4", p->d);
  unsigned long long N = 1;
  for (int k = 0; k < p->d; ++k) {
    if (p->shape[k] < 1) return fail(WCSP_EINVAL, "shape[%d] = %lld < 1", k, (long long)p->shape[k]);
    N *= (unsigned long long)p->shape[k];
    if (N > (1ull << 30)) return fail(WCSP_EINVAL, "N > 2^30 vertices");
  }
  wcsp_status st;
  if ((st = check_M(p->M)) != WCSP_REACHED) return st;
  wcsp_options opt{};
  if (o) opt = *o;
  if (opt.demote_twin) return fail(WCSP_EINVAL, "demote_twin is reserved in this version (must be 0)");
  if (opt.time_mode != WCSP_JUMP && opt.time_mode != WCSP_UNIT) return fail(WCSP_EINVAL, "bad time_mode");
  if (opt.engine < WCSP_ENGINE_PERSISTENT || opt.engine > WCSP_ENGINE_WHEEL_STEPPED)
    return fail(WCSP_EINVAL, "bad engine %d", opt.engine);
  if (opt.trace_cap < 0 || opt.cycle_budget < 0 || opt.phantom_capacity < 0) return fail(WCSP_EINVAL, "negative option");
  if (opt.halo != WCSP_HALO_COPY && opt.halo != WCSP_HALO_PEER) return fail(WCSP_EINVAL, "bad halo %d", opt.halo);

  if (opt.slabs > 1 || opt.nranks > 1 || opt.nccl_id) return create_group(p, opt, out);
  return create_impl(p, opt, nullptr, out);
}

wcsp_status wcsp_load(wcsp_handle* h, const wcsp_problem* p) {
  if (!h || !p) return fail(WCSP_EINVAL, "NULL argument");
  if (!h->children.empty()) return fail(WCSP_EINVAL, "wcsp_load: create a new slab handle instead");
  if (p->d != h->d) return fail(WCSP_EINVAL, "d differs from the handle's");
  for (int k = 0; k < h->d; ++k)
    if (p->shape[k] != h->shape[k]) return fail(WCSP_EINVAL, "shape differs from the handle's");
  CK(cudaSetDevice(h->dev));
  return load_problem(h, p);
}

wcsp_status wcsp_solve(wcsp_handle* h, wcsp_result* r) {
  if (!h || !r) return fail(WCSP_EINVAL, "NULL argument");
  CK(cudaSetDevice(h->dev));
  if (!h->children.empty()) return group_solve(h, r);
  return solve_impl(h, r);
}

wcsp_status wcsp_set_targets(wcsp_handle* h, const uint8_t* maskB, const uint8_t* present, int32_t present_all,
                             int64_t M, int32_t mem) {
  if (!h) return fail(WCSP_EINVAL, "NULL handle");
  wcsp_status st;
  if ((st = check_M(M)) != WCSP_REACHED) return st;
  if (!h->children.empty()) {
    if (maskB || present || present_all) return fail(WCSP_EINVAL, "slab handles only change M");
    if (wide_M(M)) return fail(WCSP_EINVAL, "slab engine: M > %d (wide labels) is single-device only", WCSP_M_MAX);
    h->M = M;
    return WCSP_REACHED;
  }
  CK(cudaSetDevice(h->dev));
  if (maskB && (st = copy_mask(h, h->d_maskB, maskB, mem)) != WCSP_REACHED) return st;
  if (present_all) h->present_all = true;
  else if (present) {
    if ((st = copy_mask(h, h->d_present, present, mem)) != WCSP_REACHED) return st;
    h->present_all = false;
  }
  h->M = M;
  CK(cudaStreamSynchronize(h->stream));
  return WCSP_REACHED;
}

wcsp_status wcsp_trace(wcsp_handle* h, wcsp_trace_rec* out, int64_t cap, int64_t* n) {
  if (!h || !n) return fail(WCSP_EINVAL, "NULL argument");
  const long long avail = std::min<long long>(h->last_cycles, h->opt.trace_cap);
  const long long m = std::min<long long>(avail, cap);
  static_assert(sizeof(TraceRec) == sizeof(wcsp_trace_rec), "trace record layout");
  if (m > 0 && !h->children.empty()) {     // slab group: per-cycle sums over the slabs
    std::vector<TraceRec> acc((size_t)m), one((size_t)m);
    for (size_t i = 0; i < h->children.size(); ++i) {
      CK(cudaMemcpyAsync(i ? one.data() : acc.data(), h->children[i]->trace, m * sizeof(TraceRec),
                         cudaMemcpyDeviceToHost, h->stream));
      CK(cudaStreamSynchronize(h->stream));
      if (i)
        for (long long j = 0; j < m; ++j) {
          acc[j].live_lanes += one[j].live_lanes; acc[j].phantoms += one[j].phantoms;
          acc[j].triggered += one[j].triggered; acc[j].arrivals += one[j].arrivals;
          acc[j].created += one[j].created; acc[j].relabels += one[j].relabels; acc[j].tested += one[j].tested;
          acc[j].active_vertices += one[j].active_vertices;
        }
    }
    memcpy(out, acc.data(), m * sizeof(TraceRec));
  } else if (m > 0) {
    CK(cudaMemcpyAsync(out, h->trace, m * sizeof(TraceRec), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  }
  *n = m;
  return WCSP_REACHED;
}

// Reconstruction (reading R12 in DESIGN.md).
wcsp_status wcsp_reconstruct(wcsp_handle* h, int64_t* path, int64_t cap, int64_t* len, wcsp_result* result) {
  if (!h || !len) return fail(WCSP_EINVAL, "NULL argument");
  if (!h->children.empty()) return fail(WCSP_EINVAL, "wcsp_reconstruct is not available on slab handles");
  CK(cudaSetDevice(h->dev));
  const unsigned long long N = h->N;
  wcsp_result first;
  wcsp_status st = solve_impl(h, &first);
  if (st != WCSP_REACHED) return st;
  // host views of what the driver needs: A, B, present, and the edge values at each step
  std::vector<uint8_t> A(N), B(N), pres(N, 1);
  CK(cudaMemcpyAsync(A.data(), h->d_maskA, N, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaMemcpyAsync(B.data(), h->d_maskB, N, cudaMemcpyDeviceToHost, h->stream));
  if (!h->present_all) CK(cudaMemcpyAsync(pres.data(), h->d_present, N, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  const bool saved_all = h->present_all;
  const long long saved_M = h->M;
  std::vector<uint8_t> pres0 = pres;
  std::vector<int64_t> rev;   // X, then predecessors
  rev.push_back(first.X);
  long long X = first.X, Y = first.Y, F1 = first.F1, F2 = first.F2;
  // V' = V \ B: remove every target
  std::vector<uint8_t> work = pres;
  for (unsigned long long v = 0; v < N; ++v)
    if (B[v]) work[v] = 0;
  std::vector<uint8_t> onlyY(N, 0);
  auto edge_f = [&](long long u, long long v, int* f1, int* f2) -> wcsp_status {
    const int lane = x_lane_of(h, u, v);   // weight record of u, lane toward v
    if (lane < 0) return fail(WCSP_EMISMATCH, "reconstruction: %lld and %lld are not lattice neighbours", u, v);
    const size_t lb = lane_bytes(h->d);
    unsigned char rec[16];
    CK(cudaMemcpy(rec, (const char*)h->wt + (size_t)u * 2 * lb, 2 * lb, cudaMemcpyDeviceToHost));
    *f1 = rec[lane];
    *f2 = rec[lb + lane];
    return WCSP_REACHED;
  };
  wcsp_status out = WCSP_REACHED;
  while (!A[(size_t)Y]) {
    if ((long long)rev.size() > (long long)N) { out = fail(WCSP_EMISMATCH, "reconstruction does not terminate"); break; }
    int f1x = 0, f2x = 0;
    if ((out = edge_f(Y, X, &f1x, &f2x)) != WCSP_REACHED) break;
    // B' = {Y}, M' = F2 - f2(x) + 1 (reading R12), V' = V \ (B u earlier targets)
    std::fill(onlyY.begin(), onlyY.end(), 0);
    onlyY[(size_t)Y] = 1;
    const long long Mp = saved_M == WCSP_M_INF ? WCSP_M_INF : F2 - f2x + 1;
    CK(cudaMemcpyAsync(h->d_maskB, onlyY.data(), N, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->d_present, work.data(), N, cudaMemcpyHostToDevice, h->stream));
    h->present_all = false;
    h->M = Mp;
    wcsp_result r;
    st = solve_impl(h, &r);
    h->M = saved_M;
    if (st != WCSP_REACHED) { out = fail(WCSP_EMISMATCH, "re-solve toward %lld returned status %d", Y, (int)st); break; }
    const long long want1 = F1 - f1x, want2 = saved_M == WCSP_M_INF ? -1 : F2 - f2x;
    if (r.F1 != want1 || r.F2 != want2 || r.X != Y) {
      out = fail(WCSP_EMISMATCH, "re-solve toward %lld gave (F1, F2) = (%lld, %lld), expected (%lld, %lld)", Y,
                 (long long)r.F1, (long long)r.F2, want1, want2);
      break;
    }
    rev.push_back(Y);
    work[(size_t)Y] = 0;
    X = Y; Y = r.Y; F1 = r.F1; F2 = r.F2;
  }
  if (out == WCSP_REACHED) rev.push_back(Y);
  // restore the loaded problem
  CK(cudaMemcpyAsync(h->d_maskB, B.data(), N, cudaMemcpyHostToDevice, h->stream));
  if (!saved_all) CK(cudaMemcpyAsync(h->d_present, pres0.data(), N, cudaMemcpyHostToDevice, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  h->present_all = saved_all;
  h->M = saved_M;
  if (out != WCSP_REACHED) return out;
  *len = (int64_t)rev.size();
  if (result) *result = first;
  if (!path || cap < (int64_t)rev.size()) return fail(WCSP_EINVAL, "path capacity %lld < %lld", (long long)cap, (long long)rev.size());
  for (size_t i = 0; i < rev.size(); ++i) path[i] = rev[rev.size() - 1 - i];
  return WCSP_REACHED;
}

wcsp_status wcsp_validate_path(const wcsp_problem* p, const int64_t* path, int64_t len, int64_t* F1, int64_t* F2) {
  if (!p || !path || len < 2 || p->mem != WCSP_MEM_HOST) return fail(WCSP_EINVAL, "bad arguments");
  long long N = 1, st[4] = {1, 1, 1, 1};
  for (int k = 0; k < p->d; ++k) { st[k] = N; N *= p->shape[k]; }
  auto present = [&](long long v) { return p->present == nullptr || p->present[v] != 0; };
  for (int64_t i = 0; i < len; ++i)
    if (path[i] < 0 || path[i] >= N || !present(path[i])) return fail(WCSP_EINVAL, "path[%lld] invalid", (long long)i);
  if (!p->maskA[path[0]]) return fail(WCSP_EINVAL, "path does not start in A");
  if (!p->maskB[path[len - 1]]) return fail(WCSP_EINVAL, "path does not end in B");
  long long s1 = 0, s2 = 0;
  for (int64_t i = 0; i + 1 < len; ++i) {
    const long long u = std::min(path[i], path[i + 1]), v = std::max(path[i], path[i + 1]);
    int k = -1;
    for (int j = 0; j < p->d; ++j)
      if (v - u == st[j] && (u / st[j]) % p->shape[j] + 1 < p->shape[j]) k = j;
    if (k < 0 || p->f1[(size_t)k * N + u] == 0) return fail(WCSP_EINVAL, "no edge between path[%lld] and path[%lld]", (long long)i, (long long)i + 1);
    s1 += p->f1[(size_t)k * N + u];
    s2 += p->f2[(size_t)k * N + u];
  }
  *F1 = s1;
  *F2 = s2;
  if (p->M != WCSP_M_INF && s2 >= p->M) return WCSP_INFEASIBLE;
  return WCSP_REACHED;
}

wcsp_status wcsp_staircase(wcsp_handle* h, int64_t M_max, int64_t f2_stop, int64_t* steps, int64_t cap,
                           int64_t* n, wcsp_result* result) {
  if (!h || !n || (cap > 0 && !steps)) return fail(WCSP_EINVAL, "NULL argument");
  if (!h->children.empty() || !is_wheel(h->opt.engine))
    return fail(WCSP_EINVAL, "wcsp_staircase needs a single-device wheel-engine handle");
  wcsp_status st;
  if ((st = check_M(M_max)) != WCSP_REACHED) return st;
  if (wide_M(M_max)) return fail(WCSP_EINVAL, "wcsp_staircase: M_max > %d needs the wide-label sweep engine "
                                               "(the staircase runs on the 16-bit wheel engine)", WCSP_M_MAX);
  CK(cudaSetDevice(h->dev));
  const unsigned want = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cap, 1 << 24));
  if (want > h->stair_cap) {
    if (h->stair) cudaFree(h->stair);
    h->stair = nullptr;
    h->stair_cap = 0;
    CK(cudaMalloc(&h->stair, (size_t)want * 4 * sizeof(long long)));
    h->stair_cap = want;
  }
  const long long saved_M = h->M;
  h->M = M_max;
  h->staircase = 1;
  h->f2stop = M_max == WCSP_M_INF ? (1ll << 62) : f2_stop;   // M = inf: every arrival has F2 = -1
  wcsp_result r;
  st = solve_impl(h, &r);
  h->staircase = 0;
  h->M = saved_M;
  if (st != WCSP_REACHED && st != WCSP_INFEASIBLE) return st;
  const long long k = h->h_ctl->n_stair;
  *n = k;
  const long long m = std::min<long long>(k, std::min<int64_t>(cap, h->stair_cap));
  if (m > 0) {
    CK(cudaMemcpy(steps, h->stair, (size_t)m * 4 * sizeof(long long), cudaMemcpyDeviceToHost));
  }
  if (result) *result = r;
  return st;
}

wcsp_status wcsp_slab_planes(int64_t n_last, int32_t nranks, int32_t rank, int64_t* out4) {
  if (!out4 || nranks < 1 || rank < 0 || rank >= nranks || n_last < nranks)
    return fail(WCSP_EINVAL, "slab planes: need 0 <= rank < nranks <= n_last (got %d, %d, %lld)", rank, nranks,
                (long long)n_last);
  out4[0] = (int64_t)rank * n_last / nranks;
  out4[1] = (int64_t)(rank + 1) * n_last / nranks;
  out4[2] = out4[0] - (rank > 0 ? 1 : 0);
  out4[3] = out4[1] + (rank < nranks - 1 ? 1 : 0);
  return WCSP_REACHED;
}

static wcsp_status gen_shape(int32_t d, const int64_t* shape, int64_t z0, int64_t z1, GenShape* g) {
  if (d < 1 || d > 4 || !shape) return fail(WCSP_EINVAL, "d = %d outside 1..4 (or shape NULL)", d);
  g->d = d;
  long long N = 1;
  for (int k = 0; k < 4; ++k) {
    g->n[k] = k < d ? shape[k] : 1;
    if (g->n[k] < 1) return fail(WCSP_EINVAL, "shape[%d] < 1", k);
    N *= g->n[k];
  }
  if (N > (1ll << 30)) return fail(WCSP_EINVAL, "N > 2^30 vertices");
  const long long nL = g->n[d - 1];
  if (z1 < 0) z1 = nL;
  if (z0 < 0 || z0 > z1 || z1 > nL) return fail(WCSP_EINVAL, "plane range [%lld, %lld) outside [0, %lld]", z0, z1, nL);
  g->plane = N / nL;
  g->v0 = z0 * g->plane;
  g->Nl = (z1 - z0) * g->plane;
  return WCSP_REACHED;
}

wcsp_status wcsp_generate_grid(int32_t d, const int64_t* shape, uint64_t seed, int32_t lo, int32_t hi, int64_t z0,
                               int64_t z1, uint8_t* f1, uint8_t* f2, void* stream) {
  GenShape g;
  wcsp_status st;
  if ((st = gen_shape(d, shape, z0, z1, &g)) != WCSP_REACHED) return st;
  if (lo < 1 || hi < lo || hi > 255) return fail(WCSP_EINVAL, "value range [%d, %d] outside 1..255", lo, hi);
  if (g.Nl == 0) return WCSP_REACHED;           // an empty plane range writes nothing
  if (!f1 || !f2) return fail(WCSP_EINVAL, "f1 and f2 must be device pointers");
  const int blocks = (int)std::min<long long>((g.Nl + 255) / 256, 148ll * 16);
  k_gen_grid<<<blocks, 256, 0, (cudaStream_t)stream>>>(g, splitmix64(seed), (unsigned)lo, (unsigned)(hi - lo + 1), f1, f2);
  CK(cudaGetLastError());
  return WCSP_REACHED;
}

wcsp_status wcsp_generate_mask(int32_t d, const int64_t* shape, int32_t rule, int64_t z0, int64_t z1, uint8_t* out,
                               void* stream) {
  GenShape g;
  wcsp_status st;
  if ((st = gen_shape(d, shape, z0, z1, &g)) != WCSP_REACHED) return st;
  if (rule < WCSP_SET_FACE0 || rule > WCSP_SET_CORNER1) return fail(WCSP_EINVAL, "bad set rule %d", rule);
  if (g.Nl == 0) return WCSP_REACHED;
  if (!out) return fail(WCSP_EINVAL, "out must be a device pointer");
  const int blocks = (int)std::min<long long>((g.Nl + 255) / 256, 148ll * 16);
  k_gen_mask<<<blocks, 256, 0, (cudaStream_t)stream>>>(g, rule, out);
  CK(cudaGetLastError());
  return WCSP_REACHED;
}

wcsp_status wcsp_nccl_unique_id(uint8_t* out128) {
  if (!out128) return fail(WCSP_EINVAL, "NULL argument");
  if (!nccl_api().ok) return fail(WCSP_ENCCL, "cannot load libnccl.so.2 (set WCSP_NCCL_LIB)");
  ncclUniqueId id;
  const ncclResult_t r = nccl_api().getUniqueId(&id);
  if (r != ncclSuccess) return fail(WCSP_ENCCL, "ncclGetUniqueId: %s", nccl_api().errStr(r));
  memcpy(out128, &id, sizeof(id));
  return WCSP_REACHED;
}

void wcsp_destroy(wcsp_handle* h) {
  if (!h) return;
  cudaSetDevice(h->dev);
  if (h->stream) cudaStreamSynchronize(h->stream);
  release(h);
  delete h;
}

}  // extern "C"
