// wcsp_device.cuh — device state, phase functions and kernels of the B200
// (sm_100a) active-vertex label-correcting sweep (§4, :155-227).
//
// One cycle, c = 1, 2, ...:
//   sweep  : Step 1 and Step 3 (:173) — every live lane of every
//            active vertex and every live phantom counts down by Delta; the ones
//            reaching 0 deliver water (cand = label - f2) to their destination
//            D with one 32-bit atomicMax on D's temporary label (Step 2,
//            :166-168; the "temporary replacement label" of :133).  The
//            first arrival of the cycle appends D to the triggered list (the
//            dedupe of :164).  Survivors are compacted into the next active
//            list / phantom pool (Steps 7-9, :207-227), block-aggregated.
//   treat  : Steps 4, 5 and 8.1 (:176-198, :211) for every triggered Q whose
//            temporary label beats its label (:32): an edge Q->R is triggered
//            iff L* - f2 > max(L(R), temp(R)) (:180); if Q has no live lane
//            (inactive, :189) the lane restarts with f1 (:190-192) and
//            L(Q) := L*; otherwise a phantom (Q, R, L*, f1) is created
//            (:197-198).  L* = temp(Q) (reading R23).
//   decide : Step 6 (:204) — termination 1° (:124) / 2° (:126); Delta for the
//            next cycle = min live residual (time skipping, :75, :95).
// c = 0 is the initial state: A is triggered with temp M
// and treated (reading R20).
//
// Vertex state word sw[v] (u64): low u32 = label L(v) (16 bits used), high
// u32 = temp = stamp:16 | cand:16, valid only when stamp == this cycle's.
// Targets (B) and removed vertices carry a sentinel temp with stamp 0xFFFF
// that an atomicMax never overwrites, so an arrival learns what D is from the
// atomic's return value alone.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace wcspk {

constexpr int THREADS = 256;
constexpr int SWEEP_ITEMS = 4;           // items per thread per chunk, sweep (unrolled for MLP)
constexpr int TREAT_ITEMS = 2;           // items per thread per chunk, treat
constexpr int QCAP = THREADS * SWEEP_ITEMS;   // shared-memory queue capacity (overflow -> direct global append)

constexpr unsigned LBL_REMOVED = 0xFFFFu;  // label of a vertex outside G': no S6 test passes
constexpr unsigned TMP_B = 0xFFFF0001u;    // temp sentinel of a target vertex
constexpr unsigned TMP_REMOVED = 0xFFFF0000u;
constexpr int ST_RUNNING = -1;
constexpr int ST_WRAP = 100;               // stepped engine: temp stamps wrapped, host clears temps

// phantom record (u64): src 30 | lane 3 | cand 16 | res 8  (cand = L* - f2(e), fixed at creation)
constexpr int PH_LANE = 30, PH_CAND = 33, PH_RES = 49;
constexpr unsigned STAMP_PERIOD = 65534u;  // stamps 1..0xFFFE; 0xFFFF is the sentinel

struct BArr { unsigned D, cand, src, via; };   // an arrival at a target (terminating cycle only)

struct Acc {                       // per-cycle accumulators, triple-buffered by cycle % 3
  unsigned n_act;                  // entries appended to the next active list
  unsigned n_pool;                 // phantoms appended to the next pool (may exceed capacity)
  unsigned n_trig;                 // vertices appended to the triggered list (first arrivals)
  unsigned dmin;                   // min live residual after this cycle (0xFFFFFFFF = nothing live)
  unsigned long long bhit;         // max over B arrivals of (cand << 32 | ~X)
  unsigned long long live;         // live lanes at the top of the cycle (E)
  unsigned long long arrivals, created, relabels, triggered;
  long long pend_lanes, pend_phantoms;   // timing wheel: events in flight at the top of this cycle
};

struct View {                      // cycle state every block needs
  long long t;
  unsigned c, stamp, delta, n_act, n_pool;
  int cur, status;
  unsigned region, pad_;           // timing wheel: ring region size per (block, delay)
};

struct Ctl {
  View view;
  Acc acc[3];
  unsigned long long bar;          // grid barrier arrivals (persistent engine)
  unsigned abort, n_barr;          // barrier watchdog fired; B-arrival list length
  long long F1, F2, X, Y;
  long long via;
  long long cycles, edge_updates, arrivals, triggered, created, relabels;
  long long peak_active, peak_phantoms, need_pool;
  // timing-wheel engine (wcsp_wheel.cuh)
  unsigned long long ev_head;      // logical allocation head of the event ring
  unsigned wheel_overflow, pad2_;  // 2: descriptor table full
  long long hist_t[256];           // time of cycle c (by c & 255) ...
  unsigned long long hist_head[256];     // ... and the ring head before its treat
};

struct TraceRec { long long t, delta, active_vertices, live_lanes, phantoms, triggered, arrivals, created, relabels; };

struct Dev {
  unsigned N;
  int NL;                          // lanes per vertex = 2d
  unsigned off[8];                 // lane 2k: +stride_k, lane 2k+1: -stride_k (mod 2^32)
  const void* wt;                  // weight records (f1 lane word, f2 lane word) per vertex
  void* res;                       // lane residual words, 0 = idle lane
  unsigned long long* sw;          // vertex state words (label | temp)
  unsigned* act[2];
  unsigned* trig;
  unsigned long long* pool[2];
  unsigned long long pool_cap;
  BArr* barr;
  unsigned barr_cap;
  Ctl* ctl;
  TraceRec* trace;
  long long trace_cap;
  long long budget;
  int unit, minf, M;
  // timing-wheel engine
  unsigned long long* ev;          // event ring (power-of-two capacity)
  unsigned long long ev_mask;
  unsigned long long* bdesc;       // [256][dcap] run descriptors (pos << 24 | count)
  unsigned* bndesc;                // [256] descriptors per bucket
  unsigned* bnev;                  // [256] events per bucket
  unsigned* bnlane;                // [256] lane events per bucket
  unsigned dcap;
  int f1max;
};

template <int D> struct Tr;
template <> struct Tr<1> { using LW = uint32_t; };
template <> struct Tr<2> { using LW = uint32_t; };
template <> struct Tr<3> { using LW = unsigned long long; };
template <> struct Tr<4> { using LW = unsigned long long; };

__host__ __device__ constexpr unsigned stamp_of(unsigned c) { return (c % STAMP_PERIOD) + 1u; }

__device__ __forceinline__ unsigned* tmp_ptr(unsigned long long* sw, unsigned v) {
  return reinterpret_cast<unsigned*>(sw + v) + 1;
}
__device__ __forceinline__ unsigned* lbl_ptr(unsigned long long* sw, unsigned v) {
  return reinterpret_cast<unsigned*>(sw + v);
}

// ---------------------------------------------------------------------------
// SWAR helpers on lane words (one byte per lane)
// ---------------------------------------------------------------------------
template <class LW> __device__ __forceinline__ LW rep(unsigned b) {
  return (LW)b * (sizeof(LW) == 8 ? (LW)0x0101010101010101ull : (LW)0x01010101u);
}
// 0x80 in every nonzero byte
template <class LW> __device__ __forceinline__ LW nzb(LW w) {
  const LW lo7 = rep<LW>(0x7F), hi = rep<LW>(0x80);
  return (w | ((w & lo7) + lo7)) & hi;
}
template <class LW> __device__ __forceinline__ int popc_lw(LW x) {
  if constexpr (sizeof(LW) == 8) return __popcll(x); else return __popc(x);
}
template <int D, class LW> __device__ __forceinline__ unsigned min_nonzero_byte(LW w) {
  unsigned m = 0xFFFFFFFFu;
#pragma unroll
  for (int j = 0; j < 2 * D; ++j) {
    const unsigned b = (unsigned)(w >> (8 * j)) & 0xFFu;
    if (b) m = min(m, b);
  }
  return m;
}

template <class LW> struct WRec { LW f1, f2; };

template <int D> __device__ __forceinline__ WRec<typename Tr<D>::LW> load_wt(const Dev& s, unsigned v) {
  using LW = typename Tr<D>::LW;
  WRec<LW> r;
  if constexpr (sizeof(LW) == 4) {
    uint2 q = __ldg(reinterpret_cast<const uint2*>(s.wt) + v);
    r.f1 = q.x; r.f2 = q.y;
  } else {
    uint4 q = __ldg(reinterpret_cast<const uint4*>(s.wt) + v);
    r.f1 = ((unsigned long long)q.y << 32) | q.x;
    r.f2 = ((unsigned long long)q.w << 32) | q.z;
  }
  return r;
}
template <int D> __device__ __forceinline__ typename Tr<D>::LW load_f2(const Dev& s, unsigned v) {
  if constexpr (sizeof(typename Tr<D>::LW) == 4) {
    return __ldg(reinterpret_cast<const unsigned*>(s.wt) + 2 * (size_t)v + 1);
  } else {
    return __ldg(reinterpret_cast<const unsigned long long*>(s.wt) + 2 * (size_t)v + 1);
  }
}

// ---------------------------------------------------------------------------
// Block-local append queues (shared memory), flushed with one global atomic
// per queue per chunk
// ---------------------------------------------------------------------------
struct Smem {
  unsigned q32[QCAP];              // active-vertex appends
  unsigned qt[QCAP];               // triggered-vertex appends
  unsigned long long qp[QCAP];     // phantom appends
  unsigned na, nt, np;
  unsigned base_a, base_b, flag;
  View view;
  unsigned long long bhit;
  unsigned long long red[THREADS / 32][5];
  unsigned redmin[THREADS / 32];
};

template <class T>
__device__ __forceinline__ void qpush(T* qbuf, unsigned* qn, bool pred, T x, unsigned* gcount, T* out,
                                      unsigned long long cap) {
  const unsigned m = __ballot_sync(0xFFFFFFFFu, pred);
  if (m == 0) return;
  const unsigned lane = threadIdx.x & 31u;
  const int leader = __ffs(m) - 1;
  unsigned base = 0;
  if ((int)lane == leader) base = atomicAdd(qn, (unsigned)__popc(m));
  base = __shfl_sync(0xFFFFFFFFu, base, leader);
  if (pred) {
    const unsigned idx = base + __popc(m & ((1u << lane) - 1u));
    if (idx < (unsigned)QCAP) {
      qbuf[idx] = x;
    } else {                        // rare: queue full, append straight to the global list
      const unsigned long long pos = atomicAdd(gcount, 1u);
      if (pos < cap) out[pos] = x;
    }
  }
}

// Flush two queues with one reservation round (3 block barriers per chunk).
template <class TA, class TB>
__device__ __forceinline__ void qflush2(TA* qa, unsigned* na_s, unsigned* ga, TA* outa, unsigned long long capa,
                                        TB* qb, unsigned* nb_s, unsigned* gb, TB* outb, unsigned long long capb,
                                        Smem& sm) {
  __syncthreads();
  const unsigned na = min(*na_s, (unsigned)QCAP), nb = min(*nb_s, (unsigned)QCAP);
  if (threadIdx.x == 0) {
    sm.base_a = na ? atomicAdd(ga, na) : 0u;
    sm.base_b = nb ? atomicAdd(gb, nb) : 0u;
  }
  __syncthreads();
  const unsigned long long ba = sm.base_a, bb = sm.base_b;
  for (unsigned i = threadIdx.x; i < na; i += THREADS)
    if (ba + i < capa) outa[ba + i] = qa[i];
  for (unsigned i = threadIdx.x; i < nb; i += THREADS)
    if (bb + i < capb) outb[bb + i] = qb[i];
  if (threadIdx.x == 0) { *na_s = 0; *nb_s = 0; }   // no push can happen before the barrier below
  __syncthreads();
}

// block reductions -> one global atomic per counter per block
__device__ __forceinline__ void block_reduce_commit(Smem& sm, unsigned dmin, unsigned long long a0,
                                                    unsigned long long a1, unsigned long long a2,
                                                    unsigned long long a3, unsigned long long a4, Acc* acc) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dmin = min(dmin, __shfl_xor_sync(0xFFFFFFFFu, dmin, o));
    a0 += __shfl_xor_sync(0xFFFFFFFFu, a0, o);
    a1 += __shfl_xor_sync(0xFFFFFFFFu, a1, o);
    a2 += __shfl_xor_sync(0xFFFFFFFFu, a2, o);
    a3 += __shfl_xor_sync(0xFFFFFFFFu, a3, o);
    a4 += __shfl_xor_sync(0xFFFFFFFFu, a4, o);
  }
  const unsigned w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sm.redmin[w] = dmin;
    sm.red[w][0] = a0; sm.red[w][1] = a1; sm.red[w][2] = a2; sm.red[w][3] = a3; sm.red[w][4] = a4;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned m = 0xFFFFFFFFu;
    unsigned long long s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0;
    for (int i = 0; i < THREADS / 32; ++i) {
      m = min(m, sm.redmin[i]);
      s0 += sm.red[i][0]; s1 += sm.red[i][1]; s2 += sm.red[i][2]; s3 += sm.red[i][3]; s4 += sm.red[i][4];
    }
    if (m != 0xFFFFFFFFu) atomicMin(&acc->dmin, m);
    if (s0) atomicAdd(&acc->live, s0);
    if (s1) atomicAdd(&acc->arrivals, s1);
    if (s2) atomicAdd(&acc->created, s2);
    if (s3) atomicAdd(&acc->relabels, s3);
    if (s4) atomicAdd(&acc->triggered, s4);
  }
  __syncthreads();
}

// Water of quality `cand` reaches D from `src` (quality <= 0
// cannot travel, :29): temp(D) := max(temp(D), cand) — one atomic whose
// return value says whether D is a target, removed, or triggered for the
// first time this cycle.  The comparison with L(D) ("L(S) - f2(e) > L(D)",
// :32) is made once per triggered vertex in treat: max over all arrivals
// beats L(D) iff max over the accepted ones does, and then they are equal.
// Must be called by all 32 lanes of the warp (warp-aggregated queue push).
__device__ __forceinline__ void arrive(const Dev& s, const View& v, Acc* acc, Smem& sm, bool go, unsigned D,
                                       int cand, unsigned src, unsigned via) {
  go = go && cand > 0;
  bool first = false;
  if (go) {
    const unsigned old = atomicMax(tmp_ptr(s.sw, D), (v.stamp << 16) | (unsigned)cand);
    const unsigned os = old >> 16;
    if (os == 0xFFFFu) {
      if (old == TMP_B) {          // termination 1°: a vertex of B is reached
        atomicMax(&acc->bhit, ((unsigned long long)(unsigned)cand << 32) | (0xFFFFFFFFu - D));
        const unsigned k = atomicAdd(&s.ctl->n_barr, 1u);
        if (k < s.barr_cap) s.barr[k] = BArr{D, (unsigned)cand, src, via};
      }
    } else {
      first = os != v.stamp;
    }
  }
  qpush<unsigned>(sm.qt, &sm.nt, first, D, &acc->n_trig, s.trig, 0xFFFFFFFFull);
}

// ---------------------------------------------------------------------------
// sweep: Steps 1, 3, 7 and the retirement part of 8-9
// ---------------------------------------------------------------------------
template <int D>
__device__ void phase_sweep(const Dev& s, const View& v, Smem& sm) {
  using LW = typename Tr<D>::LW;
  Acc* acc = &s.ctl->acc[v.c % 3];
  LW* res = reinterpret_cast<LW*>(s.res);
  const unsigned* act_in = s.act[v.cur];
  unsigned* act_out = s.act[v.cur ^ 1];
  const unsigned long long* pool_in = s.pool[v.cur];
  unsigned long long* pool_out = s.pool[v.cur ^ 1];
  // adaptive chunk: enough chunks to give every block work when lists are short
  const unsigned total = v.n_act + v.n_pool;
  const unsigned items = total >= 4u * THREADS * gridDim.x ? 4u : (total >= 2u * THREADS * gridDim.x ? 2u : 1u);
  const unsigned chunk = items * THREADS;
  const unsigned na_ch = (v.n_act + chunk - 1) / chunk;
  const unsigned np_ch = (v.n_pool + chunk - 1) / chunk;
  const LW dl = (LW)v.delta;
  unsigned dmin = 0xFFFFFFFFu;
  unsigned long long live = 0, arr = 0;

  for (unsigned ch = blockIdx.x; ch < na_ch + np_ch; ch += gridDim.x) {
    if (ch < na_ch) {
      unsigned vx[SWEEP_ITEMS];
      LW w[SWEEP_ITEMS];
#pragma unroll
      for (int it = 0; it < SWEEP_ITEMS; ++it) {
        const unsigned i = ch * chunk + it * THREADS + threadIdx.x;
        vx[it] = ((unsigned)it < items && i < v.n_act) ? __ldcg(act_in + i) : 0xFFFFFFFFu;
      }
#pragma unroll
      for (int it = 0; it < SWEEP_ITEMS; ++it) w[it] = vx[it] != 0xFFFFFFFFu ? __ldcg(res + vx[it]) : (LW)0;
      LW fired[SWEEP_ITEMS];
#pragma unroll
      for (int it = 0; it < SWEEP_ITEMS; ++it) {
        const LW nz = nzb<LW>(w[it]);
        const LW w2 = w[it] - dl * (nz >> 7);          // every live byte >= Delta: no borrow
        fired[it] = nz & ~nzb<LW>(w2);                 // 0x80 in every lane that reached 0
        live += popc_lw<LW>(nz);
        if (w[it] != 0) __stcg(res + vx[it], w2);
        const bool survive = w2 != 0;
        if (survive) dmin = min(dmin, min_nonzero_byte<D, LW>(w2));
        qpush<unsigned>(sm.q32, &sm.na, survive, vx[it], &acc->n_act, act_out, 0xFFFFFFFFull);
      }
      unsigned lbl[SWEEP_ITEMS];
      LW f2w[SWEEP_ITEMS];
#pragma unroll
      for (int it = 0; it < SWEEP_ITEMS; ++it) {
        lbl[it] = 0; f2w[it] = 0;
        if (fired[it]) {
          lbl[it] = s.minf ? 1u : (__ldcg(lbl_ptr(s.sw, vx[it])) & 0xFFFFu);
          if (!s.minf) f2w[it] = load_f2<D>(s, vx[it]);
        }
      }
#pragma unroll
      for (int it = 0; it < SWEEP_ITEMS; ++it) {
#pragma unroll
        for (int j = 0; j < 2 * D; ++j) {
          const bool fj = (fired[it] >> (8 * j + 7)) & 1;
          arr += fj;
          const int cand = (int)lbl[it] - (int)((f2w[it] >> (8 * j)) & 0xFF);
          arrive(s, v, acc, sm, fj, vx[it] + s.off[j], cand, vx[it], 0u);
        }
      }
      qflush2<unsigned, unsigned>(sm.q32, &sm.na, &acc->n_act, act_out, 0xFFFFFFFFull, sm.qt, &sm.nt,
                                  &acc->n_trig, s.trig, 0xFFFFFFFFull, sm);
    } else {
      const unsigned pc = ch - na_ch;
      unsigned long long p[SWEEP_ITEMS];
#pragma unroll
      for (int it = 0; it < SWEEP_ITEMS; ++it) {
        const unsigned i = pc * chunk + it * THREADS + threadIdx.x;
        p[it] = ((unsigned)it < items && i < v.n_pool) ? __ldcs(pool_in + i) : 0ull;
      }
#pragma unroll
      for (int it = 0; it < SWEEP_ITEMS; ++it) {
        const unsigned r = (unsigned)(p[it] >> PH_RES) & 0xFFu;   // 0 only for padding
        const bool fire = r != 0 && r == v.delta;
        const bool keep = r > v.delta;
        if (keep) dmin = min(dmin, r - v.delta);
        arr += fire;
        qpush<unsigned long long>(sm.qp, &sm.np, keep, p[it] - ((unsigned long long)v.delta << PH_RES),
                                  &acc->n_pool, pool_out, s.pool_cap);
        const unsigned src = (unsigned)p[it] & 0x3FFFFFFFu;
        const unsigned lane = (unsigned)(p[it] >> PH_LANE) & 7u;
        const int cand = (int)((p[it] >> PH_CAND) & 0xFFFFu);
        arrive(s, v, acc, sm, fire, src + s.off[lane], cand, src, 1u);
      }
      qflush2<unsigned long long, unsigned>(sm.qp, &sm.np, &acc->n_pool, pool_out, s.pool_cap, sm.qt, &sm.nt,
                                            &acc->n_trig, s.trig, 0xFFFFFFFFull, sm);
    }
  }
  block_reduce_commit(sm, dmin, live, arr, 0, 0, 0, acc);
}

// ---------------------------------------------------------------------------
// treat: Steps 4, 5, 8.1 (+ the activation half of 8.2 / 9)
// ---------------------------------------------------------------------------
template <int D>
__device__ void phase_treat(const Dev& s, const View& v, Smem& sm, unsigned n_trig) {
  using LW = typename Tr<D>::LW;
  Acc* acc = &s.ctl->acc[v.c % 3];
  LW* res = reinterpret_cast<LW*>(s.res);
  unsigned* act_out = s.act[v.cur ^ 1];
  unsigned long long* pool_out = s.pool[v.cur ^ 1];
  const unsigned items = n_trig >= 2u * THREADS * gridDim.x ? 2u : 1u;
  const unsigned chunk = items * THREADS;
  const unsigned nch = (n_trig + chunk - 1) / chunk;
  unsigned dmin = 0xFFFFFFFFu;
  unsigned long long created = 0, relabels = 0, triggered = 0;

  for (unsigned ch = blockIdx.x; ch < nch; ch += gridDim.x) {
    unsigned q[TREAT_ITEMS];
#pragma unroll
    for (int it = 0; it < TREAT_ITEMS; ++it) {
      const unsigned i = ch * chunk + it * THREADS + threadIdx.x;
      q[it] = ((unsigned)it < items && i < n_trig) ? __ldcg(s.trig + i) : 0xFFFFFFFFu;
    }
    unsigned long long swq[TREAT_ITEMS];
    LW w[TREAT_ITEMS];
    WRec<LW> wr[TREAT_ITEMS];
#pragma unroll
    for (int it = 0; it < TREAT_ITEMS; ++it) {
      const bool valid = q[it] != 0xFFFFFFFFu;
      swq[it] = valid ? __ldcg(s.sw + q[it]) : 0ull;
      w[it] = valid ? __ldcg(res + q[it]) : (LW)0;
      wr[it] = valid ? load_wt<D>(s, q[it]) : WRec<LW>{0, 0};
    }
#pragma unroll
    for (int it = 0; it < TREAT_ITEMS; ++it) {
      const int lq = (int)(swq[it] & 0xFFFFu);
      const int lstar = (int)((swq[it] >> 32) & 0xFFFFu);         // L* = temp(Q) (reading R23)
      const bool trig = q[it] != 0xFFFFFFFFu && lstar > lq;       // the water improves Q
      const bool inactive = trig && w[it] == 0;                   // no live lane after the decrement (R6)
      triggered += trig;
      unsigned long long swr[2 * D];
#pragma unroll
      for (int j = 0; j < 2 * D; ++j) {
        const unsigned f1j = (unsigned)(wr[it].f1 >> (8 * j)) & 0xFFu;
        const unsigned f2j = s.minf ? 0u : (unsigned)(wr[it].f2 >> (8 * j)) & 0xFFu;
        const bool test = trig && f1j != 0 && lstar - (int)f2j > 0;
        swr[j] = test ? __ldcg(s.sw + (q[it] + s.off[j])) : 0xFFFFull;   // untested lanes read as "removed"
      }
      LW neww = 0;
#pragma unroll
      for (int j = 0; j < 2 * D; ++j) {
        const unsigned f1j = (unsigned)(wr[it].f1 >> (8 * j)) & 0xFFu;
        const unsigned f2j = s.minf ? 0u : (unsigned)(wr[it].f2 >> (8 * j)) & 0xFFu;
        const int c = lstar - (int)f2j;
        const unsigned rl = (unsigned)swr[j] & 0xFFFFu;
        const unsigned rtw = (unsigned)(swr[j] >> 32);
        const unsigned rt = (rtw >> 16) == v.stamp ? (rtw & 0xFFFFu) : 0u;
        const bool pass = c > (int)max(rl, rt);                   // edge triggered
        if (pass) dmin = min(dmin, f1j);
        if (pass && inactive) neww |= (LW)f1j << (8 * j);         // activate, time restored to f1 (:192)
        const bool ph = pass && !inactive;                        // phantom (Q, R, L*, f1) (:197-198)
        created += ph;
        const unsigned long long prec = (unsigned long long)q[it] | ((unsigned long long)j << PH_LANE) |
                                        ((unsigned long long)(unsigned)c << PH_CAND) |
                                        ((unsigned long long)f1j << PH_RES);
        qpush<unsigned long long>(sm.qp, &sm.np, ph, prec, &acc->n_pool, pool_out, s.pool_cap);
      }
      if (inactive) {                                             // Step 8.1
        *lbl_ptr(s.sw, q[it]) = (unsigned)lstar;
        relabels += 1;
        if (neww) __stcg(res + q[it], neww);
      }
      qpush<unsigned>(sm.q32, &sm.na, inactive && neww != 0, q[it], &acc->n_act, act_out, 0xFFFFFFFFull);
    }
    qflush2<unsigned, unsigned long long>(sm.q32, &sm.na, &acc->n_act, act_out, 0xFFFFFFFFull, sm.qp, &sm.np,
                                          &acc->n_pool, pool_out, s.pool_cap, sm);
  }
  block_reduce_commit(sm, dmin, 0, 0, created, relabels, triggered, acc);
}

// ---------------------------------------------------------------------------
// decide: Step 6 + time skipping.  Executed by one thread; writes ctl if writer.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void reset_acc(Acc* a) {
  a->n_act = 0; a->n_pool = 0; a->n_trig = 0; a->dmin = 0xFFFFFFFFu;
  a->bhit = 0; a->live = 0; a->arrivals = 0; a->created = 0; a->relabels = 0; a->triggered = 0;
  a->pend_lanes = 0; a->pend_phantoms = 0;
}

__device__ void decide(const Dev& s, View& v, bool writer) {
  Acc* a = &s.ctl->acc[v.c % 3];
  const unsigned long long bhit = __ldcg(&a->bhit);
  const unsigned n_act = __ldcg(&a->n_act), n_pool = __ldcg(&a->n_pool), dmin = __ldcg(&a->dmin);
  View nv = v;
  Ctl* C = s.ctl;
  if (writer) {
    const unsigned long long live = __ldcg(&a->live), arrivals = __ldcg(&a->arrivals);
    const unsigned long long created = __ldcg(&a->created), relabels = __ldcg(&a->relabels);
    const unsigned long long triggered = __ldcg(&a->triggered);
    if (v.c > 0) {
      C->cycles += 1;
      C->edge_updates += (long long)(live + v.n_pool);
      if ((long long)v.c - 1 < s.trace_cap) {
        TraceRec r{v.t, (long long)v.delta, (long long)v.n_act, (long long)live, (long long)v.n_pool,
                   (long long)triggered, (long long)arrivals, (long long)created, (long long)relabels};
        s.trace[v.c - 1] = r;
      }
    }
    C->arrivals += arrivals; C->triggered += triggered; C->created += created; C->relabels += relabels;
  }
  if (bhit) {
    nv.status = 0;  // WCSP_REACHED
    if (writer) {
      const unsigned q = (unsigned)(bhit >> 32);
      const unsigned X = 0xFFFFFFFFu - (unsigned)bhit;
      // Y = smallest source among the arrivals at X carrying q; a regular edge wins over a phantom
      const unsigned nb = min(__ldcg(&C->n_barr), s.barr_cap);
      unsigned long long best = ~0ull;
      for (unsigned k = 0; k < nb; ++k) {
        const BArr b = s.barr[k];
        if (b.D == X && b.cand == q) best = min(best, ((unsigned long long)b.src << 1) | b.via);
      }
      C->F1 = v.t;
      C->F2 = s.minf ? -1 : (long long)s.M - q;
      C->X = X;
      C->Y = (long long)(best >> 1);
      C->via = (long long)(best & 1);
    }
  } else if (n_pool > s.pool_cap) {
    nv.status = 8;  // WCSP_EOVERFLOW
    if (writer) C->need_pool = n_pool;
  } else if (dmin == 0xFFFFFFFFu) {
    nv.status = 1;  // WCSP_INFEASIBLE (2°)
  } else if (s.budget > 0 && (long long)v.c >= s.budget) {
    nv.status = 4;  // WCSP_EBUDGET
  } else {
    nv.delta = s.unit ? 1u : dmin;
    nv.t = v.t + nv.delta;
    nv.c = v.c + 1;
    nv.stamp = stamp_of(nv.c);
    nv.cur = v.cur ^ 1;
    nv.n_act = n_act;
    nv.n_pool = n_pool;
    if (writer) {
      if ((long long)n_act > C->peak_active) C->peak_active = n_act;
      if ((long long)n_pool > C->peak_phantoms) C->peak_phantoms = n_pool;
    }
  }
  if (writer) C->view = nv;
  v = nv;
}

// ---------------------------------------------------------------------------
// grid barrier for the cooperative persistent kernel (monotone counter)
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Returns false if the barrier was abandoned (watchdog: a block missing for
// BARRIER_TIMEOUT_NS sets ctl->abort; every waiting block then gives up).
constexpr unsigned long long BARRIER_TIMEOUT_NS = 20ull * 1000000000ull;

__device__ __forceinline__ bool grid_sync(Ctl* ctl, unsigned long long target, Smem& sm) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(&ctl->bar, 1ull);
    const unsigned long long t0 = globaltimer_ns();
    unsigned ok = 1;
    while (ld_acquire(&ctl->bar) < target) {
      __nanosleep(32);
      if (*(volatile unsigned*)&ctl->abort) { ok = 0; break; }
      if (globaltimer_ns() - t0 > BARRIER_TIMEOUT_NS) { atomicExch(&ctl->abort, 1u); ok = 0; break; }
    }
    __threadfence();
    sm.flag = ok;
  }
  __syncthreads();
  const bool ok = sm.flag != 0;
  __syncthreads();
  return ok;
}

__device__ __forceinline__ void load_view(const Dev& s, Smem& sm, View& v) {
  if (threadIdx.x == 0) {
    volatile View* g = &s.ctl->view;
    View x;
    x.t = g->t; x.c = g->c; x.stamp = g->stamp; x.delta = g->delta; x.n_act = g->n_act;
    x.n_pool = g->n_pool; x.cur = g->cur; x.status = g->status; x.region = g->region; x.pad_ = 0;
    sm.view = x;
  }
  __syncthreads();
  v = sm.view;
}

__device__ __forceinline__ void init_smem(Smem& sm) {
  if (threadIdx.x == 0) { sm.na = 0; sm.nt = 0; sm.np = 0; }
  __syncthreads();
}

// Forget every temp (keeps the target / removed sentinels): used when the
// 16-bit cycle stamps wrap.
__device__ __forceinline__ void clear_temps(const Dev& s) {
  for (unsigned long long i = (unsigned long long)blockIdx.x * THREADS + threadIdx.x; i < s.N;
       i += (unsigned long long)gridDim.x * THREADS) {
    unsigned* t = tmp_ptr(s.sw, (unsigned)i);
    if ((*t >> 16) != 0xFFFFu) *t = 0u;
  }
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(THREADS, 4) k_persistent(Dev s) {
  __shared__ Smem sm;
  init_smem(sm);
  View v;
  load_view(s, sm, v);
  const unsigned long long G = gridDim.x;
  unsigned long long target = 0;
  while (v.status == ST_RUNNING) {
    if (v.c > 0) {
      if (blockIdx.x == 0 && threadIdx.x == 0) reset_acc(&s.ctl->acc[(v.c + 1) % 3]);
      phase_sweep<D>(s, v, sm);
      target += G;
      if (!grid_sync(s.ctl, target, sm)) return;
    }
    if (threadIdx.x == 0) {
      sm.bhit = __ldcg(&s.ctl->acc[v.c % 3].bhit);
      sm.base_a = __ldcg(&s.ctl->acc[v.c % 3].n_trig);
    }
    __syncthreads();
    const unsigned long long bhit = sm.bhit;
    const unsigned n_trig = sm.base_a;
    __syncthreads();
    if (!bhit) {                                   // S5 precedes S6: the final cycle skips the treat
      phase_treat<D>(s, v, sm, n_trig);
      target += G;
      if (!grid_sync(s.ctl, target, sm)) return;
    }
    if (threadIdx.x == 0) {
      View nv = v;
      decide(s, nv, blockIdx.x == 0);
      sm.view = nv;
    }
    __syncthreads();
    v = sm.view;
    __syncthreads();
    if (v.status == ST_RUNNING && v.stamp == 1u) { // stamps wrapped: forget every temp (rare)
      clear_temps(s);
      target += G;
      if (!grid_sync(s.ctl, target, sm)) return;
    }
  }
}

template <int D>
__global__ void __launch_bounds__(THREADS) k_sweep(Dev s) {
  __shared__ Smem sm;
  init_smem(sm);
  View v;
  load_view(s, sm, v);
  if (v.status != ST_RUNNING || v.c == 0) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) reset_acc(&s.ctl->acc[(v.c + 1) % 3]);
  phase_sweep<D>(s, v, sm);
}

template <int D>
__global__ void __launch_bounds__(THREADS, 4) k_treat(Dev s) {
  __shared__ Smem sm;
  init_smem(sm);
  View v;
  load_view(s, sm, v);
  if (v.status != ST_RUNNING) return;
  const Acc* a = &s.ctl->acc[v.c % 3];
  if (__ldcg(&a->bhit)) return;
  phase_treat<D>(s, v, sm, __ldcg(&a->n_trig));
}

__global__ void k_decide(Dev s) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  View v = s.ctl->view;
  if (v.status != ST_RUNNING) return;
  decide(s, v, true);
  if (v.status == ST_RUNNING && v.stamp == 1u) s.ctl->view.status = ST_WRAP;
}

__global__ void __launch_bounds__(THREADS) k_clear_temps(Dev s) { clear_temps(s); }

// Initial state (reading R20): L = M on A, 0 elsewhere,
// target / removed sentinels, no live lane, A triggered with temp M.
__global__ void __launch_bounds__(THREADS) k_init(Dev s, const uint8_t* maskA, const uint8_t* maskB,
                                                  const uint8_t* present, int lblA, int d) {
  Acc* acc = &s.ctl->acc[0];
  const unsigned N = s.N;
  for (unsigned long long base = (unsigned long long)blockIdx.x * THREADS; base < N;
       base += (unsigned long long)gridDim.x * THREADS) {
    const unsigned long long i = base + threadIdx.x;
    const bool valid = i < N;
    bool a = false;
    if (valid) {
      const bool p = present ? present[i] != 0 : true;
      a = p && maskA[i];
      const bool b = p && maskB[i];
      unsigned lbl = 0, tmp = 0;
      if (!p) { lbl = LBL_REMOVED; tmp = TMP_REMOVED; }
      else if (b) { lbl = 0; tmp = TMP_B; }
      else if (a) { lbl = 0; tmp = (stamp_of(0) << 16) | (unsigned)lblA; }   // treat(c = 0) sets L = M
      s.sw[i] = ((unsigned long long)tmp << 32) | lbl;
      if (d <= 2) reinterpret_cast<uint32_t*>(s.res)[i] = 0u;
      else reinterpret_cast<unsigned long long*>(s.res)[i] = 0ull;
    }
    // direct global append (order irrelevant); warp-aggregated
    const unsigned m = __ballot_sync(0xFFFFFFFFu, a);
    if (m) {
      const unsigned lane = threadIdx.x & 31u;
      const int leader = __ffs(m) - 1;
      unsigned b = 0;
      if ((int)lane == leader) b = atomicAdd(&acc->n_trig, (unsigned)__popc(m));
      b = __shfl_sync(0xFFFFFFFFu, b, leader);
      if (a) s.trig[b + __popc(m & ((1u << lane) - 1u))] = (unsigned)i;
    }
  }
}

// Weight records: lane 2k of v = edge (v, v+e_k); lane 2k+1 = edge (v-e_k, v).
template <int D>
__global__ void __launch_bounds__(THREADS) k_weights(Dev s, const uint8_t* f1, const uint8_t* f2,
                                                     long long n0, long long n1, long long n2, long long n3) {
  using LW = typename Tr<D>::LW;
  const long long n[4] = {n0, n1, n2, n3};
  const unsigned long long N = s.N;
  for (unsigned long long v = (unsigned long long)blockIdx.x * THREADS + threadIdx.x; v < N;
       v += (unsigned long long)gridDim.x * THREADS) {
    LW a = 0, b = 0;
    unsigned long long stride = 1;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const unsigned long long xk = (v / stride) % (unsigned long long)n[k];
      if (xk + 1 < (unsigned long long)n[k]) {
        a |= (LW)f1[k * N + v] << (8 * (2 * k));
        b |= (LW)f2[k * N + v] << (8 * (2 * k));
      }
      if (xk > 0) {
        a |= (LW)f1[k * N + v - stride] << (8 * (2 * k + 1));
        b |= (LW)f2[k * N + v - stride] << (8 * (2 * k + 1));
      }
      stride *= (unsigned long long)n[k];
    }
    // an absent edge (f1 = 0) carries no weight
#pragma unroll
    for (int j = 0; j < 2 * D; ++j)
      if (((a >> (8 * j)) & 0xFF) == 0) b &= ~((LW)0xFF << (8 * j));
    if constexpr (sizeof(LW) == 4) {
      reinterpret_cast<uint2*>(const_cast<void*>(s.wt))[v] = make_uint2(a, b);
    } else {
      reinterpret_cast<uint4*>(const_cast<void*>(s.wt))[v] =
          make_uint4((unsigned)a, (unsigned)(a >> 32), (unsigned)b, (unsigned)(b >> 32));
    }
  }
}

// Validation counters (wcsp.h rules): [0] |A|, [1] |B|, [2] |A n B|, [3] present edges with f2 = 0.
__global__ void __launch_bounds__(THREADS) k_validate(unsigned long long N, int d, long long n0, long long n1,
                                                      long long n2, long long n3, const uint8_t* f1,
                                                      const uint8_t* f2, const uint8_t* maskA,
                                                      const uint8_t* maskB, const uint8_t* present,
                                                      unsigned long long* out) {
  const long long n[4] = {n0, n1, n2, n3};
  unsigned long long c[4] = {0, 0, 0, 0};
  for (unsigned long long v = (unsigned long long)blockIdx.x * THREADS + threadIdx.x; v < N;
       v += (unsigned long long)gridDim.x * THREADS) {
    const bool p = present ? present[v] != 0 : true;
    const bool a = p && maskA[v], b = p && maskB[v];
    c[0] += a; c[1] += b; c[2] += a && b;
    unsigned long long stride = 1;
    for (int k = 0; k < d; ++k) {
      const unsigned long long xk = (v / stride) % (unsigned long long)n[k];
      if (xk + 1 < (unsigned long long)n[k]) c[3] += (f1[k * N + v] != 0 && f2[k * N + v] == 0);
      stride *= (unsigned long long)n[k];
    }
  }
  for (int i = 0; i < 4; ++i)
    if (c[i]) atomicAdd(out + i, c[i]);
}

}  // namespace wcspk
