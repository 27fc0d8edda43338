// wcsp_wheel.cuh — the timing-wheel engine: the same cycle
// (§4) with the residual-time bookkeeping of Steps 1, 3 and 7
// stored as absolute arrival times instead of countdowns.
//
// A live edge — an active edge or a phantom — is an *event*
// (src, lane, cand = L(src) - f2) filed in bucket (t_start + f1) mod 256 of a
// wheel.  "Decrease every time parameter by Delta" and "an edge whose time
// reaches 0 is just used" become "advance t to the next non-empty
// bucket and fire its events": each event is written once and read once
// instead of being rewritten every cycle.  The active-vertex sequence
// is implicit: vertex v is active at t iff its latest lane arrival time
// texp(v) > t (texp is kept modulo 2^16 in the spare half of the label word;
// a maintenance pass refreshes it every 2^15 time units).  Every other step
// (arrival resolution, termination, treat, relabel) is the sweep engine's, so
// outputs AND work counters (E = lane events in flight, P = phantom events in
// flight) are identical to it — tested.
//
// Event record (u64): src 30 | lane 3 | cand 16 | is_lane 1 (bit 49); bits
// 56..63 hold the delay f1 while the record sits in a block's staging queue.
#pragma once
#include "wcsp_device.cuh"

namespace wcspk {

constexpr int EV_LANE_BIT = 49;
constexpr int EV_DELAY_SHIFT = 56;
constexpr int WHEEL = 256;                 // f1 <= 255: every event lands within 255 time units
constexpr unsigned MAINT_PERIOD_T = 1u << 15;

__device__ __forceinline__ bool lane_live(unsigned texp16, long long t) {
  return ((texp16 - (unsigned)t) & 0xFFFFu) - 1u < 255u;   // texp in (t, t + 255]
}

struct WheelSmem {
  unsigned hist[WHEEL];
  unsigned hlane[WHEEL];
  unsigned long long hbase[WHEEL];
  unsigned short rank[QCAP];
};

// File a run of `cnt` events (already at ring positions pos..pos+cnt-1) into bucket b.
__device__ __forceinline__ void file_run(const Dev& s, unsigned b, unsigned long long pos, unsigned cnt,
                                         unsigned lanes) {
  const unsigned k = atomicAdd(s.bndesc + b, 1u);
  if (k < s.dcap) s.bdesc[(size_t)b * s.dcap + k] = (pos << 24) | cnt;
  else atomicOr(&s.ctl->wheel_overflow, 2u);
  atomicAdd(s.bnev + b, cnt);
  if (lanes) atomicAdd(s.bnlane + b, lanes);
}

// Stage one event per predicated lane (warp-aggregated); a full staging queue
// files the event as its own run (rare).
__device__ __forceinline__ void ev_push(const Dev& s, Smem& sm, bool pred, unsigned long long rec, unsigned delay,
                                       long long t) {
  const unsigned m = __ballot_sync(0xFFFFFFFFu, pred);
  if (m == 0) return;
  const unsigned lane = threadIdx.x & 31u;
  const int leader = __ffs(m) - 1;
  unsigned base = 0;
  if ((int)lane == leader) base = atomicAdd(&sm.np, (unsigned)__popc(m));
  base = __shfl_sync(0xFFFFFFFFu, base, leader);
  if (pred) {
    const unsigned idx = base + __popc(m & ((1u << lane) - 1u));
    if (idx < (unsigned)QCAP) {
      sm.qp[idx] = rec | ((unsigned long long)delay << EV_DELAY_SHIFT);
    } else {
      const unsigned long long pos = atomicAdd(&s.ctl->ev_head, 1ull);
      s.ev[pos & s.ev_mask] = rec;
      file_run(s, (unsigned)((t + delay) & (WHEEL - 1)), pos, 1u, (unsigned)((rec >> EV_LANE_BIT) & 1));
    }
  }
}

// Counting-sort the block's staged events by delay and file one run per delay
// (one ring allocation + one descriptor per non-empty delay).
__device__ void ev_flush(const Dev& s, Smem& sm, WheelSmem& ws, long long t) {
  __syncthreads();
  const unsigned n = min(sm.np, (unsigned)QCAP);
  for (unsigned d = threadIdx.x; d < WHEEL; d += THREADS) { ws.hist[d] = 0; ws.hlane[d] = 0; }
  __syncthreads();
  for (unsigned i = threadIdx.x; i < n; i += THREADS) {
    const unsigned long long e = sm.qp[i];
    const unsigned d = (unsigned)(e >> EV_DELAY_SHIFT);
    ws.rank[i] = (unsigned short)atomicAdd(&ws.hist[d], 1u);
    if ((e >> EV_LANE_BIT) & 1) atomicAdd(&ws.hlane[d], 1u);
  }
  __syncthreads();
  for (unsigned d = threadIdx.x; d < WHEEL; d += THREADS) {
    const unsigned cnt = ws.hist[d];
    if (cnt) {
      const unsigned long long pos = atomicAdd(&s.ctl->ev_head, (unsigned long long)cnt);
      ws.hbase[d] = pos;
      file_run(s, (unsigned)((t + d) & (WHEEL - 1)), pos, cnt, ws.hlane[d]);
    }
  }
  __syncthreads();
  for (unsigned i = threadIdx.x; i < n; i += THREADS) {
    const unsigned long long e = sm.qp[i];
    const unsigned d = (unsigned)(e >> EV_DELAY_SHIFT);
    s.ev[(ws.hbase[d] + ws.rank[i]) & s.ev_mask] = e & ((1ull << EV_DELAY_SHIFT) - 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) sm.np = 0;
  __syncthreads();
}

// fire: the events of bucket t reach their destinations (Steps 1-3).
template <int D>
__device__ void wheel_fire(const Dev& s, const View& v, Smem& sm) {
  Acc* acc = &s.ctl->acc[v.c % 3];
  const unsigned b = (unsigned)(v.t & (WHEEL - 1));
  const unsigned nd = min(__ldcg(s.bndesc + b), s.dcap);
  unsigned long long arr = 0;
  for (unsigned di = blockIdx.x; di < nd; di += gridDim.x) {
    const unsigned long long dsc = __ldcg(s.bdesc + (size_t)b * s.dcap + di);
    const unsigned long long pos = dsc >> 24;
    const unsigned cnt = (unsigned)(dsc & 0xFFFFFFu);
    for (unsigned base = 0; base < cnt; base += SWEEP_ITEMS * THREADS) {
      unsigned long long e[SWEEP_ITEMS];
#pragma unroll
      for (int it = 0; it < SWEEP_ITEMS; ++it) {
        const unsigned i = base + it * THREADS + threadIdx.x;
        e[it] = i < cnt ? __ldcs(s.ev + ((pos + i) & s.ev_mask)) : ~0ull;
      }
#pragma unroll
      for (int it = 0; it < SWEEP_ITEMS; ++it) {
        const bool valid = e[it] != ~0ull;
        arr += valid;
        const unsigned src = (unsigned)e[it] & 0x3FFFFFFFu;
        const unsigned lane = (unsigned)(e[it] >> PH_LANE) & 7u;
        const int cand = (int)((e[it] >> PH_CAND) & 0xFFFFu);
        const unsigned via = ((e[it] >> EV_LANE_BIT) & 1) ? 0u : 1u;
        arrive(s, v, acc, sm, valid, src + s.off[lane], cand, src, via);
      }
      __syncthreads();
      if (sm.nt > (unsigned)(QCAP - SWEEP_ITEMS * THREADS))
        qflush2<unsigned, unsigned>(sm.qt, &sm.nt, &acc->n_trig, s.trig, 0xFFFFFFFFull, sm.q32, &sm.na,
                                    &acc->n_act, s.act[0], 0ull, sm);
    }
  }
  qflush2<unsigned, unsigned>(sm.qt, &sm.nt, &acc->n_trig, s.trig, 0xFFFFFFFFull, sm.q32, &sm.na, &acc->n_act,
                              s.act[0], 0ull, sm);
  block_reduce_commit(sm, 0xFFFFFFFFu, 0, arr, 0, 0, 0, acc);
}

// treat: Steps 4, 5, 8.1 — identical decisions to phase_treat; new lanes and
// phantoms become events filed at t + f1.
template <int D>
__device__ void wheel_treat(const Dev& s, const View& v, Smem& sm, WheelSmem& ws, unsigned n_trig) {
  using LW = typename Tr<D>::LW;
  Acc* acc = &s.ctl->acc[v.c % 3];
  const unsigned items = n_trig >= 2u * THREADS * gridDim.x ? 2u : 1u;
  const unsigned chunk = items * THREADS;
  const unsigned nch = (n_trig + chunk - 1) / chunk;
  unsigned long long created = 0, relabels = 0, triggered = 0, lanes_started = 0;

  for (unsigned ch = blockIdx.x; ch < nch; ch += gridDim.x) {
    unsigned q[TREAT_ITEMS];
#pragma unroll
    for (int it = 0; it < TREAT_ITEMS; ++it) {
      const unsigned i = ch * chunk + it * THREADS + threadIdx.x;
      q[it] = ((unsigned)it < items && i < n_trig) ? __ldcg(s.trig + i) : 0xFFFFFFFFu;
    }
    unsigned long long swq[TREAT_ITEMS];
    WRec<LW> wr[TREAT_ITEMS];
#pragma unroll
    for (int it = 0; it < TREAT_ITEMS; ++it) {
      const bool valid = q[it] != 0xFFFFFFFFu;
      swq[it] = valid ? __ldcg(s.sw + q[it]) : 0ull;
      wr[it] = valid ? load_wt<D>(s, q[it]) : WRec<LW>{0, 0};
    }
#pragma unroll
    for (int it = 0; it < TREAT_ITEMS; ++it) {
      const int lq = (int)(swq[it] & 0xFFFFu);
      const unsigned texp = (unsigned)(swq[it] >> 16) & 0xFFFFu;
      const int lstar = (int)((swq[it] >> 32) & 0xFFFFu);         // L* = temp(Q) (reading R23)
      const bool trig = q[it] != 0xFFFFFFFFu && lstar > lq;       // the water improves Q
      const bool inactive = trig && !lane_live(texp, v.t);        // no live lane after this cycle's arrivals (R6)
      triggered += trig;
      unsigned long long swr[2 * D];
#pragma unroll
      for (int j = 0; j < 2 * D; ++j) {
        const unsigned f1j = (unsigned)(wr[it].f1 >> (8 * j)) & 0xFFu;
        const unsigned f2j = s.minf ? 0u : (unsigned)(wr[it].f2 >> (8 * j)) & 0xFFu;
        const bool test = trig && f1j != 0 && lstar - (int)f2j > 0;
        swr[j] = test ? __ldcg(s.sw + (q[it] + s.off[j])) : 0xFFFFull;
      }
      unsigned fmax = 0;
#pragma unroll
      for (int j = 0; j < 2 * D; ++j) {
        const unsigned f1j = (unsigned)(wr[it].f1 >> (8 * j)) & 0xFFu;
        const unsigned f2j = s.minf ? 0u : (unsigned)(wr[it].f2 >> (8 * j)) & 0xFFu;
        const int c = lstar - (int)f2j;
        const unsigned rl = (unsigned)swr[j] & 0xFFFFu;
        const unsigned rtw = (unsigned)(swr[j] >> 32);
        const unsigned rt = (rtw >> 16) == v.stamp ? (rtw & 0xFFFFu) : 0u;
        const bool pass = c > (int)max(rl, rt);                   // edge triggered
        if (pass && inactive) fmax = max(fmax, f1j);              // activate, time restored to f1 (:192)
        created += pass && !inactive;                             // phantom (Q, R, L*, f1) (:197-198)
        lanes_started += pass && inactive;
        const unsigned long long rec = (unsigned long long)q[it] | ((unsigned long long)j << PH_LANE) |
                                       ((unsigned long long)(unsigned)c << PH_CAND) |
                                       ((unsigned long long)(inactive ? 1u : 0u) << EV_LANE_BIT);
        ev_push(s, sm, pass, rec, f1j, v.t);
      }
      if (inactive) {                                             // Step 8.1
        const unsigned nt = (unsigned)((fmax ? v.t + fmax : v.t) & 0xFFFF);
        *lbl_ptr(s.sw, q[it]) = (unsigned)lstar | (nt << 16);
        relabels += 1;
      }
    }
    __syncthreads();
    if (sm.np > (unsigned)(QCAP - TREAT_ITEMS * THREADS * 2 * D)) ev_flush(s, sm, ws, v.t);
  }
  ev_flush(s, sm, ws, v.t);
  // created counts phantoms; lanes started ride in the 'live' slot of the accumulator
  block_reduce_commit(sm, 0xFFFFFFFFu, lanes_started, 0, created, relabels, triggered, acc);
}

// decide for the wheel: pending-event bookkeeping, next non-empty bucket, ring check.
__device__ void wheel_decide(const Dev& s, View& v, bool writer) {
  Acc* a = &s.ctl->acc[v.c % 3];
  Ctl* C = s.ctl;
  const unsigned long long bhit = __ldcg(&a->bhit);
  View nv = v;
  const unsigned b = (unsigned)(v.t & (WHEEL - 1));
  // pending counts at the top of this cycle (before its fire) are what the
  // sweep engine calls E and P; the writer advances them
  long long pl = __ldcg((const unsigned long long*)&C->pend_lanes);
  long long pp = __ldcg((const unsigned long long*)&C->pend_phantoms);
  const long long fired = v.c > 0 ? (long long)__ldcg(s.bnev + b) : 0;
  const long long fired_l = v.c > 0 ? (long long)__ldcg(s.bnlane + b) : 0;
  const long long new_l = (long long)__ldcg(&a->live);        // lanes started this cycle
  const long long new_p = (long long)__ldcg(&a->created);     // phantoms created this cycle
  if (writer) {
    const unsigned long long arrivals = __ldcg(&a->arrivals);
    const unsigned long long relabels = __ldcg(&a->relabels), triggered = __ldcg(&a->triggered);
    if (v.c > 0) {
      C->cycles += 1;
      C->edge_updates += pl + pp;
      if ((long long)v.c - 1 < s.trace_cap) {
        TraceRec r{v.t, (long long)v.delta, -1, pl, pp, (long long)triggered, (long long)arrivals,
                   new_p, (long long)relabels};
        s.trace[v.c - 1] = r;
      }
    }
    C->arrivals += arrivals; C->triggered += triggered; C->created += new_p; C->relabels += relabels;
  }
  pl += new_l - fired_l;
  pp += new_p - (fired - fired_l);
  if (bhit) {
    nv.status = 0;
    if (writer) {
      const unsigned q = (unsigned)(bhit >> 32);
      const unsigned X = 0xFFFFFFFFu - (unsigned)bhit;
      const unsigned nb = min(__ldcg(&C->n_barr), s.barr_cap);
      unsigned long long best = ~0ull;
      for (unsigned k = 0; k < nb; ++k) {
        const BArr e = s.barr[k];
        if (e.D == X && e.cand == q) best = min(best, ((unsigned long long)e.src << 1) | e.via);
      }
      C->F1 = v.t;
      C->F2 = s.minf ? -1 : (long long)s.M - q;
      C->X = X;
      C->Y = (long long)(best >> 1);
      C->via = (long long)(best & 1);
    }
  } else if (__ldcg(&C->wheel_overflow)) {
    nv.status = 8;  // WCSP_EOVERFLOW
  } else if (pl + pp == 0) {
    nv.status = 1;  // 2°: no live edge
  } else if (s.budget > 0 && (long long)v.c >= s.budget) {
    nv.status = 4;
  } else {
    unsigned k = 1;
    if (!s.unit)
      while (k < (unsigned)WHEEL && __ldcg(s.bnev + ((b + k) & (WHEEL - 1))) == 0) ++k;
    nv.delta = k;
    nv.t = v.t + k;
    nv.c = v.c + 1;
    nv.stamp = stamp_of(nv.c);
    nv.n_act = 0;
    nv.n_pool = 0;
    // ring check: every event allocated by a cycle whose time is >= t_next - f1max may be live
    const unsigned long long head = __ldcg(&C->ev_head);
    unsigned long long oldest = head;
    for (unsigned back = 0; back < (unsigned)WHEEL && back <= v.c; ++back) {
      const unsigned slot = (v.c - back) & (WHEEL - 1);
      if (__ldcg((const unsigned long long*)&C->hist_t[slot]) + s.f1max < (unsigned long long)nv.t) break;
      oldest = __ldcg(&C->hist_head[slot]);
    }
    if (head - oldest > s.ev_mask + 1) {
      nv.status = 8;
      if (writer) C->need_pool = (long long)(head - oldest);
    }
    if (writer) {
      if (pl + pp > C->peak_phantoms) C->peak_phantoms = pl + pp;
      C->hist_t[nv.c & (WHEEL - 1)] = nv.t;
      C->hist_head[nv.c & (WHEEL - 1)] = head;
    }
  }
  if (writer) {
    C->pend_lanes = pl;
    C->pend_phantoms = pp;
    if (v.c > 0) { s.bndesc[b] = 0; s.bnev[b] = 0; s.bnlane[b] = 0; }   // bucket t is consumed
    C->view = nv;
  }
  v = nv;
}

// Maintenance (rare): forget stale temps and refresh lane-expiry times so the
// 16-bit stamp and texp comparisons stay unambiguous.
__device__ __forceinline__ void wheel_maintain(const Dev& s, long long t) {
  for (unsigned long long i = (unsigned long long)blockIdx.x * THREADS + threadIdx.x; i < s.N;
       i += (unsigned long long)gridDim.x * THREADS) {
    unsigned* tp = tmp_ptr(s.sw, (unsigned)i);
    if ((*tp >> 16) != 0xFFFFu) *tp = 0u;
    unsigned* lp = lbl_ptr(s.sw, (unsigned)i);
    const unsigned lw = *lp;
    if ((lw & 0xFFFFu) != LBL_REMOVED && !lane_live(lw >> 16, t)) *lp = (lw & 0xFFFFu) | ((unsigned)(t & 0xFFFF) << 16);
  }
}

__device__ __forceinline__ bool needs_maint(const View& prev, const View& nv) {
  return nv.status == ST_RUNNING &&
         (nv.stamp == 1u || (nv.t / MAINT_PERIOD_T) != (prev.t / MAINT_PERIOD_T));
}

struct WheelAllSmem { Smem sm; WheelSmem ws; };

template <int D>
__global__ void __launch_bounds__(THREADS, 4) k_wheel_persistent(Dev s) {
  __shared__ WheelAllSmem all;
  Smem& sm = all.sm;
  init_smem(sm);
  View v;
  load_view(s, sm, v);
  const unsigned long long G = gridDim.x;
  unsigned long long target = 0;
  while (v.status == ST_RUNNING) {
    if (v.c > 0) {
      if (blockIdx.x == 0 && threadIdx.x == 0) reset_acc(&s.ctl->acc[(v.c + 1) % 3]);
      wheel_fire<D>(s, v, sm);
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
    if (!bhit) {
      wheel_treat<D>(s, v, sm, all.ws, n_trig);
      target += G;
      if (!grid_sync(s.ctl, target, sm)) return;
    }
    const View prev = v;
    if (threadIdx.x == 0) {
      View nv = v;
      wheel_decide(s, nv, blockIdx.x == 0);
      sm.view = nv;
    }
    __syncthreads();
    v = sm.view;
    __syncthreads();
    if (needs_maint(prev, v)) {
      wheel_maintain(s, v.t);
      target += G;
      if (!grid_sync(s.ctl, target, sm)) return;
    }
  }
}

template <int D>
__global__ void __launch_bounds__(THREADS) k_wheel_fire(Dev s) {
  __shared__ Smem sm;
  init_smem(sm);
  View v;
  load_view(s, sm, v);
  if (v.status != ST_RUNNING || v.c == 0) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) reset_acc(&s.ctl->acc[(v.c + 1) % 3]);
  wheel_fire<D>(s, v, sm);
}

template <int D>
__global__ void __launch_bounds__(THREADS, 4) k_wheel_treat(Dev s) {
  __shared__ WheelAllSmem all;
  init_smem(all.sm);
  View v;
  load_view(s, all.sm, v);
  if (v.status != ST_RUNNING) return;
  const Acc* a = &s.ctl->acc[v.c % 3];
  if (__ldcg(&a->bhit)) return;
  wheel_treat<D>(s, v, all.sm, all.ws, __ldcg(&a->n_trig));
}

__global__ void k_wheel_decide(Dev s) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  View v = s.ctl->view;
  if (v.status != ST_RUNNING) return;
  const View prev = v;
  wheel_decide(s, v, true);
  if (needs_maint(prev, v)) s.ctl->view.status = ST_WRAP;
}

__global__ void __launch_bounds__(THREADS) k_wheel_maintain(Dev s, long long t) { wheel_maintain(s, t); }

}  // namespace wcspk
