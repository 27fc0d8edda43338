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
// texp(v) > t (texp kept modulo 2^16 in bits 16-31 of the label word; a
// maintenance pass refreshes it every 2^15 time units).  Every other step
// (arrival resolution, termination, treat, relabel) is the sweep engine's, so
// outputs AND work counters (E = lane events in flight, P = phantom events in
// flight) equal the sweep engine's — tested.
//
// Storage: an event ring (power-of-two capacity, logical head ev_head).  In a
// treat phase every block keeps one open region of the ring per delay f1 and
// files a region as one run descriptor (pos << 24 | count) into bucket
// (t + f1) & 255 when it fills or at the end of the phase; a bucket is fired
// warp-per-run.  Event record (u64): src 30 | lane 3 | cand 16 | is_lane 1
// (bit 49); bits 56..63 carry the delay while the record sits in shared memory.
#pragma once
#include "wcsp_device.cuh"

namespace wcspk {

constexpr int EV_LANE_BIT = 49;
constexpr int EV_DELAY_SHIFT = 56;
constexpr unsigned MAINT_PERIOD_T = 1u << 15;

__device__ __forceinline__ void file_run(const Dev& s, unsigned b, unsigned long long pos, unsigned cnt) {
  const unsigned k = atomicAdd(s.bndesc + b, 1u);
  if (k < s.dcap) s.bdesc[(size_t)b * s.dcap + k] = (pos << 24) | cnt;
  else atomicOr(&s.ctl->wheel_overflow, 2u);
}

__device__ void ev_push(const Dev& s, Smem& sm, bool pred, unsigned long long rec, unsigned delay, long long t) {
  const unsigned m = __ballot_sync(0xFFFFFFFFu, pred);
  if (m == 0) return;
  const unsigned lane = threadIdx.x & 31u;
  const int leader = __ffs(m) - 1;
  unsigned base = 0;
  if ((int)lane == leader) base = atomicAdd(&sm.np, (unsigned)__popc(m));
  base = __shfl_sync(0xFFFFFFFFu, base, leader);
  if (pred) {
    const unsigned idx = base + __popc(m & ((1u << lane) - 1u));
    if (idx < (unsigned)QP_CAP) {
      sm.qp[idx] = rec | ((unsigned long long)delay << EV_DELAY_SHIFT);
    } else {                        // rare: staging full, file the event as a run of one
      const unsigned long long pos = atomicAdd(&s.ctl->ev_head, 1ull);
      s.ev[pos & s.ev_mask] = rec;
      const unsigned b = (unsigned)((t + delay) & (WHEEL - 1));
      atomicAdd(s.bnev + b, 1u);
      if ((rec >> EV_LANE_BIT) & 1) atomicAdd(s.bnlane + b, 1u);
      file_run(s, b, pos, 1u);
    }
  }
}

// Counting-sort the staged events by delay and append each delay's events to
// the block's open region for that delay (opening a new region of `region`
// slots when it is full); final_flush files every open region.
__device__ void ev_flush(const Dev& s, Smem& sm, long long t, unsigned region, bool final_flush) {
  __syncthreads();
  const unsigned n = min(sm.np, (unsigned)QP_CAP);
  if (n > 0) {
    for (unsigned d = threadIdx.x; d < WHEEL; d += THREADS) { sm.hist[d] = 0; sm.hlane[d] = 0; }
    __syncthreads();
    for (unsigned i = threadIdx.x; i < n; i += THREADS) {
      const unsigned long long e = sm.qp[i];
      const unsigned d = (unsigned)(e >> EV_DELAY_SHIFT);
      sm.rank[i] = (unsigned short)atomicAdd(&sm.hist[d], 1u);
      if ((e >> EV_LANE_BIT) & 1) atomicAdd(&sm.hlane[d], 1u);
    }
    __syncthreads();
    for (unsigned d = threadIdx.x; d < WHEEL; d += THREADS) {
      const unsigned cnt = sm.hist[d];
      if (cnt) {
        const unsigned b = (unsigned)((t + d) & (WHEEL - 1));
        if (sm.rfill[d] + cnt > sm.rcap[d]) {
          if (sm.rfill[d]) file_run(s, b, sm.rpos[d], sm.rfill[d]);
          const unsigned size = max(region, cnt);
          sm.rpos[d] = atomicAdd(&s.ctl->ev_head, (unsigned long long)size);
          sm.rfill[d] = 0;
          sm.rcap[d] = size;
        }
        sm.hbase[d] = sm.rpos[d] + sm.rfill[d];
        sm.rfill[d] += cnt;
        atomicAdd(s.bnev + b, cnt);
        if (sm.hlane[d]) atomicAdd(s.bnlane + b, sm.hlane[d]);
      }
    }
    __syncthreads();
    for (unsigned i = threadIdx.x; i < n; i += THREADS) {
      const unsigned long long e = sm.qp[i];
      const unsigned d = (unsigned)(e >> EV_DELAY_SHIFT);
      s.ev[(sm.hbase[d] + sm.rank[i]) & s.ev_mask] = e & ((1ull << EV_DELAY_SHIFT) - 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) sm.np = 0;
  }
  if (final_flush) {
    for (unsigned d = threadIdx.x; d < WHEEL; d += THREADS) {
      if (sm.rfill[d]) file_run(s, (unsigned)((t + d) & (WHEEL - 1)), sm.rpos[d], sm.rfill[d]);
      sm.rfill[d] = 0;
      sm.rcap[d] = 0;
    }
  }
  __syncthreads();
}

// Start-of-cycle bookkeeping (block 0, thread 0, before the fire phase).
__device__ __forceinline__ void wheel_cycle_start(const Dev& s, const View& v) {
  reset_acc(&s.ctl->acc[(v.c + 1) % 3]);
  const unsigned prev = (unsigned)((v.t - v.delta) & (WHEEL - 1));   // the bucket fired last cycle
  s.bndesc[prev] = 0; s.bnev[prev] = 0; s.bnlane[prev] = 0;
  s.ctl->hist_t[v.c & (WHEEL - 1)] = v.t;
  s.ctl->hist_head[v.c & (WHEEL - 1)] = *(volatile unsigned long long*)&s.ctl->ev_head;
}

// fire: the events of bucket t reach their destinations (Steps 1-3), one warp per run.
template <int D>
__device__ void wheel_fire(const Dev& s, const View& v, Smem& sm) {
  Acc* acc = &s.ctl->acc[v.c % 3];
  const unsigned b = (unsigned)(v.t & (WHEEL - 1));
  const unsigned nd = min(__ldcg(s.bndesc + b), s.dcap);
  const unsigned lane = threadIdx.x & 31u;
  const unsigned gw = blockIdx.x * WARPS + (threadIdx.x >> 5), nw = gridDim.x * WARPS;
  unsigned long long arr = 0;
  for (unsigned di = gw; di < nd; di += nw) {
    const unsigned long long dsc = __ldcg(s.bdesc + (size_t)b * s.dcap + di);
    const unsigned long long pos = dsc >> 24;
    const unsigned cnt = (unsigned)(dsc & 0xFFFFFFu);
    for (unsigned base = 0; base < cnt; base += 4 * 32) {
      unsigned long long e[4];
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        const unsigned i = base + it * 32 + lane;
        e[it] = i < cnt ? __ldcs(s.ev + ((pos + i) & s.ev_mask)) : ~0ull;
      }
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        const bool valid = e[it] != ~0ull;
        arr += valid;
        const unsigned src = (unsigned)e[it] & 0x3FFFFFFFu;
        const unsigned ln = (unsigned)(e[it] >> PH_LANE) & 7u;
        const int cand = (int)((e[it] >> PH_CAND) & 0xFFFFu);
        const unsigned via = ((e[it] >> EV_LANE_BIT) & 1) ? 0u : 1u;
        arrive(s, v, acc, valid, src + s.off[ln], cand, src, via);
      }
    }
  }
  block_reduce_commit(sm, 0xFFFFFFFFu, 0, arr, 0, 0, 0, acc);
}

// decide for the wheel: events-in-flight bookkeeping, next non-empty bucket,
// ring-capacity check.  Reads only state no block writes during decide.
__device__ void wheel_decide(const Dev& s, View& v, bool writer) {
  Acc* a = &s.ctl->acc[v.c % 3];
  Ctl* C = s.ctl;
  const unsigned long long bhit = __ldcg(&a->bhit);
  View nv = v;
  const unsigned b = (unsigned)(v.t & (WHEEL - 1));
  const long long pl = __ldcg((const long long*)&a->pend_lanes);      // E at the top of this cycle
  const long long pp = __ldcg((const long long*)&a->pend_phantoms);   // P at the top of this cycle
  const long long fired = v.c > 0 ? (long long)__ldcg(s.bnev + b) : 0;
  const long long fired_l = v.c > 0 ? (long long)__ldcg(s.bnlane + b) : 0;
  const long long new_l = (long long)__ldcg(&a->live);                // lanes started this cycle
  const long long new_p = (long long)__ldcg(&a->created);             // phantoms created this cycle
  const long long npl = pl - fired_l + new_l, npp = pp - (fired - fired_l) + new_p;
  if (writer) {
    const unsigned long long arrivals = __ldcg(&a->arrivals);
    const unsigned long long relabels = __ldcg(&a->relabels), triggered = __ldcg(&a->triggered);
    if (v.c > 0) {
      C->cycles += 1;
      C->edge_updates += pl + pp;
      if ((long long)v.c - 1 < s.trace_cap) {
        TraceRec r{v.t, (long long)v.delta, -1, pl, pp, (long long)triggered, (long long)arrivals, new_p,
                   (long long)relabels};
        s.trace[v.c - 1] = r;
      }
    }
    C->arrivals += arrivals; C->triggered += triggered; C->created += new_p; C->relabels += relabels;
  }
  if (bhit) {
    nv.status = 0;
    if (writer) resolve_hit(s, bhit, v.t);
  } else if (__ldcg(&C->wheel_overflow)) {
    nv.status = 8;  // WCSP_EOVERFLOW (descriptor table)
    if (writer) C->need_pool = -2;
  } else if (npl + npp == 0) {
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
    // region size: about the events one block files per delay per cycle (x2), in [128, 4096]
    const unsigned long long per = (unsigned long long)(new_l + new_p) * 2ull /
                                   ((unsigned long long)s.nblocks * (unsigned long long)max(1, s.f1max));
    unsigned r = 128;
    while (r < per && r < 4096u) r <<= 1;
    nv.region = r;
    // ring check: during this cycle's treat every event allocated by a cycle c' with
    // t(c') + f1max > t was still live; the treat's allocations must not have reached it
    const unsigned long long head = __ldcg(&C->ev_head);
    unsigned long long oldest = head;
    for (unsigned back = 0; back < (unsigned)WHEEL && back <= v.c; ++back) {
      const unsigned slot = (v.c - back) & (WHEEL - 1);
      if (__ldcg((const long long*)&C->hist_t[slot]) + s.f1max <= v.t) break;
      oldest = __ldcg(&C->hist_head[slot]);
    }
    if (head - oldest > s.ev_mask + 1) {
      nv.status = 8;  // live events may have been overwritten: the host grows the ring and re-runs
      if (writer) C->need_pool = (long long)(head - oldest);
    }
    if (writer) {
      if (npl + npp > C->peak_phantoms) C->peak_phantoms = npl + npp;
      C->acc[(v.c + 1) % 3].pend_lanes = npl;
      C->acc[(v.c + 1) % 3].pend_phantoms = npp;
    }
  }
  if (writer) C->view = nv;
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
    if ((lw & 0xFFFFu) != LBL_REMOVED && !lane_live(lw >> 16, t))
      *lp = (lw & 0xFFFFu) | ((unsigned)(t & 0xFFFF) << 16);
  }
}

__device__ __forceinline__ bool needs_maint(const View& prev, const View& nv) {
  return nv.status == ST_RUNNING &&
         (nv.stamp == 1u || (nv.t / MAINT_PERIOD_T) != (prev.t / MAINT_PERIOD_T));
}

template <int D>
__global__ void __launch_bounds__(THREADS, 4) k_wheel_persistent(Dev s) {
  Smem& sm = smem();
  init_smem(sm);
  View v;
  load_view(s, sm, v);
  const unsigned long long G = gridDim.x;
  unsigned long long target = 0;
  while (v.status == ST_RUNNING) {
    if (v.c > 0) {
      if (blockIdx.x == 0 && threadIdx.x == 0) wheel_cycle_start(s, v);
      wheel_fire<D>(s, v, sm);
      target += G;
      if (!grid_sync(s.ctl, target, sm)) return;
    }
    if (threadIdx.x == 0) sm.bhit = __ldcg(&s.ctl->acc[v.c % 3].bhit);
    __syncthreads();
    const unsigned long long bhit = sm.bhit;
    __syncthreads();
    if (!bhit) {
      phase_treat<D, true>(s, v, sm);
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
__global__ void __launch_bounds__(THREADS, 4) k_wheel_fire(Dev s) {
  Smem& sm = smem();
  init_smem(sm);
  View v;
  load_view(s, sm, v);
  if (v.status != ST_RUNNING || v.c == 0) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) wheel_cycle_start(s, v);
  wheel_fire<D>(s, v, sm);
}

template <int D>
__global__ void __launch_bounds__(THREADS, 4) k_wheel_treat(Dev s) {
  Smem& sm = smem();
  init_smem(sm);
  View v;
  load_view(s, sm, v);
  if (v.status != ST_RUNNING) return;
  if (__ldcg(&s.ctl->acc[v.c % 3].bhit)) return;
  phase_treat<D, true>(s, v, sm);
}

__global__ void k_wheel_decide(Dev s) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  View v = s.ctl->view;
  if (v.status != ST_RUNNING) return;
  const View prev = v;
  wheel_decide(s, v, true);
  if (needs_maint(prev, v)) s.ctl->view.status = ST_WRAP;
}

__global__ void __launch_bounds__(THREADS) k_wheel_maintain(Dev s) {
  const long long t = ((volatile View*)&s.ctl->view)->t;
  wheel_maintain(s, t);
}

}  // namespace wcspk
