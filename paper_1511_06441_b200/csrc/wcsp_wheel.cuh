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
constexpr int EV_SPECIAL_BIT = 50;        // the destination's temp is a sentinel (target / ghost): the fire
                                          // needs the atomic's old value for it
#ifndef WCSP_FIRE_RED
#define WCSP_FIRE_RED 1                   // dense single-device fires: ordinary arrivals as fire-and-forget
                                          // reductions (red.max) and an unconditional bitmap bit
#endif
#ifndef WCSP_FIRE_RED_PEER
#define WCSP_FIRE_RED_PEER 1              // ... and in the peer-halo engine (system-scope red.max)
#endif
constexpr int EV_DELAY_SHIFT = 56;
constexpr unsigned MAINT_PERIOD_T = 1u << 15;
#ifndef WCSP_FIRE_ITEMS
#define WCSP_FIRE_ITEMS 8
#endif
#ifndef WCSP_FIRE_PF
#define WCSP_FIRE_PF 0                    // 1: chunk c + 1's events load during chunk c (C2 -2 %, C3 +0.5 %: spills; off)
#endif
#ifndef WCSP_MINB
#define WCSP_MINB 3                       // resident blocks per SM the cycle kernels are compiled for
#endif
constexpr int FIRE_ITEMS = WCSP_FIRE_ITEMS;   // events per lane per fire chunk (atomics in flight)
// dense cycles, per build of the persistent kernel: the 4-blocks-per-SM build (3-D grids >= 2^21
// vertices) fires 12 events per lane (C3 135.1 -> 133.8 ms), the 3-block build 6 (C2 97.0 -> 95.1
// ms; profiles/r01/ab_v14_fire_hints.txt); sparse cycles of the 3-block build keep FIRE_ITEMS (C4 23.3 vs 26.3 ms at 6)
#ifndef WCSP_FIRE_ITEMS_4B
#define WCSP_FIRE_ITEMS_4B 12
#endif
#ifndef WCSP_FIRE_ITEMS_3B
#define WCSP_FIRE_ITEMS_3B 6
#endif
template <int MINB> __host__ __device__ constexpr int fire_items() { return MINB >= 4 ? WCSP_FIRE_ITEMS_4B : WCSP_FIRE_ITEMS_3B; }

// Runs are filed per (bucket, block): the block that treats a slab of the grid
// also fires the events its slab created, so the atomics of a fire phase
// walk compact regions of the state array (L2-resident) instead of the
// whole front at once.
// A storage overflow in a treat at time t: the flag for the host, and the earliest such time, which
// the hybrid kernel's decision reads only once every treat up to that time is complete.
__device__ __forceinline__ void flag_overflow(const Dev& s, unsigned bit, long long t) {
  atomicOr(&s.ctl->wheel_overflow, bit);
  atomicMin(&s.ctl->ovf_t, t);
}
__device__ __forceinline__ void file_run(const Dev& s, const Smem& sm, unsigned b, unsigned long long pos, unsigned cnt,
                                         long long t) {
  // after the ring guard fired in this block (hybrid kernel) nothing more is filed: the run is void
  // and is retried, but a neighbour's or this block's next fire must not read unwritten slots
  if (sm.ovf) return;
  const size_t slot = (size_t)b * s.nblocks + (blockIdx.x - s.blk0);
  const unsigned k = atomicAdd(s.bndesc + slot, 1u);
  if (k < s.dcap) s.bdesc[slot * s.dcap + k] = (pos << 24) | cnt;
  else flag_overflow(s, 2u, t);
}

__device__ void ev_stage(const Dev& s, Smem& sm, unsigned idx, unsigned long long rec, unsigned delay, long long t) {
  if (idx < (unsigned)QP_CAP) {
    sm.qp[idx] = rec | ((unsigned long long)delay << EV_DELAY_SHIFT);
    return;
  }
  // staging full: append to the block's open region for this delay while it has room (rfill,
  // rcap and rpos do not change between flushes; the next flush adopts the appended events) ...
  const unsigned k = atomicAdd(&sm.ofill[delay], 1u);
  if (k < sm.rcap[delay] - sm.rfill[delay]) {
    if (sm.ovf) return;                // the open region lies past the hybrid guard: drop (run retried)
    const unsigned b = (unsigned)((t + delay) & (WHEEL - 1));
    st_hint(s.ev + ((sm.rpos[delay] + sm.rfill[delay] + k) & s.ev_mask), rec, pol_first());
    atomicAdd(s.bnev + b, 1u);
    if ((rec >> EV_LANE_BIT) & 1) atomicAdd(s.bnlane + b, 1u);
    return;
  }
  const unsigned ks = atomicAdd(&sm.nspill, 1u);   // ... else spill it (sorted at the next flush) ...
  if (ks < s.spill_cap) {
    s.spill[(size_t)(blockIdx.x - s.blk0) * s.spill_cap + ks] = rec | ((unsigned long long)delay << EV_DELAY_SHIFT);
  } else {                          // ... else file the event as a run of one (rare)
    const unsigned long long pos = atomicAdd(&s.ctl->ev_head, 1ull);
    if (pos + 1 > sm.alloc_lim) { sm.ovf = 1; flag_overflow(s, 4u, t); return; }
    s.ev[pos & s.ev_mask] = rec;
    const unsigned b = (unsigned)((t + delay) & (WHEEL - 1));
    atomicAdd(s.bnev + b, 1u);
    if ((rec >> EV_LANE_BIT) & 1) atomicAdd(s.bnlane + b, 1u);
    file_run(s, sm, b, pos, 1u, t);
  }
}

__device__ void ev_push(const Dev& s, Smem& sm, bool pred, unsigned long long rec, unsigned delay, long long t) {
  const unsigned m = __ballot_sync(0xFFFFFFFFu, pred);
  if (m == 0) return;
  const unsigned lane = threadIdx.x & 31u;
  const int leader = __ffs(m) - 1;
  unsigned base = 0;
  if ((int)lane == leader) base = atomicAdd(&sm.np, (unsigned)__popc(m));
  base = __shfl_sync(0xFFFFFFFFu, base, leader);
  if (pred) ev_stage(s, sm, base + __popc(m & ((1u << lane) - 1u)), rec, delay, t);
}

#if WCSP_WARP_FLUSH
constexpr unsigned WQ = QP_CAP / WARPS;   // staging slots per warp

// Warp-level filing: the calling warp sorts its staged events by delay (warp-private
// histogram and ranks), reserves each delay's slots in the block's open region for that
// delay under a per-delay lock (opening a new region — and filing the full one as a run —
// when it has no room), and writes its events.  Only __syncwarp; other warps go on.
__device__ void warp_flush(const Dev& s, Smem& sm, long long t, unsigned region) {
  const unsigned w = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const unsigned n = sm.wnp[w];
  if (n == 0) return;
  unsigned* hist = sm.whist[w];
  const unsigned long long* q = sm.qp + (size_t)w * WQ;
  unsigned short* rk = sm.wrank + (size_t)w * WQ;
  for (unsigned d = lane; d < WHEEL; d += 32) hist[d] = 0;
  __syncwarp();
  for (unsigned i = lane; i < n; i += 32) {
    const unsigned long long e = q[i];
    const unsigned d = (unsigned)(e >> EV_DELAY_SHIFT);
    rk[i] = (unsigned short)(atomicAdd(&hist[d], 1u | ((unsigned)((e >> EV_LANE_BIT) & 1) << 16)) & 0xFFFFu);
  }
  __syncwarp();
  for (unsigned d = lane; d < WHEEL; d += 32) {
    const unsigned h = hist[d], cnt = h & 0xFFFFu;
    if (!cnt) continue;
    const unsigned b = (unsigned)((t + d) & (WHEEL - 1));
    while (atomicCAS(&sm.rlock[d], 0, 1) != 0) { }
    volatile unsigned* rfill = sm.rfill;
    volatile unsigned* rcap = sm.rcap;
    volatile unsigned long long* rpos = sm.rpos;
    if (rfill[d] + cnt > rcap[d]) {
      if (rfill[d]) file_run(s, sm, b, rpos[d], rfill[d], t);
      const unsigned size = max(region, cnt);
      rpos[d] = atomicAdd(&s.ctl->ev_head, (unsigned long long)size);
      rfill[d] = 0;
      rcap[d] = size;
    }
    const unsigned long long base = rpos[d] + rfill[d];
    rfill[d] = rfill[d] + cnt;
    __threadfence_block();
    atomicExch(&sm.rlock[d], 0);
    hist[d] = (unsigned)(base & s.ev_mask);   // the ring holds at most 2^32 slots
    atomicAdd(s.bnev + b, cnt);
    if (h >> 16) atomicAdd(s.bnlane + b, h >> 16);
  }
  __syncwarp();
  for (unsigned i = lane; i < n; i += 32) {
    const unsigned long long e = q[i];
    const unsigned d = (unsigned)(e >> EV_DELAY_SHIFT);
    st_hint(s.ev + ((hist[d] + (unsigned long long)rk[i]) & s.ev_mask), e & ((1ull << EV_DELAY_SHIFT) - 1),
            pol_first());
  }
  __syncwarp();
  if (lane == 0) sm.wnp[w] = 0;
  __syncwarp();
}

__device__ void ev_push_warp(const Dev& s, Smem& sm, bool pred, unsigned long long rec, unsigned delay, long long t,
                             unsigned region) {
  const unsigned m = __ballot_sync(0xFFFFFFFFu, pred);
  if (m == 0) return;
  const unsigned w = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  unsigned n = sm.wnp[w];
  if (n + (unsigned)__popc(m) > WQ) {
    warp_flush(s, sm, t, region);
    n = 0;
  }
  if (pred) sm.qp[(size_t)w * WQ + n + __popc(m & ((1u << lane) - 1u))] = rec | ((unsigned long long)delay << EV_DELAY_SHIFT);
  __syncwarp();
  if (lane == 0) sm.wnp[w] = n + (unsigned)__popc(m);
  __syncwarp();
}

// End of a treat phase: after every warp has filed its events, file the open regions.
__device__ void regions_close(const Dev& s, Smem& sm, long long t) {
  __syncthreads();
  for (unsigned d = threadIdx.x; d < WHEEL; d += THREADS) {
    if (sm.rfill[d]) file_run(s, sm, (unsigned)((t + d) & (WHEEL - 1)), sm.rpos[d], sm.rfill[d], t);
    sm.rfill[d] = 0;
    sm.rcap[d] = 0;
  }
  __syncthreads();
}
#endif

// Counting-sort sm.qp[0, n) by delay and append each delay's events to the
// block's open region for that delay (opening a new region of `region` slots
// when it is full).
__device__ void flush_sorted(const Dev& s, Smem& sm, long long t, unsigned region, unsigned n) {
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
        if (sm.rfill[d]) file_run(s, sm, b, sm.rpos[d], sm.rfill[d], t);
        const unsigned size = max(region, cnt);
        sm.rpos[d] = atomicAdd(&s.ctl->ev_head, (unsigned long long)size);
        sm.rfill[d] = 0;
        sm.rcap[d] = size;
        if (sm.rpos[d] + size > sm.alloc_lim) {   // would overwrite live events (hybrid kernel): drop
          sm.ovf = 1;                             // this treat's stores, flag, the run is retried
          flag_overflow(s, 4u, t);
        }
      }
      sm.hbase[d] = sm.rpos[d] + sm.rfill[d];
      sm.rfill[d] += cnt;
      atomicAdd(s.bnev + b, cnt);
      if (sm.hlane[d]) atomicAdd(s.bnlane + b, sm.hlane[d]);
    }
  }
  __syncthreads();
  if (!sm.ovf) {
    for (unsigned i = threadIdx.x; i < n; i += THREADS) {
      const unsigned long long e = sm.qp[i];
      const unsigned d = (unsigned)(e >> EV_DELAY_SHIFT);
      st_hint(s.ev + ((sm.hbase[d] + sm.rank[i]) & s.ev_mask), e & ((1ull << EV_DELAY_SHIFT) - 1), pol_first());
    }
  }
  __syncthreads();
}

// Flush the staging: events appended past it into open regions are adopted, the
// staged events are sorted into regions, then the spilled ones (QP_CAP at a time
// through the staging); final_flush files every open region.
__device__ void ev_flush(const Dev& s, Smem& sm, long long t, unsigned region, bool final_flush) {
  __syncthreads();
  const unsigned n = min(sm.np, (unsigned)QP_CAP);
  const unsigned ns = min(sm.nspill, s.spill_cap);
  unsigned appended = 0;
  for (unsigned d = threadIdx.x; d < WHEEL; d += THREADS) {
    const unsigned o = sm.ofill[d];
    if (o) {
      const unsigned a = min(o, sm.rcap[d] - sm.rfill[d]);
      sm.rfill[d] += a;
      sm.ofill[d] = 0;
      appended += a;
    }
  }
  // staging-overflow statistics (rare paths; tests check they were exercised)
  if (appended) atomicAdd(&s.ctl->n_appended, (unsigned long long)appended);
  if (threadIdx.x == 0 && sm.nspill) {
    atomicAdd(&s.ctl->n_spilled, (unsigned long long)ns);
    if (sm.nspill > ns) atomicAdd(&s.ctl->n_single, (unsigned long long)(sm.nspill - ns));
  }
  if (n > 0) flush_sorted(s, sm, t, region, n);
  const unsigned long long* sp = s.spill + (size_t)(blockIdx.x - s.blk0) * s.spill_cap;
  for (unsigned c0 = 0; c0 < ns; c0 += QP_CAP) {
    const unsigned cn = min((unsigned)QP_CAP, ns - c0);
    __syncthreads();
    for (unsigned i = threadIdx.x; i < cn; i += THREADS) sm.qp[i] = __ldcg(sp + c0 + i);
    flush_sorted(s, sm, t, region, cn);
  }
  __syncthreads();
  if (threadIdx.x == 0) { sm.np = 0; sm.nspill = 0; }
  if (final_flush) {
    for (unsigned d = threadIdx.x; d < WHEEL; d += THREADS) {
      if (sm.rfill[d]) file_run(s, sm, (unsigned)((t + d) & (WHEEL - 1)), sm.rpos[d], sm.rfill[d], t);
      sm.rfill[d] = 0;
      sm.rcap[d] = 0;
    }
  }
  __syncthreads();
}

// Start-of-cycle bookkeeping (block 0, thread 0, before the fire phase).
__device__ __forceinline__ void wheel_cycle_start(const Dev& s, const View& v) {
  reset_acc(&s.ctl->acc[(v.c + 1) % NACC]);
  s.ctl->ts0 = globaltimer_ns();
  // staircase: target arrivals are resolved per cycle; the list of the previous cycle's parity (read by
  // its decide, which this thread ran) is emptied for the next cycle — the fires of THIS cycle, which
  // other blocks may already have started, append to the other parity's list
  if (s.staircase) s.ctl->n_barr2[(v.c + 1) & 1] = 0;
  unsigned long long* nf = &s.ctl->fin[(v.c + 1) & 1][0][0];
  nf[0] = 0; nf[1] = 0; nf[2] = 0; nf[3] = 0;
  const unsigned prev = (unsigned)((v.t - v.delta) & (WHEEL - 1));   // the bucket fired last cycle
  s.bnev[prev] = 0; s.bnlane[prev] = 0;
  s.ctl->hist_t[v.c & (WHEEL - 1)] = v.t;
  s.ctl->hist_head[v.c & (WHEEL - 1)] = *(volatile unsigned long long*)&s.ctl->ev_head;
}

// fire: the events of bucket t reach their destinations (Steps 1-3).  Block k
// fires the runs its own slab filed; the runs are cut into chunks of
// FIRE_ITEMS * 32 events that the block's warps take in turn (a prefix sum of
// chunk counts over the block's runs lives in shared memory).
// run descriptors staged per pass: dpos[MAXD] (u64) + dchunk[MAXD + 1] (u32) in the wl union
constexpr unsigned FIRE_WL_BYTES = sizeof(Smem::wl);
constexpr unsigned FIRE_MAXD = ((FIRE_WL_BYTES - 4) / 12 >= 512 ? 512u : ((FIRE_WL_BYTES - 4) / 12) & ~31u);
static_assert(FIRE_MAXD >= 32 && FIRE_MAXD * 8 + (FIRE_MAXD + 1) * 4 <= FIRE_WL_BYTES,
              "descriptor staging exceeds Smem::wl");

// One pass of the fire's descriptor staging (warp 0): descriptors [d0, d0 + n) and the prefix sum of
// their chunk counts, chunks of CH events.
template <unsigned CH>
__device__ __forceinline__ void fire_stage(Smem& sm, const unsigned long long* dl, unsigned d0, unsigned n) {
  unsigned long long* dpos = reinterpret_cast<unsigned long long*>(&sm.wl[0][0]);   // [MAXD]
  unsigned* dchunk = reinterpret_cast<unsigned*>(dpos + FIRE_MAXD);                   // [MAXD + 1] prefix
  const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  if (warp != 0) return;
  unsigned carry = 0;
  for (unsigned i0 = 0; i0 < n; i0 += 32) {
    const unsigned i = i0 + lane;
    unsigned long long dsc = 0;
    unsigned ch = 0;
    if (i < n) {
      dsc = __ldcg(dl + d0 + i);
      ch = ((unsigned)(dsc & 0xFFFFFFu) + CH - 1) / CH;
      dpos[i] = dsc;
    }
    unsigned x = ch;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if ((int)lane >= o) x += y;
    }
    if (i < n) dchunk[i] = carry + x - ch;
    carry += __shfl_sync(0xFFFFFFFFu, x, 31);
  }
  if (lane == 0) dchunk[n] = carry;
}

// The part of the fire of cycle v that reads only this block's own data: reset of the previous
// bucket's descriptor count, the block-local bitmap's range and zeroing, and the first pass of the
// descriptor staging.  The hybrid kernel runs it before its neighbourhood wait (the block's runs for
// the next bucket are complete once its own treat is), so those dependent loads overlap the wait.
template <int D, bool PEER = false, int FI = FIRE_ITEMS>
__device__ void fire_prologue(const Dev& s, const View& v, Smem& sm) {
  const unsigned b = (unsigned)(v.t & (WHEEL - 1));
  const unsigned vb = blockIdx.x - s.blk0;
  if (threadIdx.x == 0) s.bndesc[(size_t)((v.t - v.delta) & (WHEEL - 1)) * s.nblocks + vb] = 0;
  const size_t slot = (size_t)b * s.nblocks + vb;
  const unsigned nd = min(__ldcg(s.bndesc + slot), s.dcap);
  const bool local_bits = (PEER || !s.slab) && !v.lmode;
  if (local_bits) {
    if (threadIdx.x == 0) {
      const unsigned long long ww = s.win_words;
      unsigned wlo, whi, rounds;
      block_windows(s, blockIdx.x - s.blk0, (unsigned)((s.nwords + ww - 1) / ww), wlo, whi, rounds);
      const unsigned long long vlo = (unsigned long long)wlo * ww * 32ull;
      const unsigned long long vhi = min((unsigned long long)s.N, (unsigned long long)whi * ww * 32ull);
      const unsigned long long S = s.off[s.NL - 2], cap = (unsigned long long)QP_CAP * 64ull;
      unsigned long long lo = vlo >= S ? vlo - S : 0ull, hi = min((unsigned long long)s.N, vhi + S);
      if (PEER) {                  // never a ghost plane: those are the neighbours' vertices
        lo = max(lo, (unsigned long long)s.plo_end);
        hi = min(hi, (unsigned long long)s.ghost_hi_start);
      }
      if (hi - lo + 32 > cap) { lo = vlo; hi = vhi; }
      if (vlo >= vhi || hi <= lo || hi - lo + 32 > cap || s.ileave) { lo = 0; hi = 0; }   // interleaved: no own slab
      lo &= ~31ull;
      sm.bm_lo = (unsigned)lo;
      sm.bm_words = (unsigned)((hi - lo + 31) / 32);
    }
    __syncthreads();
    uint4* bm4 = reinterpret_cast<uint4*>(sm.qp);   // 16-byte stores (qp is 16-byte aligned)
    for (unsigned i = threadIdx.x; i < (sm.bm_words + 3) / 4; i += THREADS) bm4[i] = make_uint4(0u, 0u, 0u, 0u);
  } else if (threadIdx.x == 0) {
    sm.bm_lo = 0;
    sm.bm_words = 0;
  }
  __syncthreads();
  if (nd > 0) fire_stage<FI * 32>(sm, s.bdesc + slot * s.dcap, 0, min(FIRE_MAXD, nd));
  if (threadIdx.x == 0) { sm.f_nd = nd; sm.f_prep = 1; }
  __syncthreads();
}

template <int D, bool PEER = false, int FI = FIRE_ITEMS>   // FI: events per lane per chunk
__device__ void wheel_fire(const Dev& s, const View& v, Smem& sm) {
  Acc* acc = &s.ctl->acc[v.c % NACC];
  const unsigned b = (unsigned)(v.t & (WHEEL - 1));
  const unsigned vb = blockIdx.x - s.blk0;
  if (!sm.f_prep) fire_prologue<D, PEER, FI>(s, v, sm);   // not yet run ahead by the hybrid kernel
  const size_t slot = (size_t)b * s.nblocks + vb;
  const unsigned nd = sm.f_nd;
  const unsigned long long* dl = s.bdesc + slot * s.dcap;
  constexpr unsigned CH = FI * 32;
  constexpr unsigned MAXD = FIRE_MAXD;
  unsigned long long* dpos = reinterpret_cast<unsigned long long*>(&sm.wl[0][0]);   // [MAXD]
  unsigned* dchunk = reinterpret_cast<unsigned*>(dpos + MAXD);                        // [MAXD + 1] prefix
  const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  unsigned arr = 0;
  // Dense cycles: first arrivals near the block's own slab of the grid (its treat windows and one
  // plane of the last axis on either side: where the events it fires lead) set bits of a
  // shared-memory bitmap (the treat staging is free during the fire; set up by fire_prologue),
  // merged into the global bitmap with one atomicOr per word at the end; sparse cycles list them.
  const bool local_bits = (PEER || !s.slab) && !v.lmode;
  const bool redmode = local_bits;
  for (unsigned d0 = 0; d0 < nd; d0 += MAXD) {
    const unsigned n = min(MAXD, nd - d0);
    if (d0 > 0) {                  // pass 0 was staged by fire_prologue
      __syncthreads();
      fire_stage<CH>(sm, dl, d0, n);
    }
    __syncthreads();
    const unsigned nchunks = dchunk[n];
    // warp w fires a contiguous range of chunks (the descriptor index then advances by at most
    // one per chunk); the first descriptor is found by binary search over the prefix sums
    // s.fstride: the block's warps take chunks in turn (c = warp, warp + WARPS, ...), so every
    // block walks its run lists front to back — i.e. in the order its treat rounds filed them — and
    // the whole device fires the events of about one treat round per block at a time (a working set
    // of ~3 x rounds' state words instead of the whole front).  Otherwise warp w fires a contiguous
    // eighth of the list.
    const unsigned cstep = s.fstride ? (unsigned)WARPS : 1u;
    const unsigned c_lo = s.fstride ? warp : (unsigned)((unsigned long long)nchunks * warp / WARPS);
    const unsigned c_hi = s.fstride ? nchunks : (unsigned)((unsigned long long)nchunks * (warp + 1) / WARPS);
    unsigned di = 0;
    {
      unsigned lo = 0, hi = n;                   // largest di with dchunk[di] <= c_lo
      while (hi - lo > 1) {
        const unsigned mid = (lo + hi) >> 1;
        if (dchunk[mid] <= c_lo) lo = mid; else hi = mid;
      }
      di = lo;
    }
    // chunk c's events: descriptor di (advanced monotonically), FIRE_ITEMS per lane
    auto load_chunk = [&](unsigned c, unsigned long long (&ev)[FI]) {
      while (dchunk[di + 1] <= c) ++di;
      const unsigned long long dsc = dpos[di];
      const unsigned long long pos = dsc >> 24;
      const unsigned cnt = (unsigned)(dsc & 0xFFFFFFu);
      const unsigned base = (c - dchunk[di]) * CH;
#pragma unroll
      for (int it = 0; it < FI; ++it) {
        const unsigned i = base + it * 32 + lane;
        ev[it] = i < cnt ? ld_hint(s.ev + ((pos + i) & s.ev_mask), pol_first()) : ~0ull;
      }
    };
    unsigned long long e[FI];
    if (c_lo < c_hi) load_chunk(c_lo, e);
    for (unsigned c = c_lo; c < c_hi; c += cstep) {
#if WCSP_FIRE_PF
      unsigned long long en[FI];   // the next chunk's events load while this one fires
      if (c + cstep < c_hi) load_chunk(c + cstep, en);
#endif
      unsigned old[FI];
#pragma unroll
      for (int it = 0; it < FI; ++it) {   // put every atomic in flight before using a result
        const bool valid = e[it] != ~0ull;
        arr += valid;
        const unsigned src = (unsigned)e[it] & 0x3FFFFFFFu;
        const unsigned ln = (unsigned)(e[it] >> PH_LANE) & 7u;
        WCSP_CHECK(!valid || (src < s.N && ln < (unsigned)s.NL && src + s.off[ln] < s.N), "fire: event record",
                   e[it], s.N);
#if WCSP_FIRE_RED
        if constexpr (PEER) {
#if WCSP_FIRE_RED_PEER
          // the same with system-scope reductions (a neighbour's words may live on another GPU)
          if (redmode && valid && !((e[it] >> EV_SPECIAL_BIT) & 1)) {
            const unsigned dst = src + s.off[ln];
            const Loc L = locate<true>(s, dst);
            red_max_sys(tmp_ptr(L.sw, L.idx), (v.stamp << 16) | (unsigned)((e[it] >> PH_CAND) & 0xFFFFu));
            const unsigned r = dst - sm.bm_lo;
            if (L.sw == s.sw && r < sm.bm_words * 32u)
              atomicOr(reinterpret_cast<unsigned*>(sm.qp) + (r >> 5), 1u << (r & 31u));
            else
              atom_or_sys(L.tb + (L.idx >> 5), 1u << (L.idx & 31u));
            old[it] = v.stamp << 16;
            continue;
          }
#endif
        } else {
          // No first-arrival test needed here: the bit of D is set on every arrival (same set
          // of bits), so only sentinel destinations (targets, ghosts) need the old value.
          if (redmode && valid && !((e[it] >> EV_SPECIAL_BIT) & 1)) {
            const unsigned dst = src + s.off[ln];
            red_max_hint(tmp_ptr(s.sw, dst), (v.stamp << 16) | (unsigned)((e[it] >> PH_CAND) & 0xFFFFu), pol_last());
            const unsigned r = dst - sm.bm_lo;
            if (r < sm.bm_words * 32u) atomicOr(reinterpret_cast<unsigned*>(sm.qp) + (r >> 5), 1u << (r & 31u));
            else atomicOr(s.tbits + (dst >> 5), 1u << (dst & 31u));
            old[it] = v.stamp << 16;       // as if a later arrival of this cycle: arrive_post does nothing
            continue;
          }
        }
#endif
        old[it] = arrive_atomic<PEER>(s, v, valid, src + s.off[ln], (int)((e[it] >> PH_CAND) & 0xFFFFu));
      }
#pragma unroll
      for (int it = 0; it < FI; ++it) {
        const unsigned src = (unsigned)e[it] & 0x3FFFFFFFu;
        const unsigned ln = (unsigned)(e[it] >> PH_LANE) & 7u;
        const unsigned via = ((e[it] >> EV_LANE_BIT) & 1) ? 0u : 1u;
        arrive_post<PEER, true>(s, v, acc, old[it], src + s.off[ln], (int)((e[it] >> PH_CAND) & 0xFFFFu),
                                src + s.goff, via, local_bits || (!s.slab && v.lmode) ? &sm : nullptr);
      }
#if WCSP_FIRE_PF
#pragma unroll
      for (int it = 0; it < FI; ++it) e[it] = en[it];
#else
      if (c + cstep < c_hi) load_chunk(c + cstep, e);
#endif
    }
  }
  if (local_bits) {                 // merge the shared-memory bitmap
    __syncthreads();
    const uint4* bm4 = reinterpret_cast<const uint4*>(sm.qp);
    const unsigned w0 = sm.bm_lo >> 5, nw = sm.bm_words;
    for (unsigned i = threadIdx.x; i < (nw + 3) / 4; i += THREADS) {
      const uint4 q4 = bm4[i];
      const unsigned ws[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const unsigned w = ws[k], j = 4 * i + k;
        if (w && j < nw) {
          if constexpr (PEER) atom_or_sys(s.tbits + w0 + j, w);   // the neighbours OR into it too
          else atomicOr(s.tbits + w0 + j, w);
        }
      }
    }
  }
  if constexpr (!PEER) {            // publish the block's triggered list for its treat (sparse cycles)
    if (!s.slab && v.lmode) {
      __syncthreads();
      const unsigned n = sm.na, m = min(n, (unsigned)QA_CAP);
      if (threadIdx.x == 0) {
        sm.base_a = m ? atomicAdd(&acc->tl_total, m) : 0u;   // sum over blocks <= nblocks * QA_CAP
        if (n > m) atomicOr(&acc->tl_over, 1u);
      }
      __syncthreads();
      for (unsigned i = threadIdx.x; i < m; i += THREADS) s.tlist[(size_t)sm.base_a + i] = sm.qa[i];
    }
  }
  block_reduce_commit(sm, 0xFFFFFFFFu, 0, arr, 0, 0, 0, acc);   // (ends with a block barrier:
  if (threadIdx.x == 0) { sm.na = 0; sm.f_prep = 0; }           //  every thread has read sm.na)
}

// The wheel's local proposal for the decision of cycle c (see Prop): best
// target arrival, steps to the next non-empty bucket, any live edge, and the
// storage checks (descriptor table; event ring: during this cycle's treat every
// event allocated by a cycle c' with t(c') + f1max > t was still live and the
// treat's allocations must not have reached it).  *need = ring slots needed.
__device__ Prop wheel_propose(const Dev& s, const View& v, long long* need) {
  Acc* a = &s.ctl->acc[v.c % NACC];
  Ctl* C = s.ctl;
  const unsigned b = (unsigned)(v.t & (WHEEL - 1));
  const long long pl = __ldcg((const long long*)&a->pend_lanes);
  const long long pp = __ldcg((const long long*)&a->pend_phantoms);
  const long long fired = v.c > 0 ? (long long)__ldcg(s.bnev + b) : 0;
  const long long fired_l = v.c > 0 ? (long long)__ldcg(s.bnlane + b) : 0;
  const long long npl = pl - fired_l + (long long)__ldcg(&a->started);
  const long long npp = pp - (fired - fired_l) + (long long)__ldcg(&a->created);
  Prop p;
  p.bhit = (long long)__ldcg(&a->bhit);
  p.pending = npl + npp > 0;
  unsigned k = 1;
  if (!s.unit)
    while (k < (unsigned)WHEEL && __ldcg(s.bnev + ((b + k) & (WHEEL - 1))) == 0) ++k;
  p.negk = -(long long)k;
  const unsigned long long head = __ldcg(&C->ev_head);
  unsigned long long oldest = head;
  for (unsigned back = 0; back < (unsigned)WHEEL && back <= v.c; ++back) {
    const unsigned slot = (v.c - back) & (WHEEL - 1);
    if (__ldcg((const long long*)&C->hist_t[slot]) + s.f1max <= v.t) break;
    oldest = __ldcg(&C->hist_head[slot]);
  }
  *need = 0;
  p.overflow = 0;
  if (__ldcg(&C->wheel_overflow)) { p.overflow = 1; *need = -2; }
  if (head - oldest > s.ev_mask + 1) { p.overflow = 1; *need = (long long)(head - oldest); }
  return p;
}

// The same proposal computed by a whole warp (every lane calls it): the scan for the next
// non-empty bucket and the walk back over the cycles whose events may still be live read
// 32 slots per step instead of one dependent load after another.
__device__ Prop wheel_propose_warp(const Dev& s, const View& v, long long* need) {
  const unsigned lane = threadIdx.x & 31u;
  Acc* a = &s.ctl->acc[v.c % NACC];
  Ctl* C = s.ctl;
  const unsigned b = (unsigned)(v.t & (WHEEL - 1));
  Prop p;
  {
    const long long pl = __ldcg((const long long*)&a->pend_lanes);
    const long long pp = __ldcg((const long long*)&a->pend_phantoms);
    const long long fired = v.c > 0 ? (long long)__ldcg(s.bnev + b) : 0;
    const long long fired_l = v.c > 0 ? (long long)__ldcg(s.bnlane + b) : 0;
    const long long npl = pl - fired_l + (long long)__ldcg(&a->started);
    const long long npp = pp - (fired - fired_l) + (long long)__ldcg(&a->created);
    p.bhit = (long long)__ldcg(&a->bhit);
    p.pending = npl + npp > 0;
  }
  unsigned k = 1;
  if (!s.unit) {
    k = WHEEL;
    for (unsigned k0 = 1; k0 < (unsigned)WHEEL; k0 += 32) {
      const unsigned kk = k0 + lane;
      const bool nz = kk < (unsigned)WHEEL && __ldcg(s.bnev + ((b + kk) & (WHEEL - 1))) != 0;
      const unsigned m = __ballot_sync(0xFFFFFFFFu, nz);
      if (m) { k = k0 + (unsigned)(__ffs(m) - 1); break; }
    }
  }
  p.negk = -(long long)k;
  const unsigned long long head = __ldcg(&C->ev_head);
  const unsigned lim = min((unsigned)WHEEL, v.c + 1u);   // slots back = 0 .. lim - 1
  unsigned B = lim;                                      // first back whose cycle's events are all fired
  for (unsigned b0 = 0; b0 < lim; b0 += 32) {
    const unsigned back = b0 + lane;
    const bool done = back < lim &&
                      __ldcg((const long long*)&C->hist_t[(v.c - back) & (WHEEL - 1)]) + s.f1max <= v.t;
    const unsigned m = __ballot_sync(0xFFFFFFFFu, done);
    if (m) { B = b0 + (unsigned)(__ffs(m) - 1); break; }
  }
  const unsigned long long oldest = B == 0 ? head : __ldcg(&C->hist_head[(v.c - (B - 1)) & (WHEEL - 1)]);
  *need = 0;
  p.overflow = 0;
  if (__ldcg(&C->wheel_overflow)) { p.overflow = 1; *need = -2; }
  if (head - oldest > s.ev_mask + 1) { p.overflow = 1; *need = (long long)(head - oldest); }
  return p;
}

// decide for the wheel (Step 6 + time skipping).  Single device: g = its own
// proposal; slab engine: g = the max-combined proposals of all slabs.  Reads
// only state no block writes during decide.
__device__ void wheel_decide(const Dev& s, View& v, bool writer, const Prop* gext = nullptr,
                             const Prop* lpre = nullptr, long long need_pre = 0) {
  Acc* a = &s.ctl->acc[v.c % NACC];
  Ctl* C = s.ctl;
  View nv = v;
  const unsigned b = (unsigned)(v.t & (WHEEL - 1));
  const long long pl = __ldcg((const long long*)&a->pend_lanes);      // E at the top of this cycle
  const long long pp = __ldcg((const long long*)&a->pend_phantoms);   // P at the top of this cycle
  const long long fired = v.c > 0 ? (long long)__ldcg(s.bnev + b) : 0;
  const long long fired_l = v.c > 0 ? (long long)__ldcg(s.bnlane + b) : 0;
  const long long new_l = (long long)__ldcg(&a->started);             // lanes started this cycle
  const long long new_p = (long long)__ldcg(&a->created);             // phantoms created this cycle
  const long long npl = pl - fired_l + new_l, npp = pp - (fired - fired_l) + new_p;
  long long need = need_pre;
  const Prop L = lpre ? *lpre : wheel_propose(s, v, &need);
  Prop G = L;
  if (gext) {
    G = *gext;
  } else if (s.slab) {
    const volatile Prop* gp = &C->gprop;
    G.bhit = gp->bhit; G.negk = gp->negk; G.pending = gp->pending; G.overflow = gp->overflow;
  }
  if (writer) {
    const unsigned long long arrivals = __ldcg(&a->arrivals);
    const unsigned long long relabels = __ldcg(&a->relabels), triggered = __ldcg(&a->triggered);
    if (v.c > 0) {
      C->cycles += 1;
      C->edge_updates += pl + pp;
      if ((long long)v.c - 1 < s.trace_cap) {
        const unsigned long long t2 = globaltimer_ns();
        TraceRec r{v.t, (long long)v.delta, (long long)__ldcg(s.bndesc + (size_t)b * s.nblocks), pl, pp,
                   (long long)triggered, (long long)arrivals, new_p, (long long)relabels,
                   (long long)__ldcg(&a->tested), (long long)(C->ts1 - C->ts0), (long long)(t2 - C->ts1),
                   (long long)(C->fin[v.c & 1][0][0] - C->fin[v.c & 1][0][1] / s.nblocks),
                   (long long)(C->fin[v.c & 1][1][0] - C->fin[v.c & 1][1][1] / s.nblocks)};
        s.trace[v.c - 1] = r;
      }
    }
    C->arrivals += arrivals; C->triggered += triggered; C->created += new_p; C->relabels += relabels;
    C->started += new_l;
  }
  // staircase mode: a target arrival that beats every earlier one is a step of
  // the F1*(M) staircase; the run goes on until nothing is live (or a step reaches f2_stop)
  bool hit_stop = G.bhit != 0;
  if (G.bhit && s.staircase) {
    const long long q = (long long)((unsigned long long)G.bhit >> 32);
    if (writer && q > C->stair_q) {
      resolve_hit(s, (unsigned long long)G.bhit, v.t, v.c);
      const unsigned k = C->n_stair;
      if (k < s.stair_cap) {
        s.stair[4 * k] = v.t;
        s.stair[4 * k + 1] = C->F2;
        s.stair[4 * k + 2] = C->X;
        s.stair[4 * k + 3] = C->Y;
      }
      C->n_stair = k + 1;
      C->stair_q = q;
    }
    hit_stop = (s.minf ? -1 : (long long)s.M - q) <= s.f2stop;
  }
  if (hit_stop) {
    nv.status = 0;
    if (writer && !s.staircase) resolve_hit(s, (unsigned long long)G.bhit, v.t, v.c);
  } else if (G.overflow) {
    nv.status = 8;  // WCSP_EOVERFLOW: the host grows the event ring / descriptor table and re-runs
    if (writer) C->need_pool = need;
  } else if (!G.pending) {
    nv.status = s.staircase && __ldcg(&C->n_stair) ? 0 : 1;  // 2°: no live edge
  } else if (s.budget > 0 && (long long)v.c >= s.budget) {
    nv.status = 4;
  } else {
    const unsigned k = (unsigned)(-G.negk);
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
    // sparse cycles (thin fronts: C4, the 2-D grids) list their triggered vertices instead of
    // having the treat scan the whole bitmap; the previous cycle's count predicts the next one's
    nv.lmode = !s.slab && __ldcg(&a->triggered) <= s.list_max;
    if (writer) {
      if (npl + npp > C->peak_phantoms) C->peak_phantoms = npl + npp;
      C->acc[(v.c + 1) % NACC].pend_lanes = npl;
      C->acc[(v.c + 1) % NACC].pend_phantoms = npp;
    }
  }
  if (writer) C->view = nv;
  v = nv;
}

// ---------------------------------------------------------------------------
// slab engine: the grid is cut into slabs along its last axis;
// each slab keeps one ghost plane per neighbour.  Water arriving at a ghost
// vertex is max-combined into ghost_out_* (stamp | cand | ~src | !via) and
// handed to the owner, which applies it like a local arrival before its treat.
// After the treat the owner's boundary labels refresh the neighbour's ghost
// labels (stale by at most one cycle: they only weaken the Step-4 pruning,
// which stays exact — SURVEY E6, E14).
// ---------------------------------------------------------------------------
__global__ void k_slab_propose(Dev s) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const View v = s.ctl->view;
  if (v.status != ST_RUNNING) return;
  long long need = 0;
  s.ctl->prop = wheel_propose(s, v, &need);
}

// virtual slabs on one device: combine the proposals (element-wise max)
__global__ void k_slab_reduce(Ctl* const* ctls, int nslabs) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (((volatile View*)&ctls[0]->view)->status != ST_RUNNING) return;
  Prop g = ctls[0]->prop;
  for (int i = 1; i < nslabs; ++i) {
    const Prop p = ctls[i]->prop;
    g.bhit = max(g.bhit, p.bhit); g.negk = max(g.negk, p.negk);
    g.pending = max(g.pending, p.pending); g.overflow = max(g.overflow, p.overflow);
  }
  for (int i = 0; i < nslabs; ++i) ctls[i]->gprop = g;
}

// apply the water a neighbour handed over for this slab's boundary plane
__global__ void __launch_bounds__(THREADS) k_slab_apply(Dev s, const unsigned long long* in, unsigned dst0) {
  const View v = s.ctl->view;
  if (v.status != ST_RUNNING || v.c == 0) return;
  Acc* acc = &s.ctl->acc[v.c % NACC];
  for (unsigned i = blockIdx.x * THREADS + threadIdx.x; i < s.plane; i += gridDim.x * THREADS) {
    const unsigned long long w = __ldcg(in + i);
    if ((unsigned)(w >> 48) != v.stamp) continue;
    const unsigned D = dst0 + i;
    const int cand = (int)((w >> 32) & 0xFFFFu);
    const unsigned src = 0x7FFFFFFFu - (unsigned)((w >> 1) & 0x7FFFFFFFu);
    const unsigned via = (w & 1) ? 0u : 1u;
    const unsigned old = atomicMax(tmp_ptr(s.sw, D), (v.stamp << 16) | (unsigned)cand);
    arrive_post(s, v, acc, old, D, cand, src, via);
  }
}

// boundary labels -> plane buffer, and plane buffer -> ghost labels
__global__ void __launch_bounds__(THREADS) k_slab_gather_labels(Dev s, unsigned src0, unsigned* out) {
  for (unsigned i = blockIdx.x * THREADS + threadIdx.x; i < s.plane; i += gridDim.x * THREADS)
    out[i] = *lbl_ptr(s.sw, src0 + i) & 0xFFFFu;
}
__global__ void __launch_bounds__(THREADS) k_slab_scatter_labels(Dev s, const unsigned* in, unsigned dst0) {
  for (unsigned i = blockIdx.x * THREADS + threadIdx.x; i < s.plane; i += gridDim.x * THREADS) {
    unsigned* lp = lbl_ptr(s.sw, dst0 + i);
    if ((*lp & 0xFFFFu) != LBL_REMOVED) *lp = in[i];
  }
}

// Maintenance (rare): forget stale temps and refresh lane-expiry times so the
// 16-bit stamp and texp comparisons stay unambiguous.
__device__ __forceinline__ void wheel_maintain(const Dev& s, long long t) {
  for (unsigned long long i = (unsigned long long)(blockIdx.x - s.blk0) * THREADS + threadIdx.x; i < s.N;
       i += (unsigned long long)s.nblocks * THREADS) {
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

// MINB: resident blocks per SM the kernel is compiled for.  4 (64 registers) wins on big grids
// (C3 157.8 -> 135.6 ms: more warps hide the treat's gather latency), 3 (80 registers) on thin or
// small ones (C2, C4: fewer blocks in every grid barrier, no spills); the host picks by grid size.
template <int D, int MINB = WCSP_MINB>
__global__ void __launch_bounds__(THREADS, MINB) k_wheel_persistent(Dev s) {
  Smem& sm = smem();
  init_smem(sm);
  View v;
  load_view(s, sm, v);
  const unsigned long long G = gridDim.x;
  unsigned long long target = 0;
  while (v.status == ST_RUNNING) {
    if (v.c > 0) {
      if (blockIdx.x == 0 && threadIdx.x == 0) wheel_cycle_start(s, v);
      if (threadIdx.x == 0) sm.tphase = globaltimer_ns();
      // 3-block build: sparse cycles (thin fronts) keep FIRE_ITEMS; the 4-block build has no
      // registers for a second copy of the fire (spills) and fires 12 per lane throughout
      if (MINB < 4 && v.lmode) wheel_fire<D, false, FIRE_ITEMS>(s, v, sm);
      else wheel_fire<D, false, fire_items<MINB>()>(s, v, sm);
      target += G;
      if (!grid_sync(s.ctl, target, sm, s.trace_cap > 0 ? &s.ctl->fin[v.c & 1][0][0] : nullptr)) return;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) s.ctl->ts1 = globaltimer_ns();
    if (threadIdx.x == 0) sm.bhit = __ldcg(&s.ctl->acc[v.c % NACC].bhit);
    __syncthreads();
    const unsigned long long bhit = sm.bhit;
    __syncthreads();
    if (!bhit || s.staircase) {
      if (threadIdx.x == 0) sm.tphase = globaltimer_ns();
      phase_treat<D, true>(s, v, sm);
      target += G;
      if (!grid_sync(s.ctl, target, sm, s.trace_cap > 0 ? &s.ctl->fin[v.c & 1][1][0] : nullptr)) return;
    }
    const View prev = v;
    if (threadIdx.x < 32) {          // warp 0: the proposal in parallel, then lane 0 decides
      long long need = 0;
      const Prop L = wheel_propose_warp(s, v, &need);
      if (threadIdx.x == 0) {
        View nv = v;
        wheel_decide(s, nv, blockIdx.x == 0, nullptr, &L, need);
        sm.view = nv;
      }
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
__global__ void __launch_bounds__(THREADS, WCSP_MINB) k_wheel_fire(Dev s) {
  Smem& sm = smem();
  init_smem(sm);
  View v;
  load_view(s, sm, v);
  if (v.status != ST_RUNNING || v.c == 0) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) wheel_cycle_start(s, v);
  wheel_fire<D>(s, v, sm);
}

template <int D>
__global__ void __launch_bounds__(THREADS, WCSP_MINB) k_wheel_treat(Dev s) {
  Smem& sm = smem();
  init_smem(sm);
  View v;
  load_view(s, sm, v);
  if (v.status != ST_RUNNING) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) s.ctl->ts1 = globaltimer_ns();
  if (__ldcg(&s.ctl->acc[v.c % NACC].bhit) && !s.staircase) return;
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

// ---------------------------------------------------------------------------
// One-barrier hybrid kernel (single device, dense wheel cycles).  The two-barrier kernel meets the
// whole grid after every fire and after every treat.  Here a block starts fire(c+1) as soon as the
// blocks within hyb_R of it have finished treat(c) — the only blocks whose treat reads or clears
// state words, temporary labels or bitmap words its fire writes (neighbours are at most one stride
// of the last axis away, so block distances are bounded) — and only the barrier after the fire,
// which every decision needs (a target reached, nothing live, an overflow), stays global.  The
// decision for cycle c is taken after that barrier from fire(c) and treat(c - 1); time advances by 1
// whenever fire(c) delivered anything (treat(c) may start edges with f1 = 1) and otherwise jumps to
// the next bucket the finished treats filled, and a cycle is counted only if it fired something,
// so outputs AND every work counter equal the two-barrier kernel's (tier 5's).  Sparse (listed)
// cycles treat vertices anywhere, so they end with a grid barrier as before.  Requires f1max < 64
// (the bucket of cycle c - 3 is recycled while far blocks may still be filing events of cycles c - 1, c).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void wheel_cycle_start_hyb(const Dev& s, const View& v) {
  reset_acc(&s.ctl->acc[(v.c + 1) % NACC]);
  s.ctl->ts0 = globaltimer_ns();
  unsigned long long* nf = &s.ctl->fin[(v.c + 1) & 1][0][0];
  nf[0] = 0; nf[1] = 0; nf[2] = 0; nf[3] = 0;
  if (v.c >= 3) {                  // bucket of cycle c - 3: the last decision that read its count (that
                                   // of cycle c - 2) ended before the barrier of cycle c - 1 that this
                                   // block has passed; with f1max < 64 no treat still running files into it
    const unsigned b3 = (unsigned)(__ldcg((const long long*)&s.ctl->hist_t[(v.c - 3) & (WHEEL - 1)]) & (WHEEL - 1));
    s.bnev[b3] = 0; s.bnlane[b3] = 0;
  }
  s.ctl->hist_t[v.c & (WHEEL - 1)] = v.t;
  s.ctl->hist_head[v.c & (WHEEL - 1)] = *(volatile unsigned long long*)&s.ctl->ev_head;
}

// Neighbourhood wait (warp 0, one progress word per lane, polled together): every block within
// hyb_R has published prog >= c.
// One warp polls every block within hyb_R for prog >= c; false if the watchdog fired.
__device__ __forceinline__ unsigned neigh_wait_warp(const Dev& s, unsigned long long c) {
  const unsigned lane = threadIdx.x & 31u;
  const int b = (int)blockIdx.x, G = (int)gridDim.x;
  const int lo = max(0, b - s.hyb_R), hi = min(G - 1, b + s.hyb_R);
  const unsigned long long t0 = globaltimer_ns();
  unsigned ok = 1;
  for (int j0 = lo; j0 <= hi; j0 += 32) {
    const int j = j0 + (int)lane;
    for (;;) {
      const bool done = j > hi || ld_acquire(s.prog + j) >= c;
      if (__all_sync(0xFFFFFFFFu, done)) break;
      __nanosleep(32);
      unsigned bad = 0;
      if (lane == 0) {
        if (*(volatile unsigned*)&s.ctl->abort) bad = 1;
        else if (globaltimer_ns() - t0 > BARRIER_TIMEOUT_NS) { atomicExch(&s.ctl->abort, 1u); bad = 1; }
      }
      if (__shfl_sync(0xFFFFFFFFu, bad, 0)) { ok = 0; break; }
    }
    if (!ok) break;
  }
  __threadfence();
  return ok;
}

__device__ __forceinline__ bool local_wait(const Dev& s, Smem& sm, unsigned long long c) {
  __syncthreads();
  if (threadIdx.x < 32) {
    const unsigned ok = neigh_wait_warp(s, c);
    if (threadIdx.x == 0) sm.flag = ok;
  }
  __syncthreads();
  const bool ok = sm.flag != 0;
  __syncthreads();
  return ok;
}

__device__ __forceinline__ void publish_treat(const Dev& s, unsigned long long done) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    st_release_gpu(s.prog + blockIdx.x, done);
  }
}

// The decision after fire(c) (warp 0 of every block; lane 0 of block 0 writes the totals).  Returns
// the view of cycle c + 1 or a terminal status; *lim = ring positions treat(c) may allocate below.
__device__ View decide_hyb(const Dev& s, const View& v, bool writer, unsigned long long* lim) {
  const unsigned lane = threadIdx.x & 31u;
  Ctl* C = s.ctl;
  Acc* a = &C->acc[v.c % NACC];                        // fire(c); pend at the top of cycle c-1 in ap
  Acc* ap = &C->acc[(v.c + NACC - 1) % NACC];          // treat(c - 1)
  const unsigned b = (unsigned)(v.t & (WHEEL - 1));
  const long long fired = v.c > 0 ? (long long)__ldcg(s.bnev + b) : 0;
  const long long fired_l = v.c > 0 ? (long long)__ldcg(s.bnlane + b) : 0;
  long long pl = 0, pp = 0;                            // events in flight at the top of cycle c
  if (v.c > 0) {
    const unsigned bp = (unsigned)((v.t - v.delta) & (WHEEL - 1));   // the bucket of cycle c - 1
    const long long fp = v.c > 1 ? (long long)__ldcg(s.bnev + bp) : 0;
    const long long fpl = v.c > 1 ? (long long)__ldcg(s.bnlane + bp) : 0;
    pl = __ldcg((const long long*)&ap->pend_lanes) - fpl + (long long)__ldcg(&ap->started);
    pp = __ldcg((const long long*)&ap->pend_phantoms) - (fp - fpl) + (long long)__ldcg(&ap->created);
  }
  const bool counted = v.c > 0 && (s.unit || fired > 0);
  const unsigned long long bhit = v.c > 0 ? __ldcg(&a->bhit) : 0ull;
  // ring: the oldest cycle whose events may still be live after t(c) (as wheel_propose_warp)
  const unsigned long long head = __ldcg(&C->ev_head);
  const unsigned limc = min((unsigned)WHEEL, v.c + 1u);
  unsigned B = limc;
  unsigned long long oldest = head;
  for (unsigned b0 = 0; b0 < limc; b0 += 32) {
    // each lane loads its cycle's time AND allocation head together, so the head of the oldest live
    // cycle comes from a shuffle instead of a second dependent load
    const unsigned back = b0 + lane;
    const unsigned slot = (v.c - back) & (WHEEL - 1);
    const long long ht = back < limc ? __ldcg((const long long*)&C->hist_t[slot]) : 0;
    const unsigned long long hh = back < limc ? __ldcg(&C->hist_head[slot]) : 0ull;
    const bool done = back < limc && ht + s.f1max <= v.t;
    const unsigned m = __ballot_sync(0xFFFFFFFFu, done);
    const unsigned first = m ? (unsigned)(__ffs(m) - 1) : 32u;          // in this group of 32
    const unsigned long long hsel = __shfl_sync(0xFFFFFFFFu, hh, first == 0 ? 0 : first - 1);
    if (m) {
      B = b0 + first;
      if (B > 0) oldest = first > 0 ? hsel : oldest;   // first == 0: the last lane of the previous group
      break;
    }
    oldest = __shfl_sync(0xFFFFFFFFu, hh, min(31u, limc - 1u - b0));   // whole group live: its oldest
  }
  if (B == 0) oldest = head;
  *lim = oldest + s.ev_mask + 1;
  // an overflow of treat(c - 1) or earlier (every decision input is frozen by the barrier after fire(c):
  // a treat(c) already running elsewhere may flag its own overflow, which the next decision sees)
  const bool ovf = v.c > 0 && __ldcg((const long long*)&C->ovf_t) < v.t;
  // next time: + 1 after a fire that delivered something (treat(c) may file delay-1 events) or at
  // c = 0 (the treatment of A); otherwise the next bucket the finished treats filled
  unsigned k = 1;
  if (!s.unit && v.c > 0 && fired == 0) {
    k = WHEEL;
    for (unsigned k0 = 1; k0 < (unsigned)WHEEL; k0 += 32) {
      const unsigned kk = k0 + lane;
      const bool nz = kk < (unsigned)WHEEL && __ldcg(s.bnev + ((b + kk) & (WHEEL - 1))) != 0;
      const unsigned m = __ballot_sync(0xFFFFFFFFu, nz);
      if (m) { k = k0 + (unsigned)(__ffs(m) - 1); break; }
    }
  }
  View nv = v;
  if (lane == 0) {
    if (writer) {
      // trace: the record of a counted cycle gets its fire half now and its treat half (triggered,
      // created, relabels, tested) at the next decision, which is when treat(c - 1) is complete
      if (v.pad_ && v.ncount > 0 && (long long)v.ncount - 1 < s.trace_cap) {
        TraceRec& r = s.trace[v.ncount - 1];
        r.triggered = (long long)__ldcg(&ap->triggered);
        r.created = (long long)__ldcg(&ap->created);
        r.relabels = (long long)__ldcg(&ap->relabels);
        r.tested = (long long)__ldcg(&ap->tested);
      }
      if (counted) {
        C->cycles += 1;
        C->edge_updates += pl + pp;
        if ((long long)v.ncount < s.trace_cap) {
          TraceRec r{v.t, (long long)v.delta, 0, pl, pp, 0, (long long)__ldcg(&a->arrivals), 0, 0, 0, 0, 0, 0, 0};
          s.trace[v.ncount] = r;
        }
      }
      C->arrivals += __ldcg(&a->arrivals);
      C->triggered += __ldcg(&ap->triggered); C->created += __ldcg(&ap->created);
      C->relabels += __ldcg(&ap->relabels); C->started += __ldcg(&ap->started);
      if (pl + pp > C->peak_phantoms) C->peak_phantoms = pl + pp;
      a->pend_lanes = pl;              // read as "pend at the top of cycle c" by the next decision
      a->pend_phantoms = pp;
    }
    nv.ncount = v.ncount + (counted ? 1u : 0u);
    nv.pad_ = counted ? 1u : 0u;      // "the previous cycle was counted" for the next decision
    if (bhit) {
      nv.status = 0;                   // 1°: the terminating cycle skips the treat (reading R-new-3)
      if (writer) resolve_hit(s, bhit, v.t, v.c);
    } else if (ovf) {
      nv.status = 8;
      if (writer) C->need_pool = __ldcg(&C->wheel_overflow) & 2u ? -2 : (long long)(head - oldest) + 1;
      (void)head;
    } else if (v.c > 0 && pl + pp == 0) {
      nv.status = 1;                   // 2°: nothing was in flight at the top of cycle c
    } else if (s.budget > 0 && (long long)nv.ncount >= s.budget) {
      nv.status = 4;
    } else {
      nv.delta = k;
      nv.t = v.t + k;
      nv.c = v.c + 1;
      nv.stamp = stamp_of(nv.c);
      const unsigned long long per = (unsigned long long)(__ldcg(&ap->started) + __ldcg(&ap->created)) * 2ull /
                                     ((unsigned long long)s.nblocks * (unsigned long long)max(1, s.f1max));
      unsigned r = 128;
      while (r < per && r < 4096u) r <<= 1;
      nv.region = v.c > 0 ? r : v.region;
      nv.lmode = __ldcg(&ap->triggered) <= s.list_max && v.c > 0;
    }
    if (writer) C->view = nv;
  }
  return nv;
}

template <int D, int MINB = WCSP_MINB>
__global__ void __launch_bounds__(THREADS, MINB) k_wheel_hybrid(Dev s) {
  Smem& sm = smem();
  init_smem(sm);
  View v;
  load_view(s, sm, v);
  const unsigned long long G = gridDim.x;
  unsigned long long target = 0;
  bool glob = true;                // the previous treat ended with a grid barrier (or there was none)
  long long t_list = -(1ll << 40); // time of the last listed (sparse) treat: its vertices lay anywhere,
                                   // so the events it filed fire from blocks far from their sources
                                   // until t_list + f1max — those fires need the grid barrier too
  while (v.status == ST_RUNNING) {
    if (v.c > 0) {
      if (!glob) {
        // the fire's own-data prologue first (descriptor count and staging, bitmap zeroing): its
        // dependent loads overlap the wait for the neighbourhood to finish treat(c - 1)
        if (s.hyb_prep) {
          if (MINB < 4 && v.lmode) fire_prologue<D, false, FIRE_ITEMS>(s, v, sm);
          else fire_prologue<D, false, fire_items<MINB>()>(s, v, sm);
        }
        if (!local_wait(s, sm, v.c)) return;
      }
      if (blockIdx.x == 0 && threadIdx.x == 0) wheel_cycle_start_hyb(s, v);
      if (threadIdx.x == 0) sm.tphase = globaltimer_ns();
      if (MINB < 4 && v.lmode) wheel_fire<D, false, FIRE_ITEMS>(s, v, sm);
      else wheel_fire<D, false, fire_items<MINB>()>(s, v, sm);
      target += G;
      if (!grid_sync(s.ctl, target, sm, s.trace_cap > 0 ? &s.ctl->fin[v.c & 1][0][0] : nullptr)) return;
    }
    if (threadIdx.x < 32) {
      unsigned long long lim = 0;
      const View nv = decide_hyb(s, v, blockIdx.x == 0, &lim);
      if (threadIdx.x == 0) { sm.view = nv; sm.alloc_lim = lim; }
    }
    __syncthreads();
    const View nv = sm.view;
    __syncthreads();
    if (nv.status != ST_RUNNING) break;
    if (threadIdx.x == 0) sm.tphase = globaltimer_ns();
    phase_treat<D, true>(s, v, sm);                     // treat(c) with cycle c's view
    if (v.lmode) t_list = v.t;
    if (v.lmode || needs_maint(v, nv) || nv.t <= t_list + s.f1max) {   // listed vertices / their events / maint
      target += G;
      if (!grid_sync(s.ctl, target, sm)) return;
      if (needs_maint(v, nv)) {
        wheel_maintain(s, nv.t);
        target += G;
        if (!grid_sync(s.ctl, target, sm)) return;
      }
      glob = true;
    } else {
      publish_treat(s, (unsigned long long)v.c + 1);
      glob = false;
    }
    v = nv;
  }
}

// ---------------------------------------------------------------------------
// Lagged-decision wheel kernel (single device, dense wheel cycles; the default where the hybrid
// applies).  The hybrid kernel still meets the whole grid after every fire, because the decision
// for cycle c (a target reached, nothing in flight, an overflow, the budget) needs the complete
// fire(c).  Here no cycle waits for its own decision:
//   * time steps by one every cycle (t(c) = c; a cycle whose bucket is empty fires nothing and is
//     not counted, so outputs and counters are those of the jumping wheel, i.e. tier 5's);
//   * treat(c) waits only for the fire(c) of the blocks within hyb_R, fire(c + 1) only for their
//     treat(c) (progress words: 2c + 1 = fire(c) done, 2c + 2 = treat(c) done);
//   * decision x is taken by every block (identically, in order) once every block has counted
//     its fire(x) in slot x (nfire == G), after the block's treat(x + 1) and before its fire(x + 2):
//     the decision's loads overlap the wait for the neighbours' treats, and no block waits for the
//     slowest block's fire of its own cycle;
//   * cycles that need the whole grid's fire(c) before treat(c) (sparse cycles, whose treat walks
//     the global list, and the f1max time units after one, whose fires write far from their
//     slabs) take decision c before treat(c), as the hybrid does.
// A terminating decision x is seen after fire(x + 1) and treat(x + 1) ran: they are discarded
// (their counters sit in slot x + 1, which no decision reads; they write no target list of cycle
// x; an overflow they flag carries a later time).  Blocks are at most two cycles apart (fire(c + 2)
// anywhere needs decision c, which needs every fire(c)); hence NACC >= 7, the reset of slot c + 2
// and of the bucket of cycle c - 5 at block 0's fire(c), and the ring head recorded there for
// cycle c + 2 (a treat(c + 1) may already be allocating elsewhere).
// ---------------------------------------------------------------------------
static_assert(NACC >= 7, "k_wheel_lag: slots of cycles up to two apart plus their readers");

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void wheel_cycle_start_lag(const Dev& s, const View& v) {
  reset_acc(&s.ctl->acc[(v.c + 2) % NACC]);
  if (v.c >= 5) {                  // last read by decision c - 4, which every block has taken
    const unsigned b5 = (v.c - 5) & (WHEEL - 1);
    s.bnev[b5] = 0; s.bnlane[b5] = 0;
  }
  s.ctl->hist_t[v.c & (WHEEL - 1)] = v.t;
  // every event allocated before this point comes from a treat of cycle <= c + 1 (treat(c + 2)
  // anywhere follows that block's fire(c + 2), which needs decision c, i.e. this block's fire(c))
  s.ctl->hist_head[(v.c + 2) & (WHEEL - 1)] = *(volatile unsigned long long*)&s.ctl->ev_head;
}

// Decision of cycle x = L.dn (warp 0; lane 0 updates L; lane 0 of block 0 writes the totals).
// Inputs: fire(x) (slot x), treat(x - 1) (slot x - 1) and the bucket counts of cycles x, x - 1 —
// all final once every block has counted fire(x).
__device__ void decide_lag(const Dev& s, LagState& L, bool writer) {
  const unsigned lane = threadIdx.x & 31u;
  Ctl* C = s.ctl;
  const unsigned x = L.dn;
  const long long t = (long long)x;
  Acc* a = &C->acc[x % NACC];
  Acc* ap = &C->acc[(x + NACC - 1) % NACC];
  if (lane == 0) {
    const unsigned b = (unsigned)(t & (WHEEL - 1)), bp = (unsigned)((t - 1) & (WHEEL - 1));
    const long long fired = x > 0 ? (long long)__ldcg(s.bnev + b) : 0;
    const long long fp = x > 1 ? (long long)__ldcg(s.bnev + bp) : 0;
    const long long fpl = x > 1 ? (long long)__ldcg(s.bnlane + bp) : 0;
    const unsigned long long bhit = x > 0 ? __ldcg(&a->bhit) : 0ull;
    const unsigned long long started = __ldcg(&ap->started), created = __ldcg(&ap->created);
    const unsigned long long triggered = __ldcg(&ap->triggered);
    const long long ovft = __ldcg((const long long*)&C->ovf_t);
    long long pl = 0, pp = 0;                         // events in flight at the top of cycle x
    if (x > 0) {
      pl = L.pl - fpl + (long long)started;
      pp = L.pp - (fp - fpl) + (long long)created;
    }
    const bool counted = x > 0 && (s.unit || fired > 0);
    if (writer) {
      if (counted) { C->cycles += 1; C->edge_updates += pl + pp; }
      C->arrivals += __ldcg(&a->arrivals);
      C->triggered += triggered; C->created += created;
      C->relabels += __ldcg(&ap->relabels); C->started += started;
      if (pl + pp > C->peak_phantoms) C->peak_phantoms = pl + pp;
    }
    L.pl = pl; L.pp = pp;
    L.ncount += counted ? 1u : 0u;
    L.pad_ = counted ? 1u : 0u;
    int st = ST_RUNNING;
    if (bhit) {
      st = 0;                                         // the target reached (reading R-new-3)
      if (writer) resolve_hit(s, bhit, t, x);
    } else if (x > 0 && ovft < t) {
      st = 8;                                         // an overflow of treat(x - 1) or earlier
      if (writer) {
        // live events: those of cycles after cd = x - f1max (the newest whose events all fired);
        // hist_head[cd + 1] precedes every allocation of a treat after cd
        const long long cd = (long long)x - s.f1max;
        const unsigned long long oldest = cd >= 0 ? __ldcg(&C->hist_head[(cd + 1) & (WHEEL - 1)]) : 0ull;
        C->need_pool = __ldcg(&C->wheel_overflow) & 2u ? -2 : (long long)(__ldcg(&C->ev_head) - oldest) + 1;
      }
    } else if (x > 0 && pl + pp == 0) {
      st = 1;                                         // nothing was in flight at the top of cycle x
    } else if (s.budget > 0 && (long long)L.ncount >= s.budget) {
      st = 4;
    } else {
      const unsigned long long per = (started + created) * 2ull /
                                     ((unsigned long long)s.nblocks * (unsigned long long)max(1, s.f1max));
      unsigned r = 128;
      while (r < per && r < 4096u) r <<= 1;
      if (x > 0) L.region = r;
      L.lmode = triggered <= s.list_max && x > 0;
    }
    L.status = st;
    if (writer && st != ST_RUNNING) {
      View nv{};
      nv.t = t; nv.c = x; nv.stamp = stamp_of(x); nv.delta = 1; nv.status = st;
      nv.region = L.region; nv.lmode = L.lmode; nv.ncount = L.ncount; nv.pad_ = L.pad_;
      C->view = nv;
    }
    L.dn = x + 1;
  }
  __syncwarp();
}

// Take the decisions up to cycle `upto` (warp 0 waits for each cycle's fire count) and, if
// wait_c > 0, wait for the neighbourhood's prog >= wait_c at the same time (warp 1).  False: abort.
// nowait: take only the decisions whose fire counts are already complete (no polling; the rest
// are taken by a later call).
__device__ bool decide_upto(const Dev& s, Smem& sm, unsigned upto, unsigned long long wait_c = 0,
                            bool nowait = false) {
  if (wait_c > 0 && threadIdx.x >= 32 && threadIdx.x < 64) {
    const unsigned ok = neigh_wait_warp(s, wait_c);
    if (threadIdx.x == 32) sm.flag2 = ok;
  }
  if (threadIdx.x < 32) {
    const unsigned lane = threadIdx.x;
    const unsigned G = gridDim.x;
    unsigned ok = 1;
    for (;;) {
      __syncwarp();
      const unsigned x = sm.lag.dn;
      if (x > upto || sm.lag.status != ST_RUNNING) break;
      if (x > 0 && nowait && !__all_sync(0xFFFFFFFFu, ld_acquire_u32(&s.ctl->acc[x % NACC].nfire) >= G)) break;
      if (x > 0) {
        const unsigned long long t0 = globaltimer_ns();
        while (!__all_sync(0xFFFFFFFFu, ld_acquire_u32(&s.ctl->acc[x % NACC].nfire) >= G)) {
          __nanosleep(32);
          unsigned bad = 0;
          if (lane == 0) {
            if (*(volatile unsigned*)&s.ctl->abort) bad = 1;
            else if (globaltimer_ns() - t0 > BARRIER_TIMEOUT_NS) { atomicExch(&s.ctl->abort, 1u); bad = 1; }
          }
          if (__shfl_sync(0xFFFFFFFFu, bad, 0)) { ok = 0; break; }
        }
        if (!ok) break;
      }
      decide_lag(s, sm.lag, blockIdx.x == 0);
    }
    if (lane == 0) sm.flag = ok;
  }
  __syncthreads();
  const bool ok = sm.flag != 0 && (wait_c == 0 || sm.flag2 != 0);
  __syncthreads();
  return ok;
}

template <int D, int MINB = WCSP_MINB>
__global__ void __launch_bounds__(THREADS, MINB) k_wheel_lag(Dev s) {
  Smem& sm = smem();
  init_smem(sm);
  View v;
  load_view(s, sm, v);             // c = 0, t = 0: the treatment of A
  if (threadIdx.x == 0) {
    LagState& L = sm.lag;
    L.pl = 0; L.pp = 0; L.dn = v.c; L.ncount = v.ncount; L.pad_ = v.pad_;
    L.region = v.region; L.lmode = v.lmode; L.status = ST_RUNNING;
  }
  __syncthreads();
  const unsigned long long G = gridDim.x;
  unsigned long long target = 0;   // grid_sync counter (after sparse treats, maintenance)
  bool glob = true;                // the previous treat ended with a grid barrier (or there was none)
  long long t_list = -(1ll << 40); // time of the last listed (sparse) treat (see k_wheel_hybrid)
  for (;;) {
    const unsigned c = v.c;
    const bool sync = v.lmode || v.t <= t_list + s.f1max;   // treat(c) needs the whole grid's fire(c)
    if (c > 0) {
      if (!glob) {
        if (s.hyb_prep) {          // own-data prologue first: its loads overlap the neighbourhood wait
          if (MINB < 4 && v.lmode) fire_prologue<D, false, FIRE_ITEMS>(s, v, sm);
          else fire_prologue<D, false, fire_items<MINB>()>(s, v, sm);
        }
        if (!local_wait(s, sm, 2ull * c)) return;
      }
      if (blockIdx.x == 0 && threadIdx.x == 0) wheel_cycle_start_lag(s, v);
      if (MINB < 4 && v.lmode) wheel_fire<D, false, FIRE_ITEMS>(s, v, sm);
      else wheel_fire<D, false, fire_items<MINB>()>(s, v, sm);
      __syncthreads();
      if (threadIdx.x == 0) {      // count fire(c) in its slot, publish it to the neighbourhood
        __threadfence();
        atomicAdd(&s.ctl->acc[c % NACC].nfire, 1u);
        st_release_gpu(s.prog + blockIdx.x, 2ull * c + 1);
      }
    }
    // async cycle: treat(c) after the neighbourhood's fire(c), then decision c - 1 (its latency
    // overlaps the neighbours' treats); a treat that needs the whole fire(c) (and c = 0) takes the
    // decisions up to c first
    const bool early = c == 0 || sync;
    if (early) {
      if (!decide_upto(s, sm, c)) return;
      if (sm.lag.status != ST_RUNNING) break;
    } else if (s.lag_pre) {        // decision c - 1 (warp 0) beside the wait for the neighbours' fire(c)
      if (!decide_upto(s, sm, c - 1, s.lag_par ? 2ull * c + 1 : 0ull, s.lag_pre == 2)) return;
      if (sm.lag.status != ST_RUNNING) break;
      if (!s.lag_par && !local_wait(s, sm, 2ull * c + 1)) return;
    } else if (!local_wait(s, sm, 2ull * c + 1)) return;
    if (threadIdx.x == 0) {
      // ring: every block has fired cycles <= c - 2, so events of cycles cd <= c - 2 - f1max are
      // dead; hist_head[cd + 1] precedes every allocation of a later treat
      const long long cd = (long long)c - 2 - s.f1max;
      const unsigned long long oldest = cd >= 0 ? __ldcg(&s.ctl->hist_head[(cd + 1) & (WHEEL - 1)]) : 0ull;
      sm.alloc_lim = oldest + s.ev_mask + 1;
    }
    __syncthreads();
    phase_treat<D, true>(s, v, sm);                     // treat(c) with cycle c's view
    publish_treat(s, 2ull * c + 2);
    if (!early && s.lag_pre != 1) {  // (lag_pre 2: only what the try before treat(c) left)
      if (!decide_upto(s, sm, c - 1)) return;
      if (sm.lag.status != ST_RUNNING) break;
    }
    if (v.lmode) t_list = v.t;
    View nv = v;
    nv.c = c + 1; nv.t = v.t + 1; nv.delta = 1; nv.stamp = stamp_of(c + 1);
    nv.region = sm.lag.region; nv.lmode = sm.lag.lmode;
    const bool maint = nv.stamp == 1u || (nv.t / MAINT_PERIOD_T) != (v.t / MAINT_PERIOD_T);
    if (v.lmode || maint || nv.t <= t_list + s.f1max) {  // listed vertices / their events / maint
      target += G;
      if (!grid_sync(s.ctl, target, sm)) return;
      if (maint) {
        wheel_maintain(s, nv.t);
        target += G;
        if (!grid_sync(s.ctl, target, sm)) return;
      }
      glob = true;
    } else {
      glob = false;                // treat(c) is published: fire(c + 1) waits for the neighbourhood
    }
    v = nv;
  }
}

// ---------------------------------------------------------------------------
// Peer halo: every slab runs the persistent wheel cycle in
// ONE cooperative kernel per device, and the halo is fused into it — water
// that crosses a slab boundary is a system-scope atomicMax straight into the
// neighbour's state word (plus its bitmap bit), and the Step-4 neighbour test
// reads the neighbour's current label in its own memory.  No ghost copies, no
// host round trip, no stale labels: outputs AND work counters equal the
// single-device run.  Across GPUs the neighbour's arrays are NVLink peer
// memory (CUDA IPC); on one device (virtual slabs) they are the other slabs'
// allocations and the slabs are groups of blocks of the same launch.
//
// Barrier: the blocks of a slab meet on its control block (ctl->bar); the
// slab's leader block then meets the other leaders on the cross-slab counter
// (system scope) and releases its slab with ctl->rel = epoch.
// ---------------------------------------------------------------------------
constexpr int MAX_VSLABS = 8;
struct DevSet { Dev d[MAX_VSLABS]; unsigned per; int n; };

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_add_release_sys(unsigned long long* p, unsigned long long x) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(x) : "memory");
}

// propose: the leader, once every block of its slab has arrived (the slab's treat is
// complete), writes the slab's proposal for the cycle decision before joining the other
// slabs, so one barrier both ends the treat and publishes the proposals.
__device__ __forceinline__ bool peer_sync(const Dev& s, Smem& sm, unsigned long long epoch,
                                          unsigned long long* fin = nullptr, const View* propose = nullptr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (fin) {
      const unsigned long long busy = globaltimer_ns() - sm.tphase;
      atomicMax(fin, busy);
      atomicAdd(fin + 1, busy);
    }
    __threadfence_system();        // this block's writes, remote atomics included, before arriving
    atomicAdd(&s.ctl->bar, 1ull);
    const unsigned long long t0 = globaltimer_ns();
    unsigned ok = 1;
    auto timed_out = [&]() {
      if (*(volatile unsigned*)&s.ctl->abort || *(volatile unsigned*)s.xabort) return true;
      if (globaltimer_ns() - t0 > BARRIER_TIMEOUT_NS) {
        atomicExch(&s.ctl->abort, 1u);
        atomicExch(s.xabort, 1u);
        return true;
      }
      return false;
    };
    if (blockIdx.x == s.blk0) {    // leader: all blocks of the slab, then all slabs
      while (ld_acquire(&s.ctl->bar) < epoch * s.nblocks) {
        __nanosleep(32);
        if (timed_out()) { ok = 0; break; }
      }
      if (ok) {
        if (propose) {
          long long need = 0;
          s.ctl->prop = wheel_propose(s, *propose, &need);
          s.ctl->prop_need = need;     // read back by this same thread in the decision
        }
        __threadfence_system();
        red_add_release_sys(s.xbar, 1ull);
        while (ld_acquire_sys(s.xbar) < epoch * (unsigned long long)s.nslab) {
          __nanosleep(64);
          if (timed_out()) { ok = 0; break; }
        }
      }
      if (ok) st_release_gpu(&s.ctl->rel, epoch);
    } else {
      while (ld_acquire(&s.ctl->rel) < epoch) {
        __nanosleep(32);
        if (timed_out()) { ok = 0; break; }
      }
    }
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    sm.flag = ok;
  }
  __syncthreads();
  const bool ok = sm.flag != 0;
  __syncthreads();
  return ok;
}

template <int D, int MINB = WCSP_MINB>   // MINB: as k_wheel_persistent
__global__ void __launch_bounds__(THREADS, MINB) k_wheel_peer(const __grid_constant__ DevSet set) {
  const Dev& s = set.d[blockIdx.x / set.per];
  Smem& sm = smem();
  init_smem(sm);
  View v;
  load_view(s, sm, v);
  const bool leader = blockIdx.x == s.blk0;
  unsigned long long epoch = 0;
  while (v.status == ST_RUNNING) {
    if (v.c > 0) {
      if (leader && threadIdx.x == 0) wheel_cycle_start(s, v);
      if (threadIdx.x == 0) sm.tphase = globaltimer_ns();
      wheel_fire<D, true>(s, v, sm);
      if (!peer_sync(s, sm, ++epoch, s.trace_cap > 0 ? &s.ctl->fin[v.c & 1][0][0] : nullptr)) return;
    }
    if (leader && threadIdx.x == 0) s.ctl->ts1 = globaltimer_ns();
    if (threadIdx.x == 0) {          // a target reached in any slab ends the run (1°)
      unsigned long long bh = 0;
      for (int i = 0; i < s.nslab; ++i) bh = max(bh, __ldcv(&s.pctl[i]->acc[v.c % NACC].bhit));
      sm.bhit = bh;
    }
    __syncthreads();
    const unsigned long long bhit = sm.bhit;
    __syncthreads();
    if (!bhit) {
      if (threadIdx.x == 0) sm.tphase = globaltimer_ns();
      phase_treat<D, true, true>(s, v, sm);
    }
    // end of the treat + every slab's proposal for the decision, in one barrier
    if (!peer_sync(s, sm, ++epoch, bhit || s.trace_cap <= 0 ? nullptr : &s.ctl->fin[v.c & 1][1][0], &v)) return;
    const View prev = v;
    if (threadIdx.x == 0) {          // every slab takes the same decision from the combined proposal
      Prop G{0, -(long long)WHEEL, 0, 0};
      for (int i = 0; i < s.nslab; ++i) {
        const volatile Prop* p = &s.pctl[i]->prop;
        G.bhit = max(G.bhit, (long long)p->bhit); G.negk = max(G.negk, (long long)p->negk);
        G.pending = max(G.pending, (long long)p->pending); G.overflow = max(G.overflow, (long long)p->overflow);
      }
      View nv = v;
      // the slab's own proposal was computed by its leader in peer_sync (only the writer needs its
      // ring need); the decision itself uses the combined G, so nobody re-runs wheel_propose here
      wheel_decide(s, nv, leader, &G, &G, leader ? s.ctl->prop_need : 0);
      sm.view = nv;
    }
    __syncthreads();
    v = sm.view;
    __syncthreads();
    if (needs_maint(prev, v)) {
      wheel_maintain(s, v.t);
      if (!peer_sync(s, sm, ++epoch)) return;
    }
  }
}

}  // namespace wcspk
