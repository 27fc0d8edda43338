// wcsp_device.cuh — device state, phase functions and kernels of the B200
// (sm_100a) active-vertex label-correcting sweep (§4, :155-227).
//
// One cycle, c = 1, 2, ...:
//   sweep  : Step 1 and Step 3 (:173) — every live lane of every
//            active vertex and every live phantom counts down by Delta; the ones
//            reaching 0 deliver water (cand = label - f2) to their destination
//            D with one 32-bit atomicMax on D's temporary label (Step 2,
//            :166-168; the "temporary replacement label" of :133).  The
//            first arrival of the cycle sets D's bit in the triggered bitmap
//            (the dedupe of :164).  Survivors are compacted into the next
//            active list / phantom pool (Steps 7-9, :207-227), block-aggregated.
//   treat  : Steps 4, 5 and 8.1 (:176-198, :211) for every triggered Q, taken
//            from the bitmap in vertex order, whose temporary label beats its
//            label (:32): an edge Q->R is triggered iff L* - f2 >
//            max(L(R), temp(R)) (:180); if Q has no live lane (inactive,
//            :189) the lane restarts with f1 (:190-192) and L(Q) := L*;
//            otherwise a phantom (Q, R, L*, f1) is created (:197-198).
//            L* = temp(Q) (reading R23).
//   decide : Step 6 (:204) — termination 1° (:124) / 2° (:126); Delta for the
//            next cycle = min live residual (time skipping, :75, :95).
// c = 0 is the initial state: A is triggered with temp M
// and treated (reading R20).  The timing-wheel engine (wcsp_wheel.cuh) runs
// the same treat with events instead of residual countdowns.
//
// Vertex state word sw[v] (u64): low u32 = label L(v) (bits 0-15; bits 16-31
// hold the wheel engine's lane-expiry time), high u32 = temp = stamp:16 |
// cand:16, valid only when stamp == this cycle's.  Targets (B) and removed
// vertices carry a temp sentinel with stamp 0xFFFF that an atomicMax never
// overwrites, so an arrival learns what D is from the atomic's return value.
#pragma once
#include <cstdint>
#include <cstdio>
#include <type_traits>
#include <cuda_runtime.h>

namespace wcspk {

constexpr int THREADS = 256;
constexpr int WARPS = THREADS / 32;
constexpr int SWEEP_ITEMS = 4;           // items per thread per chunk, sweep (unrolled for MLP)
constexpr int CHUNK_MAX = THREADS * SWEEP_ITEMS;
#ifndef WCSP_MINB_SWEEP
#define WCSP_MINB_SWEEP 4          // resident blocks per SM the sweep engine's kernels are compiled for
#endif
#ifndef WCSP_BAR_GROUPS
#define WCSP_BAR_GROUPS 1          // > 1: two-level grid-barrier arrivals (per-group counters)
#endif
#ifndef WCSP_QP_CAP
#define WCSP_QP_CAP 3072
#endif
constexpr int QP_CAP = WCSP_QP_CAP;             // shared staging of phantoms / events (overflow -> direct append)
constexpr int QA_CAP = 2048;             // shared staging of active-list appends (never overflows)
#ifndef WCSP_WIN_MAX
#define WCSP_WIN_MAX 16
#endif
constexpr int WIN_WORDS = WCSP_WIN_MAX;  // max triggered-bitmap words per warp window (Dev.win_words: 8 or 16)
// Frontier-granularity experiment (SURVEY §8(a) "frontier granularity", build option): stage each
// treat round's band of vertex state words — the round's 32 * WARPS * ww vertices plus one stride of
// axis 1 on either side — into shared memory with one TMA bulk copy (cp.async.bulk + mbarrier), so
// Q's own word and its +-x / +-y neighbour tests read shared memory; +-z stays global.
// Checked build (-DWCSP_CHECKS=1, tests only): device-side bounds checks on every vertex index the
// fire, treat and sweep derive from a list, bitmap or event record, and a poisoned event ring, so a
// stale or torn read traps (compute-sanitizer is closed on this pool).
#ifndef WCSP_CHECKS
#define WCSP_CHECKS 0
#endif
#if WCSP_CHECKS
#define WCSP_CHECK(cond, what, a, b)                                                              \
  do {                                                                                           \
    if (!(cond)) {                                                                               \
      printf("WCSP_CHECK failed: %s (%llu, %llu) block %d thread %d\n", what, (unsigned long long)(a), \
             (unsigned long long)(b), (int)blockIdx.x, (int)threadIdx.x);                        \
      __trap();                                                                                  \
    }                                                                                            \
  } while (0)
#else
#define WCSP_CHECK(cond, what, a, b) do { } while (0)
#endif
constexpr unsigned long long EV_POISON = 0x7FFFFFFFFFFFFFFFull;   // src 0x3FFFFFFF: out of range

#ifndef WCSP_TREAT_STAGE
#define WCSP_TREAT_STAGE 0
#endif
#ifndef WCSP_STAGE_WORDS
#define WCSP_STAGE_WORDS 4096
#endif
constexpr int WIN_VERTS = WIN_WORDS * 32;

constexpr unsigned LBL_REMOVED = 0xFFFFu;  // label of a vertex outside G': no S6 test passes
constexpr unsigned TMP_B = 0xFFFF0001u;    // temp sentinel of a target vertex
constexpr unsigned TMP_REMOVED = 0xFFFF0000u;
constexpr unsigned TMP_GHOST = 0xFFFF0002u;    // slab engine: a neighbouring slab's boundary vertex
constexpr unsigned TMP_GHOST_B = 0xFFFF0003u;  // ... that is a target
// Wide labels (budgets M > WCSP_M_MAX, include/wcsp.h; sweep engine only): label L(v) is a u32 in
// Dev::lab, the state word sw[v] holds only temp = stamp:32 | cand:32 (64-bit atomicMax); sentinel
// stamp 0xFFFFFFFF as in the 16-bit layout.  Phantom records are 16 bytes (see PhW).
constexpr unsigned LBL_REMOVED_W = 0x7FFFFFFFu;   // > any cand (M <= 2^31 - 2): no S6 test passes
constexpr unsigned long long TMPW_SENT = 0xFFFFFFFFull << 32;
constexpr unsigned long long TMPW_REMOVED = TMPW_SENT | 0ull;
constexpr unsigned long long TMPW_B = TMPW_SENT | 1ull;
struct __align__(16) PhW { unsigned long long x, y; };   // x: src 30 | lane 3 | res 8 (bit 33); y: cand
constexpr int PHW_RES = 33;
constexpr int ST_RUNNING = -1;
constexpr int ST_WRAP = 100;               // stepped engines: maintenance pass needed (host launches it)

// phantom record (u64): src 30 | lane 3 | cand 16 | res 8  (cand = L* - f2(e), fixed at creation)
constexpr int PH_LANE = 30, PH_CAND = 33, PH_RES = 49;
constexpr unsigned STAMP_PERIOD = 65534u;  // stamps 1..0xFFFE; 0xFFFF is the sentinel
constexpr int WHEEL = 256;                 // timing wheel buckets (f1 <= 255)

struct BArr { unsigned D, cand, src, via; };   // an arrival at a target (terminating cycle only)

// Per-cycle accumulators live in NACC slots (slot c % NACC).  The two-barrier kernels need three
// (the next cycle's slot is reset while this one is read); the one-barrier hybrid kernel reads a
// cycle's fire half and the previous cycle's treat half in the same decision, so it needs four;
// the lagged-decision kernel (blocks up to two cycles apart) needs seven (k_wheel_lag).
constexpr int NACC = 8;
struct Acc {                       // per-cycle accumulators, slot c % NACC
  unsigned n_act;                  // entries appended to the next active list
  unsigned n_pool;                 // phantoms appended to the next pool (may exceed capacity)
  unsigned tl_over;                // wheel: first arrivals beyond some block's list went to the bitmap
  unsigned tl_total;               // wheel, sparse cycles: vertices in the cycle's global triggered list
  unsigned dmin;                   // min live residual after this cycle (0xFFFFFFFF = nothing live)
  unsigned long long bhit;         // max over B arrivals of (cand << 32 | ~X)
  unsigned long long live;         // sweep: live lanes at the top of the cycle (E); wheel: lanes started
  unsigned long long arrivals, created, relabels, triggered, started, tested;
  long long pend_lanes, pend_phantoms;   // timing wheel: events in flight at the top of this cycle
  unsigned nfire, pad_;            // lagged-decision kernel: blocks that finished this cycle's fire
};

// A slab's proposal for the decision of one cycle; the slabs' proposals are
// combined with an element-wise max (NCCL allreduce max, or a kernel for
// virtual slabs): bhit = best target arrival, negk = -(steps to the next
// non-empty wheel bucket), pending = any live edge, overflow = any storage overflow.
struct Prop { long long bhit, negk, pending, overflow; };

struct View {                      // cycle state every block needs
  long long t;
  unsigned c, stamp, delta, n_act, n_pool;
  int cur, status;
  unsigned region;                 // timing wheel: ring region size per (block, delay)
  unsigned lmode;                  // timing wheel: sparse cycle, fire lists the vertices it triggers
  unsigned ncount;                 // hybrid kernel: counted (non-empty) cycles so far
  unsigned pad_;                   // hybrid kernel: the previous cycle was counted
};

struct Ctl {
  View view;
  Acc acc[NACC];                   // per-cycle accumulators, slot c % NACC
  unsigned long long bar;          // grid barrier arrivals (persistent engines)
  unsigned long long rel;          // peer halo: epoch released by this slab's leader block
  unsigned abort, pad1_;           // barrier watchdog fired
  unsigned n_barr2[2];             // B-arrival list length per cycle parity (list c & 1 at barr[(c & 1) * barr_cap])
  long long F1, F2, X, Y;
  long long via;
  long long cycles, edge_updates, arrivals, triggered, created, relabels, started;
  long long peak_active, peak_phantoms, need_pool;
  unsigned long long ts0, ts1, ts2;   // globaltimer at cycle start / after arrivals / after treat (block 0)
  unsigned long long fin[2][2][2];    // [cycle & 1][phase][max, sum] block busy times (persistent engines)
  // timing-wheel engine (wcsp_wheel.cuh)
  unsigned long long ev_head;      // logical allocation head of the event ring
  unsigned wheel_overflow, pad2_;  // 2: descriptor table full, 4: ring guard (hybrid)
  long long ovf_t;                 // earliest treat time that flagged an overflow (LLONG_MAX: none)
  long long hist_t[WHEEL];         // time of cycle c (slot c & 255) ...
  unsigned long long hist_head[WHEEL];   // ... and the ring head before its treat
  Prop prop, gprop;                // slab engine: local proposal / reduced proposal
  unsigned long long ybest;        // (src << 1 | via) of the best arrival at X seen by this slab
  unsigned n_stair, pad3_;         // staircase steps recorded
  long long stair_q;               // best target quality so far
  long long prop_need;             // peer halo: ring slots the leader's proposal asked for (with prop)
  unsigned long long n_appended;   // wheel treat: events past the shared staging appended to open regions
  unsigned long long n_spilled;    // ... past those, written to the block's spill buffer
  unsigned long long n_single;     // ... past the spill buffer, filed as runs of one
  alignas(128) unsigned long long grel;   // grid barrier: the last block to arrive releases this target
  unsigned long long pad4_[15];           // (its own 128-byte line: pollers do not slow the arrivals)
  alignas(128) unsigned long long bsub[WCSP_BAR_GROUPS][16];   // WCSP_BAR_GROUPS > 1: per-group arrivals
};

struct TraceRec {
  long long t, delta, active_vertices, live_lanes, phantoms, triggered, arrivals, created, relabels;
  long long tested, ns_arrive, ns_treat;   // bitmap entries examined; phase times seen by block 0
  long long ns_arrive_spread, ns_treat_spread;   // max block busy time minus the mean (load imbalance)
};

struct Dev {
  unsigned N;
  int NL;                          // lanes per vertex = 2d
  unsigned off[8];                 // lane 2k: +stride_k, lane 2k+1: -stride_k (mod 2^32)
  const void* wt;                  // weight records (f1 lane word, f2 lane word) per vertex
  void* res;                       // sweep engine: lane residual words, 0 = idle lane
  unsigned long long* sw;          // vertex state words (label | temp); wide: temp only
  unsigned* lab;                   // wide labels (M > WCSP_M_MAX): L(v) as u32
  int wide;
  unsigned* tbits;                 // triggered bitmap (first arrivals of the cycle)
  unsigned nwords;                 // words of the bitmap
  unsigned win_words;              // bitmap words per warp window of the treat (8 or 16)
  unsigned ileave;                 // treat rounds interleaved across blocks (chunk-at-a-time; see phase_treat)
  unsigned fstride;                // fire: warps take run chunks in turn (list order), see wheel_fire
  unsigned wbal;                   // treat: balanced window slabs per block (block_windows)
  unsigned* act[2];
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
  unsigned long long* spill;       // [nblocks][spill_cap] events past a block's staging, per flush period
  unsigned* tlist;                 // [nblocks * QA_CAP] wheel, sparse cycles: the vertices the fire triggered
                                   // (first arrivals), appended block by block (acc->tl_total)
  unsigned long long list_max;     // a cycle is sparse (listed) if the previous one triggered at most this many
  unsigned spill_cap;
  unsigned nblocks;                // grid size of the cycle kernels (wheel region sizing)
  // one-barrier hybrid kernel (k_wheel_hybrid): per-block treat progress and the block radius
  // within which blocks' fires and treats touch the same state words
  unsigned long long* prog;        // [nblocks] treats completed (monotone per solve)
  int hyb_R;
  int hyb_prep;                    // run the fire's own-data prologue before the neighbourhood wait
  int lag_pre;                     // k_wheel_lag: decision c - 1 before treat(c) (1), after (0), before if ready (2)
  int lag_par;                     // k_wheel_lag: that decision (warp 0) and the neighbourhood wait (warp 1) together
  // slab partition (multi-GPU / virtual slabs): local index + goff = global index
  unsigned goff;
  unsigned plane;                  // vertices per plane of the partitioned (last) axis
  unsigned ghost_hi_start;         // local index of the upper ghost plane (N if none)
  unsigned long long* ghost_out_lo;   // water handed to the lower neighbour's boundary plane
  unsigned long long* ghost_out_hi;   // ... to the upper neighbour's
  int slab;                        // 1: decide uses the reduced global proposal (ctl->gprop)
  unsigned blk0;                   // first block of this slab in the launch (peer halo: slab * nblocks)
  // peer halo: a ghost index resolves to the neighbouring slab's own memory
  // (the same device for virtual slabs, NVLink peer memory mapped with CUDA IPC across GPUs)
  int peer;
  unsigned plo_end;                // local indices < plo_end are the lower ghost plane
  unsigned long long* psw[2];      // lower / upper neighbour's state words
  unsigned* ptb[2];                // lower / upper neighbour's triggered bitmaps
  unsigned pshift[2];              // ghost index + pshift = the neighbour's local index (mod 2^32)
  unsigned pgoff[2];               // the neighbour's global offset
  Ctl* const* pctl;                // every slab's control block (proposals, target hits)
  int nslab, islab;
  unsigned long long* xbar;        // cross-slab barrier arrivals (monotone)
  unsigned* xabort;                // cross-slab watchdog flag
  // staircase mode (wcsp_staircase): record every strictly better target arrival, keep going
  int staircase;
  long long f2stop;
  long long* stair;                // [stair_cap][4] (F1, F2, X, Y)
  unsigned stair_cap;
};

template <int D> struct Tr;
template <> struct Tr<1> { using LW = uint32_t; };
template <> struct Tr<2> { using LW = uint32_t; };
template <> struct Tr<3> { using LW = unsigned long long; };
template <> struct Tr<4> { using LW = unsigned long long; };

__host__ __device__ constexpr unsigned stamp_of(unsigned c) { return (c % STAMP_PERIOD) + 1u; }

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// L2 residency control (createpolicy + .L2::cache_hint): the vertex state
// words are the hot, reused set (evict-last); events and weight records
// stream through (evict-first).  WCSP_L2_HINTS=0 at build time disables it.
#ifndef WCSP_L2_HINTS
#define WCSP_L2_HINTS 1
#endif
#ifndef WCSP_POL_PURE
#define WCSP_POL_PURE 1            // createpolicy as a pure asm (one per kernel after CSE, not one per access)
#endif
__device__ __forceinline__ unsigned long long pol_first() {
  unsigned long long p = 0;
#if WCSP_L2_HINTS
#if WCSP_POL_PURE
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));   // pure: CSE / hoisting allowed
#else
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
#endif
#endif
  return p;
}
__device__ __forceinline__ unsigned long long pol_last() {
  unsigned long long p = 0;
#if WCSP_L2_HINTS
#if WCSP_POL_PURE
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));   // pure: CSE / hoisting allowed
#else
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
#endif
#endif
  return p;
}
__device__ __forceinline__ unsigned long long ld_hint(const unsigned long long* a, unsigned long long pol) {
#if WCSP_L2_HINTS
  unsigned long long v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol) : "memory");
  return v;
#else
  return __ldcg(a);
#endif
}
__device__ __forceinline__ void st_hint(unsigned long long* a, unsigned long long v, unsigned long long pol) {
#if WCSP_L2_HINTS
  asm volatile("st.global.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(a), "l"(v), "l"(pol) : "memory");
#else
  __stcs(a, v);
#endif
}
__device__ __forceinline__ unsigned atom_max_hint(unsigned* a, unsigned v, unsigned long long pol) {
#if WCSP_L2_HINTS
  unsigned old;
  asm volatile("atom.global.L2::cache_hint.max.u32 %0, [%1], %2, %3;" : "=r"(old) : "l"(a), "r"(v), "l"(pol) : "memory");
  return old;
#else
  return atomicMax(a, v);
#endif
}

__device__ __forceinline__ void red_max_hint(unsigned* a, unsigned v, unsigned long long pol) {
#if WCSP_L2_HINTS
  asm volatile("red.global.max.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(a), "r"(v), "l"(pol) : "memory");
#else
  atomicMax(a, v);
#endif
}

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
// streaming variant (evict-first): weight records of triggered vertices are
// read once per cycle and must not push the vertex state words out of L2
// (WCSP_WT_POLICY = 1: normal caching, 2: evict-last — A/B options)
#ifndef WCSP_WT_POLICY
#define WCSP_WT_POLICY 0
#endif
template <int D> __device__ __forceinline__ WRec<typename Tr<D>::LW> load_wt_cs(const Dev& s, unsigned v) {
  using LW = typename Tr<D>::LW;
  WRec<LW> r;
  if constexpr (sizeof(LW) == 4) {
#if WCSP_WT_POLICY == 0
    uint2 q = __ldcs(reinterpret_cast<const uint2*>(s.wt) + v);
#else
    uint2 q = __ldcg(reinterpret_cast<const uint2*>(s.wt) + v);
#endif
    r.f1 = q.x; r.f2 = q.y;
  } else {
#if WCSP_WT_POLICY == 0
    uint4 q = __ldcs(reinterpret_cast<const uint4*>(s.wt) + v);
    r.f1 = ((unsigned long long)q.y << 32) | q.x;
    r.f2 = ((unsigned long long)q.w << 32) | q.z;
#elif WCSP_WT_POLICY == 1
    uint4 q = __ldcg(reinterpret_cast<const uint4*>(s.wt) + v);
    r.f1 = ((unsigned long long)q.y << 32) | q.x;
    r.f2 = ((unsigned long long)q.w << 32) | q.z;
#else
    unsigned long long a, b;
    asm volatile("ld.global.L2::cache_hint.v2.u64 {%0, %1}, [%2], %3;"
                 : "=l"(a), "=l"(b) : "l"(reinterpret_cast<const unsigned long long*>(s.wt) + 2 * (size_t)v), "l"(pol_last()));
    r.f1 = a; r.f2 = b;
#endif
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
// Shared memory (dynamic; one layout for every kernel)
// ---------------------------------------------------------------------------
struct LagState {                  // k_wheel_lag: the decision chain (identical in every block)
  long long pl, pp;                // events in flight at the top of the next cycle to decide
  unsigned dn;                     // next cycle to decide
  unsigned ncount, pad_;           // counted cycles so far; the last decided cycle was counted
  unsigned region, lmode;          // the latest decision's parameters for the next views
  int status;                      // ST_RUNNING or the terminal status
};

struct Smem {
  unsigned long long qp[QP_CAP];   // phantom / event staging (wheel: delay in bits 56..63)
  unsigned qa[QA_CAP];             // active-list staging
  union {
    unsigned short wl[WARPS][WIN_VERTS];   // per-warp list of the triggered vertices of its window
                                           // (offsets in the window: a small footprint leaves L1 room)
    unsigned short rank[QP_CAP];   // wheel flush: rank of an event within its delay bin
  };
  unsigned hist[WHEEL], hlane[WHEEL], rfill[WHEEL], rcap[WHEEL];
  unsigned ofill[WHEEL];           // wheel: events appended past the staging into the open regions
  unsigned long long hbase[WHEEL], rpos[WHEEL];
#if WCSP_WARP_FLUSH
  // warp-level event filing: warp w stages in qp[w * WQ, (w + 1) * WQ) and files its own
  // events into the block's open regions (per-delay locks) without block barriers
  unsigned wnp[WARPS];
  unsigned whist[WARPS][WHEEL];    // (count | lane events << 16), then the ring index of the delay's slot
  unsigned short wrank[QP_CAP];
  int rlock[WHEEL];
#endif
  unsigned wtot[WARPS];            // treat, shared rounds: triggered vertices per warp window
  unsigned claim;                  // treat, shared rounds: next unclaimed 32-vertex batch (WCSP_CLAIM)
  unsigned na, np, nspill;
  unsigned bm_lo, bm_words;        // wheel fire, dense cycles: the block's triggered bitmap in qp covers
                                   // vertices [bm_lo, bm_lo + 32 * bm_words)
  unsigned base_a, base_b, flag, ovf;
  unsigned flag2;                  // k_wheel_lag: warp 1's neighbourhood wait beside warp 0's decisions
  unsigned f_nd, f_prep;           // fire: descriptors of this block's bucket; prologue already run
  unsigned long long alloc_lim;    // event-ring allocations of this treat must stay below (hybrid guard)
  View view;
  unsigned long long bhit;
  unsigned long long tphase;       // globaltimer at the start of this block's phase
  unsigned long long red[WARPS][7];
  unsigned redmin[WARPS];
#if WCSP_TREAT_STAGE
  alignas(16) unsigned long long stg[WCSP_STAGE_WORDS];   // the round's band of state words
  unsigned long long stg_bar;      // mbarrier of the bulk copy
  unsigned stg_lo, stg_n, stg_phase;
#endif
  LagState lag;                    // k_wheel_lag only
};

__device__ __forceinline__ Smem& smem() {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  return *reinterpret_cast<Smem*>(smem_raw);
}

#if WCSP_TREAT_STAGE
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
// thread 0: stage words [lo, lo + n) of sw into sm.stg (n even, lo even: 16-byte granules)
__device__ __forceinline__ void stage_issue(const Dev& s, Smem& sm, unsigned lo, unsigned n) {
  const unsigned bar = smem_u32(&sm.stg_bar), dst = smem_u32(sm.stg), bytes = n * 8u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");    // generic reads of the old band first
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(s.sw + lo), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void stage_wait(Smem& sm, unsigned phase) {
  const unsigned bar = smem_u32(&sm.stg_bar);
  unsigned done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(bar), "r"(phase) : "memory");
}
#endif

template <class T>
__device__ __forceinline__ void qpush(T* qbuf, unsigned qcap, unsigned* qn, bool pred, T x, unsigned* gcount,
                                      T* out, unsigned long long cap) {
  const unsigned m = __ballot_sync(0xFFFFFFFFu, pred);
  if (m == 0) return;
  const unsigned lane = threadIdx.x & 31u;
  const int leader = __ffs(m) - 1;
  unsigned base = 0;
  if ((int)lane == leader) base = atomicAdd(qn, (unsigned)__popc(m));
  base = __shfl_sync(0xFFFFFFFFu, base, leader);
  if (pred) {
    const unsigned idx = base + __popc(m & ((1u << lane) - 1u));
    if (idx < qcap) {
      qbuf[idx] = x;
    } else {                        // rare: queue full, append straight to the global list
      const unsigned long long pos = atomicAdd(gcount, 1u);
      if (pos < cap) out[pos] = x;
    }
  }
}

// Flush the active-list and phantom queues with one reservation round (P: the phantom record,
// u64 or the wide layout's PhW staged in the same shared buffer).
template <class P = unsigned long long>
__device__ __forceinline__ void qflush(Smem& sm, unsigned* ga, unsigned* outa, unsigned* gp, P* outp,
                                       unsigned long long capp) {
  constexpr unsigned QCAP = QP_CAP * sizeof(unsigned long long) / sizeof(P);
  const P* qp = reinterpret_cast<const P*>(sm.qp);
  __syncthreads();
  const unsigned na = min(sm.na, (unsigned)QA_CAP), np = min(sm.np, QCAP);
  if (na == 0 && np == 0) return;                 // uniform: every thread read the same counts
  if (threadIdx.x == 0) {
    sm.base_a = na ? atomicAdd(ga, na) : 0u;
    sm.base_b = np ? atomicAdd(gp, np) : 0u;
  }
  __syncthreads();
  const unsigned long long ba = sm.base_a, bb = sm.base_b;
  for (unsigned i = threadIdx.x; i < na; i += THREADS) outa[ba + i] = sm.qa[i];
  for (unsigned i = threadIdx.x; i < np; i += THREADS)
    if (bb + i < capp) outp[bb + i] = qp[i];
  if (threadIdx.x == 0) { sm.na = 0; sm.np = 0; }  // no push can happen before the barrier below
  __syncthreads();
}

// block reductions -> one global atomic per counter per block
__device__ __forceinline__ void block_reduce_commit(Smem& sm, unsigned dmin, unsigned long long a0,
                                                    unsigned long long a1, unsigned long long a2,
                                                    unsigned long long a3, unsigned long long a4, Acc* acc,
                                                    unsigned long long a5 = 0, unsigned long long a6 = 0) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dmin = min(dmin, __shfl_xor_sync(0xFFFFFFFFu, dmin, o));
    a0 += __shfl_xor_sync(0xFFFFFFFFu, a0, o);
    a1 += __shfl_xor_sync(0xFFFFFFFFu, a1, o);
    a2 += __shfl_xor_sync(0xFFFFFFFFu, a2, o);
    a3 += __shfl_xor_sync(0xFFFFFFFFu, a3, o);
    a4 += __shfl_xor_sync(0xFFFFFFFFu, a4, o);
    a5 += __shfl_xor_sync(0xFFFFFFFFu, a5, o);
    a6 += __shfl_xor_sync(0xFFFFFFFFu, a6, o);
  }
  const unsigned w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    sm.redmin[w] = dmin;
    sm.red[w][0] = a0; sm.red[w][1] = a1; sm.red[w][2] = a2; sm.red[w][3] = a3; sm.red[w][4] = a4;
    sm.red[w][5] = a5;
    sm.red[w][6] = a6;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned m = 0xFFFFFFFFu;
    unsigned long long s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0, s6 = 0;
    for (int i = 0; i < WARPS; ++i) {
      m = min(m, sm.redmin[i]);
      s0 += sm.red[i][0]; s1 += sm.red[i][1]; s2 += sm.red[i][2]; s3 += sm.red[i][3]; s4 += sm.red[i][4];
      s5 += sm.red[i][5];
      s6 += sm.red[i][6];
    }
    if (m != 0xFFFFFFFFu) atomicMin(&acc->dmin, m);
    if (s0) atomicAdd(&acc->live, s0);
    if (s1) atomicAdd(&acc->arrivals, s1);
    if (s2) atomicAdd(&acc->created, s2);
    if (s3) atomicAdd(&acc->relabels, s3);
    if (s4) atomicAdd(&acc->triggered, s4);
    if (s5) atomicAdd(&acc->started, s5);
    if (s6) atomicAdd(&acc->tested, s6);
  }
  __syncthreads();
}

// Water of quality `cand` reaches D from `src` (quality <= 0
// cannot travel, :29): temp(D) := max(temp(D), cand) — one atomic whose
// return value says whether D is a target, removed, or triggered for the
// first time this cycle.  The comparison with L(D) ("L(S) - f2(e) > L(D)",
// :32) is made once per triggered vertex in treat: max over all arrivals
// beats L(D) iff max over the accepted ones does, and then they are equal
// (reading R-new-1).  Split in two so a thread can put several atomics in
// flight before it needs their results: arrive_atomic issues the atomicMax,
// arrive_post acts on its return value (the bitmap OR is a fire-and-forget
// reduction).
// Peer halo: where local index D lives (its owner's state words and bitmap, the index
// there, the owner's global offset).  Without PEER every index is local.
struct Loc { unsigned long long* sw; unsigned* tb; unsigned idx; unsigned goff; };
template <bool PEER>
__device__ __forceinline__ Loc locate(const Dev& s, unsigned D) {
  if constexpr (PEER) {
    if (D < s.plo_end) return Loc{s.psw[0], s.ptb[0], D + s.pshift[0], s.pgoff[0]};
    if (D >= s.ghost_hi_start) return Loc{s.psw[1], s.ptb[1], D + s.pshift[1], s.pgoff[1]};
  }
  return Loc{s.sw, s.tbits, D, s.goff};
}

// Every state-word atomic of the peer halo is system-scoped: the neighbour GPU's
// threads update the same words.
__device__ __forceinline__ unsigned atom_max_sys(unsigned* a, unsigned v) {
  unsigned old;
  asm volatile("atom.relaxed.sys.global.max.u32 %0, [%1], %2;" : "=r"(old) : "l"(a), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_max_sys(unsigned* a, unsigned v) {
  asm volatile("red.relaxed.sys.global.max.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void atom_or_sys(unsigned* a, unsigned v) {
  asm volatile("red.relaxed.sys.global.or.b32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}

template <bool PEER = false>
__device__ __forceinline__ unsigned arrive_atomic(const Dev& s, const View& v, bool go, unsigned D, int cand) {
  if constexpr (PEER) {
    if (!go) return v.stamp << 16;
    const Loc L = locate<true>(s, D);
    return atom_max_sys(tmp_ptr(L.sw, L.idx), (v.stamp << 16) | (unsigned)cand);
  } else {
    return go ? atom_max_hint(tmp_ptr(s.sw, D), (v.stamp << 16) | (unsigned)cand, pol_last()) : (v.stamp << 16);
  }
}

// src is a GLOBAL vertex index (local index + s.goff); D is local.
template <bool PEER = false, bool LIST = false>
__device__ __forceinline__ void arrive_post(const Dev& s, const View& v, Acc* acc, unsigned old, unsigned D,
                                            int cand, unsigned src, unsigned via, Smem* sm = nullptr) {
  const unsigned os = old >> 16;
  if (os == 0xFFFFu) {
    if (old == TMP_B) {            // termination 1°: a vertex of B is reached
      const Loc L = locate<PEER>(s, D);
      const unsigned Dg = L.idx + L.goff;
      atomicMax(&acc->bhit, ((unsigned long long)(unsigned)cand << 32) | (0xFFFFFFFFu - Dg));
      const unsigned par = v.c & 1u;
      const unsigned k = atomicAdd(&s.ctl->n_barr2[par], 1u);
      if (k < s.barr_cap) s.barr[(size_t)par * s.barr_cap + k] = BArr{Dg, (unsigned)cand, src, via};
    } else if (!PEER && old >= TMP_GHOST) {   // D belongs to a neighbouring slab: hand the water to its owner
      unsigned long long* slot = D < s.plane ? s.ghost_out_lo + D : s.ghost_out_hi + (D - s.ghost_hi_start);
      atomicMax(slot, ((unsigned long long)v.stamp << 48) | ((unsigned long long)(unsigned)cand << 32) |
                          ((unsigned long long)(0x7FFFFFFFu - src) << 1) | (unsigned long long)(via ? 0u : 1u));
    }
  } else if (os != v.stamp) {      // first arrival of the cycle: D is triggered (dedupe)
    if (LIST && sm) {
      if (v.lmode) {               // sparse cycle: the firing block lists it for its own treat while it has room
        const unsigned k = atomicAdd(&sm->na, 1u);
        if (k < (unsigned)QA_CAP) { sm->qa[k] = D; return; }
      } else {                     // dense cycle: near the block's own slab, a shared-memory bit first
        const unsigned r = D - sm->bm_lo;
        if (r < sm->bm_words * 32u && (!PEER || (D >= s.plo_end && D < s.ghost_hi_start))) {
          atomicOr(reinterpret_cast<unsigned*>(sm->qp) + (r >> 5), 1u << (r & 31u));
          return;
        }
      }
    }
    if constexpr (PEER) {
      const Loc L = locate<true>(s, D);
      atom_or_sys(L.tb + (L.idx >> 5), 1u << (L.idx & 31u));
    } else {
      atomicOr(s.tbits + (D >> 5), 1u << (D & 31u));
    }
  }
}

// The same two halves for wide labels: temp(D) = stamp:32 | cand:32, one 64-bit atomicMax.
__device__ __forceinline__ unsigned long long arrive_atomic_w(const Dev& s, const View& v, bool go, unsigned D,
                                                              int cand) {
  const unsigned long long key = ((unsigned long long)v.stamp << 32) | (unsigned)cand;
  return go ? atomicMax(s.sw + D, key) : key;
}
__device__ __forceinline__ void arrive_post_w(const Dev& s, const View& v, Acc* acc, unsigned long long old,
                                              unsigned D, int cand, unsigned src, unsigned via) {
  const unsigned os = (unsigned)(old >> 32);
  if (os == 0xFFFFFFFFu) {
    if (old == TMPW_B) {           // termination 1°
      const unsigned Dg = D + s.goff;
      atomicMax(&acc->bhit, ((unsigned long long)(unsigned)cand << 32) | (0xFFFFFFFFu - Dg));
      const unsigned par = v.c & 1u;
      const unsigned k = atomicAdd(&s.ctl->n_barr2[par], 1u);
      if (k < s.barr_cap) s.barr[(size_t)par * s.barr_cap + k] = BArr{Dg, (unsigned)cand, src, via};
    }
  } else if (os != v.stamp) {      // first arrival of the cycle
    atomicOr(s.tbits + (D >> 5), 1u << (D & 31u));
  }
}
template <bool W> using OldT = std::conditional_t<W, unsigned long long, unsigned>;
template <bool W>
__device__ __forceinline__ OldT<W> arrive_a(const Dev& s, const View& v, bool go, unsigned D, int cand) {
  if constexpr (W) return arrive_atomic_w(s, v, go, D, cand);
  else return arrive_atomic(s, v, go, D, cand);
}
template <bool W>
__device__ __forceinline__ void arrive_p(const Dev& s, const View& v, Acc* acc, OldT<W> old, unsigned D, int cand,
                                         unsigned src, unsigned via) {
  if constexpr (W) arrive_post_w(s, v, acc, old, D, cand, src, via);
  else arrive_post(s, v, acc, old, D, cand, src, via);
}

// ---------------------------------------------------------------------------
// sweep: Steps 1, 3, 7 and the retirement part of 8-9 (sweep engine)
// ---------------------------------------------------------------------------
template <int D, bool W = false>
__device__ void phase_sweep(const Dev& s, const View& v, Smem& sm) {
  using LW = typename Tr<D>::LW;
  Acc* acc = &s.ctl->acc[v.c % NACC];
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
        WCSP_CHECK(vx[it] == 0xFFFFFFFFu || vx[it] < s.N, "sweep: active-list entry", vx[it], s.N);
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
        qpush<unsigned>(sm.qa, QA_CAP, &sm.na, survive, vx[it], &acc->n_act, act_out, 0xFFFFFFFFull);
      }
      unsigned lbl[SWEEP_ITEMS];
      LW f2w[SWEEP_ITEMS];
#pragma unroll
      for (int it = 0; it < SWEEP_ITEMS; ++it) {
        lbl[it] = 0; f2w[it] = 0;
        if (fired[it]) {
          if constexpr (W) lbl[it] = s.minf ? 1u : __ldcg(s.lab + vx[it]);
          else lbl[it] = s.minf ? 1u : (__ldcg(lbl_ptr(s.sw, vx[it])) & 0xFFFFu);
          if (!s.minf) f2w[it] = load_f2<D>(s, vx[it]);
        }
      }
#pragma unroll
      for (int it = 0; it < SWEEP_ITEMS; ++it) {
        if (!fired[it]) continue;
        OldT<W> old[2 * D];
#pragma unroll
        for (int j = 0; j < 2 * D; ++j) {
          const bool fj = (fired[it] >> (8 * j + 7)) & 1;
          arr += fj;
          const int cand = (int)lbl[it] - (int)((f2w[it] >> (8 * j)) & 0xFF);
          old[j] = arrive_a<W>(s, v, fj && cand > 0, vx[it] + s.off[j], cand);
        }
#pragma unroll
        for (int j = 0; j < 2 * D; ++j) {
          const int cand = (int)lbl[it] - (int)((f2w[it] >> (8 * j)) & 0xFF);
          arrive_p<W>(s, v, acc, old[j], vx[it] + s.off[j], cand, vx[it] + s.goff, 0u);
        }
      }
    } else if constexpr (W) {        // wide phantoms: 16-byte records, 64-bit temp atomics
      const unsigned pc = ch - na_ch;
      const PhW* pin = reinterpret_cast<const PhW*>(pool_in);
      PhW* pout = reinterpret_cast<PhW*>(pool_out);
      PhW p[SWEEP_ITEMS];
#pragma unroll
      for (int it = 0; it < SWEEP_ITEMS; ++it) {
        const unsigned i = pc * chunk + it * THREADS + threadIdx.x;
        if ((unsigned)it < items && i < v.n_pool) {
          const ulonglong2 q2 = __ldcs(reinterpret_cast<const ulonglong2*>(pin + i));
          p[it] = PhW{q2.x, q2.y};
        } else {
          p[it] = PhW{0ull, 0ull};
        }
      }
      unsigned long long old[SWEEP_ITEMS];
#pragma unroll
      for (int it = 0; it < SWEEP_ITEMS; ++it) {
        const unsigned r = (unsigned)(p[it].x >> PHW_RES) & 0xFFu;   // 0 only for padding
        const bool fire = r != 0 && r == v.delta;
        const bool keep = r > v.delta;
        if (keep) dmin = min(dmin, r - v.delta);
        arr += fire;
        qpush<PhW>(reinterpret_cast<PhW*>(sm.qp), QP_CAP / 2, &sm.np, keep,
                   PhW{p[it].x - ((unsigned long long)v.delta << PHW_RES), p[it].y}, &acc->n_pool, pout, s.pool_cap);
        const unsigned src = (unsigned)p[it].x & 0x3FFFFFFFu;
        const unsigned lane = (unsigned)(p[it].x >> PH_LANE) & 7u;
        old[it] = arrive_atomic_w(s, v, fire, src + s.off[lane], (int)(unsigned)p[it].y);
      }
#pragma unroll
      for (int it = 0; it < SWEEP_ITEMS; ++it) {
        const unsigned src = (unsigned)p[it].x & 0x3FFFFFFFu;
        const unsigned lane = (unsigned)(p[it].x >> PH_LANE) & 7u;
        arrive_post_w(s, v, acc, old[it], src + s.off[lane], (int)(unsigned)p[it].y, src + s.goff, 1u);
      }
    } else {
      const unsigned pc = ch - na_ch;
      unsigned long long p[SWEEP_ITEMS];
#pragma unroll
      for (int it = 0; it < SWEEP_ITEMS; ++it) {
        const unsigned i = pc * chunk + it * THREADS + threadIdx.x;
        p[it] = ((unsigned)it < items && i < v.n_pool) ? __ldcs(pool_in + i) : 0ull;
        WCSP_CHECK(p[it] == 0ull || (((unsigned)p[it] & 0x3FFFFFFFu) < s.N && ((p[it] >> PH_LANE) & 7u) < (unsigned)s.NL),
                   "sweep: phantom record", p[it], s.N);
      }
      unsigned old[SWEEP_ITEMS];
#pragma unroll
      for (int it = 0; it < SWEEP_ITEMS; ++it) {
        const unsigned r = (unsigned)(p[it] >> PH_RES) & 0xFFu;   // 0 only for padding
        const bool fire = r != 0 && r == v.delta;
        const bool keep = r > v.delta;
        if (keep) dmin = min(dmin, r - v.delta);
        arr += fire;
        qpush<unsigned long long>(sm.qp, QP_CAP, &sm.np, keep, p[it] - ((unsigned long long)v.delta << PH_RES),
                                  &acc->n_pool, pool_out, s.pool_cap);
        const unsigned src = (unsigned)p[it] & 0x3FFFFFFFu;
        const unsigned lane = (unsigned)(p[it] >> PH_LANE) & 7u;
        old[it] = arrive_atomic(s, v, fire, src + s.off[lane], (int)((p[it] >> PH_CAND) & 0xFFFFu));
      }
#pragma unroll
      for (int it = 0; it < SWEEP_ITEMS; ++it) {
        const unsigned src = (unsigned)p[it] & 0x3FFFFFFFu;
        const unsigned lane = (unsigned)(p[it] >> PH_LANE) & 7u;
        arrive_post(s, v, acc, old[it], src + s.off[lane], (int)((p[it] >> PH_CAND) & 0xFFFFu), src + s.goff, 1u);
      }
    }
    if constexpr (W) qflush<PhW>(sm, &acc->n_act, act_out, &acc->n_pool, reinterpret_cast<PhW*>(pool_out), s.pool_cap);
    else qflush(sm, &acc->n_act, act_out, &acc->n_pool, pool_out, s.pool_cap);
  }
  block_reduce_commit(sm, dmin, live, arr, 0, 0, 0, acc);
}

// ---------------------------------------------------------------------------
// Triggered-bitmap windows: warp w of the block takes window
// (round * gridDim + block) * WARPS + w, clears it and lists its set bits in
// ascending vertex order (sorted processing: neighbouring Q share sectors).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned window_take(const Dev& s, unsigned win, unsigned short* list) {
  // every lane takes 32 / lpw bits of one word (lpw lanes per word), so the serial
  // bit extraction is short and all 32 lanes share it
  const unsigned lane = threadIdx.x & 31u;
  const unsigned ww = s.win_words, lg = __ffs(ww) - 1u, bpl = ww;   // ww: a power of two (no divisions)
  const unsigned wi = win * ww + (lane >> (5u - lg)), sub = lane & ((32u >> lg) - 1u);
  unsigned w = wi < s.nwords ? __ldcg(s.tbits + wi) : 0u;
  __syncwarp();
  if (sub == 0 && w) s.tbits[wi] = 0u;
  w = (w >> (sub * bpl)) & (bpl == 32u ? 0xFFFFFFFFu : ((1u << bpl) - 1u));
  const unsigned c = __popc(w);
  unsigned x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if ((int)lane >= o) x += y;
  }
  const unsigned total = __shfl_sync(0xFFFFFFFFu, x, 31);
  unsigned pos = x - c;
  const unsigned vbase = (lane >> (5u - lg)) * 32u + sub * bpl;   // offset in the window
  while (w) {
    list[pos++] = (unsigned short)(vbase + (unsigned)(__ffs(w) - 1));
    w &= w - 1u;
  }
  __syncwarp();
  return total;
}

// Shared rounds (WCSP_ROUND_SHARE): the WARPS windows of a round form one list in vertex
// order that all warps of the block work through together, so a round lasts the mean of its
// windows' work instead of the max.  window_bits loads and clears one window and returns this
// lane's share of its bits; window_emit writes them at `base` as offsets in the round.
__device__ __forceinline__ unsigned window_bits(const Dev& s, unsigned win, unsigned nwin) {
  const unsigned lane = threadIdx.x & 31u;
  const unsigned ww = s.win_words, lg = __ffs(ww) - 1u, bpl = ww;   // ww: a power of two (no divisions)
  const unsigned wi = win * ww + (lane >> (5u - lg)), sub = lane & ((32u >> lg) - 1u);
  unsigned w = win < nwin && wi < s.nwords ? __ldcg(s.tbits + wi) : 0u;
  __syncwarp();
  if (sub == 0 && w) s.tbits[wi] = 0u;
  return (w >> (sub * bpl)) & (bpl == 32u ? 0xFFFFFFFFu : ((1u << bpl) - 1u));
}
// The same in two steps, so the load of the next round's window can be in flight while the
// current round is treated: window_load issues it; window_use (at the next round) clears the
// word and returns this lane's share of its bits.
__device__ __forceinline__ unsigned window_load(const Dev& s, unsigned win, unsigned nwin) {
  const unsigned lane = threadIdx.x & 31u;
  const unsigned ww = s.win_words, lg = __ffs(ww) - 1u;
  const unsigned wi = win * ww + (lane >> (5u - lg));
  return win < nwin && wi < s.nwords ? __ldcg(s.tbits + wi) : 0u;
}
__device__ __forceinline__ unsigned window_use(const Dev& s, unsigned win, unsigned w) {
  const unsigned lane = threadIdx.x & 31u;
  const unsigned ww = s.win_words, lg = __ffs(ww) - 1u, bpl = ww;   // ww: a power of two (no divisions)
  const unsigned wi = win * ww + (lane >> (5u - lg)), sub = lane & ((32u >> lg) - 1u);
  if (sub == 0 && w) s.tbits[wi] = 0u;
  return (w >> (sub * bpl)) & (bpl == 32u ? 0xFFFFFFFFu : ((1u << bpl) - 1u));
}
__device__ __forceinline__ void window_emit(const Dev& s, unsigned bits, unsigned base, unsigned short* list,
                                            unsigned woff) {
  const unsigned lane = threadIdx.x & 31u;
  const unsigned ww = s.win_words, lg = __ffs(ww) - 1u, bpl = ww, sub = lane & ((32u >> lg) - 1u);
  const unsigned cnt = __popc(bits);
  unsigned x = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if ((int)lane >= o) x += y;
  }
  unsigned pos = base + x - cnt;
  const unsigned vbase = woff + (lane >> (5u - lg)) * 32u + sub * bpl;
  while (bits) {
    list[pos++] = (unsigned short)(vbase + (unsigned)(__ffs(bits) - 1));
    bits &= bits - 1u;
  }
}

// ---------------------------------------------------------------------------
// treat: Steps 4, 5, 8.1 for one triggered vertex q (both engines).
// WHEEL = false: lanes are residual bytes in res[q]; phantoms go to the pool.
// WHEEL = true : lanes and phantoms are events filed at t + f1 (wcsp_wheel.cuh).
// ---------------------------------------------------------------------------
template <int D, bool WHEEL_ENGINE, bool PEER = false, bool W = false>
__device__ __forceinline__ void treat_one(const Dev& s, const View& v, Smem& sm, Acc* acc, unsigned q,
                                          unsigned& dmin, unsigned& created,
                                          unsigned& relabels, unsigned& triggered,
                                          unsigned& lanes_started, unsigned& tested);

__device__ __forceinline__ bool lane_live(unsigned texp16, long long t) {
  return ((texp16 - (unsigned)t) & 0xFFFFu) - 1u < 255u;   // texp in (t, t + 255]
}

// Stage events for the wheel (defined in wcsp_wheel.cuh): at a reserved staging slot, or
// one per predicated lane (warp-aggregated).
#ifndef WCSP_TREAT_EAGER
#define WCSP_TREAT_EAGER 2         // 1: issue the neighbour loads together with Q's own; 2: on 2-D grids only
#endif                             // (lagged kernel: C2 85.3 -> 83.4 ms, C3 +3.8 % with 1; ab_treat_lag*.txt)
__host__ __device__ constexpr bool treat_eager(int d) { return WCSP_TREAT_EAGER == 1 || (WCSP_TREAT_EAGER == 2 && d == 2); }
#ifndef WCSP_ROUND_SHARE
#define WCSP_ROUND_SHARE 1         // the warps of a block share each treat round's vertices
#endif
#ifndef WCSP_WARP_FLUSH
#define WCSP_WARP_FLUSH 0          // 1: every warp files its own events (no block barriers in the treat);
                                   //    measured on C3: treat +9 %, fire +64 % (interleaved runs) -- off
#endif
#ifndef WCSP_WIN_PREFETCH
#define WCSP_WIN_PREFETCH 1        // 1: the next round's bitmap words load while this round is treated (with TREAT_PF
                                   // on the lagged kernel: C3 123.2 -> 121.85, C2 85.3 -> 83.6 ms; ab_treat_lag2.txt)
#endif
#ifndef WCSP_CLAIM
#define WCSP_CLAIM 0               // 1: warps claim a round's batches dynamically (measured: C3 +0.6 %, C2 +1.8 %; off)
#endif
#ifndef WCSP_NB_L2
#define WCSP_NB_L2 0               // 1: the Step-4 neighbour words bypass L1 (A/B)
#endif
#ifndef WCSP_TREAT_PF
#define WCSP_TREAT_PF 1            // 1: prefetch the next batch's state word (L2) and weight record (L1)
#endif
#ifndef WCSP_TREAT_AGG
#define WCSP_TREAT_AGG 1           // one warp-scan staging reservation per treat batch (not one per lane direction)
#endif
#ifndef WCSP_FLUSH_LAZY
#define WCSP_FLUSH_LAZY (WCSP_QP_CAP / 2)   // > 0: treat flushes its staged events only above this many
#endif
__device__ void ev_stage(const Dev& s, Smem& sm, unsigned idx, unsigned long long rec, unsigned delay, long long t);
__device__ void ev_push(const Dev& s, Smem& sm, bool pred, unsigned long long rec, unsigned delay, long long t);
__device__ void ev_push_warp(const Dev& s, Smem& sm, bool pred, unsigned long long rec, unsigned delay, long long t,
                             unsigned region);
__device__ void warp_flush(const Dev& s, Smem& sm, long long t, unsigned region);
__device__ void regions_close(const Dev& s, Smem& sm, long long t);

template <int D, bool WHEEL_ENGINE, bool PEER, bool W>
__device__ __forceinline__ void treat_one(const Dev& s, const View& v, Smem& sm, Acc* acc, unsigned q,
                                          unsigned& dmin, unsigned& created,
                                          unsigned& relabels, unsigned& triggered,
                                          unsigned& lanes_started, unsigned& tested) {
  using LW = typename Tr<D>::LW;
  const bool valid = q != 0xFFFFFFFFu;
  WCSP_CHECK(!valid || q < s.N, "treat: vertex index", q, s.N);
  tested += valid;
  if constexpr (W) {
    static_assert(!WHEEL_ENGINE && !PEER, "wide labels: sweep engine, single device");
    // Wide labels: the same Steps 4, 5, 8.1 on L(v) = lab[v] (u32) and temp = stamp:32 | cand:32
    const unsigned long long tq = valid ? __ldcg(s.sw + q) : 0ull;
    const int lq = valid ? (int)__ldcg(s.lab + q) : 0;
    const WRec<LW> wr = valid ? load_wt_cs<D>(s, q) : WRec<LW>{0, 0};
    const LW w = valid ? __ldcg(reinterpret_cast<LW*>(s.res) + q) : (LW)0;
    const int lstar = (int)(unsigned)tq;                         // L* = temp(Q) (reading R23)
    const bool trig = valid && lstar > lq;
    const bool inactive = trig && w == 0;                        // reading R6
    triggered += trig;
    int rl[2 * D];
    unsigned long long rtw[2 * D];
#pragma unroll
    for (int j = 0; j < 2 * D; ++j) {
      const unsigned f1j = (unsigned)(wr.f1 >> (8 * j)) & 0xFFu;
      const unsigned f2j = s.minf ? 0u : (unsigned)(wr.f2 >> (8 * j)) & 0xFFu;
      const bool test = trig && f1j != 0 && lstar - (int)f2j > 0;
      rl[j] = test ? (int)__ldcg(s.lab + (q + s.off[j])) : (int)LBL_REMOVED_W;
      rtw[j] = test ? __ldcg(s.sw + (q + s.off[j])) : 0ull;
    }
    LW neww = 0;
#pragma unroll
    for (int j = 0; j < 2 * D; ++j) {
      const unsigned f1j = (unsigned)(wr.f1 >> (8 * j)) & 0xFFu;
      const unsigned f2j = s.minf ? 0u : (unsigned)(wr.f2 >> (8 * j)) & 0xFFu;
      const int c = lstar - (int)f2j;
      const int rt = (unsigned)(rtw[j] >> 32) == v.stamp ? (int)(unsigned)rtw[j] : 0;
      const bool pass = c > max(rl[j], rt);                      // edge triggered
      const bool ph = pass && !inactive;                         // phantom
      created += ph;
      lanes_started += pass && inactive;                         // time restored to f1
      if (pass) dmin = min(dmin, f1j);
      if (pass && inactive) neww |= (LW)f1j << (8 * j);
      const PhW prec{(unsigned long long)q | ((unsigned long long)j << PH_LANE) | ((unsigned long long)f1j << PHW_RES),
                     (unsigned long long)(unsigned)c};
      qpush<PhW>(reinterpret_cast<PhW*>(sm.qp), QP_CAP / 2, &sm.np, ph, prec, &acc->n_pool,
                 reinterpret_cast<PhW*>(s.pool[v.cur ^ 1]), s.pool_cap);
    }
    if (inactive) {                                              // Step 8.1
      relabels += 1;
      s.lab[q] = (unsigned)lstar;
      if (neww) __stcg(reinterpret_cast<LW*>(s.res) + q, neww);
    }
    qpush<unsigned>(sm.qa, QA_CAP, &sm.na, inactive && neww != 0, q, &acc->n_act, s.act[v.cur ^ 1], 0xFFFFFFFFull);
    return;
  }
#if WCSP_TREAT_STAGE
  const unsigned slo = sm.stg_lo, sn = sm.stg_n;
  auto staged = [&](unsigned u) { return u - slo < sn; };
  const unsigned long long swq = valid ? (staged(q) ? sm.stg[q - slo] : ld_hint(s.sw + q, pol_last())) : 0ull;
#else
  const unsigned long long swq = valid ? ld_hint(s.sw + q, pol_last()) : 0ull;
#endif
  const WRec<LW> wr = valid ? load_wt_cs<D>(s, q) : WRec<LW>{0, 0};
  unsigned long long swr[2 * D];
  if constexpr (!PEER && treat_eager(D)) {   // neighbours loaded with Q's own words: one round trip
#pragma unroll
    for (int j = 0; j < 2 * D; ++j) {
      const unsigned u = q + s.off[j];
      swr[j] = valid && u < s.N ? s.sw[u] : 0xFFFFull;
    }
  }
  LW w = 0;
  if constexpr (!WHEEL_ENGINE) w = valid ? __ldcg(reinterpret_cast<LW*>(s.res) + q) : (LW)0;
  const int lq = (int)(swq & 0xFFFFu);
  const int lstar = (int)((swq >> 32) & 0xFFFFu);                 // L* = temp(Q) (reading R23)
  const bool trig = valid && lstar > lq;                          // the water improves Q
  bool inactive;
  if constexpr (WHEEL_ENGINE) inactive = trig && !lane_live((unsigned)(swq >> 16) & 0xFFFFu, v.t);
  else inactive = trig && w == 0;                                 // no live lane after the decrement (R6)
  triggered += trig;
#pragma unroll
  for (int j = 0; j < 2 * D; ++j) {
    const unsigned f1j = (unsigned)(wr.f1 >> (8 * j)) & 0xFFu;
    const unsigned f2j = s.minf ? 0u : (unsigned)(wr.f2 >> (8 * j)) & 0xFFu;
    const bool test = trig && f1j != 0 && lstar - (int)f2j > 0;
    if constexpr (!PEER && treat_eager(D)) {
      if (!test) swr[j] = 0xFFFFull;   // untested lanes read as "removed"
      continue;
    }
    // L1-cached read: this phase never writes the temp half, the label half only moves to
    // max(L, temp) (benign), and the grid barrier before the phase invalidated L1
    if constexpr (PEER) {            // a neighbour in the next slab is read in its owner's memory
      const Loc L = locate<true>(s, q + s.off[j]);
      swr[j] = test ? (L.sw == s.sw ? s.sw[L.idx] : __ldcv(L.sw + L.idx)) : 0xFFFFull;
    } else {
      WCSP_CHECK(!test || q + s.off[j] < s.N, "treat: neighbour index", q, j);
#if WCSP_TREAT_STAGE
      const unsigned u = q + s.off[j];
      swr[j] = test ? (staged(u) ? sm.stg[u - slo] : s.sw[u]) : 0xFFFFull;
#else
#if WCSP_NB_L2
      swr[j] = test ? __ldcg(s.sw + (q + s.off[j])) : 0xFFFFull;   // A/B: neighbour words from L2
#else
      swr[j] = test ? s.sw[q + s.off[j]] : 0xFFFFull;   // untested lanes read as "removed"
#endif
#endif
    }
  }
  LW neww = 0;
  unsigned fmax = 0;
  unsigned pm = 0, spm = 0;          // WCSP_TREAT_AGG: the lanes whose edge passed (bit j), and those
                                     // whose destination holds a sentinel temp (target, ghost: bit 50)
#pragma unroll
  for (int j = 0; j < 2 * D; ++j) {
    const unsigned f1j = (unsigned)(wr.f1 >> (8 * j)) & 0xFFu;
    const unsigned f2j = s.minf ? 0u : (unsigned)(wr.f2 >> (8 * j)) & 0xFFu;
    const int c = lstar - (int)f2j;
    const unsigned rl = (unsigned)swr[j] & 0xFFFFu;
    const unsigned rtw = (unsigned)(swr[j] >> 32);
    const unsigned rt = (rtw >> 16) == v.stamp ? (rtw & 0xFFFFu) : 0u;
    const bool pass = c > (int)max(rl, rt);                       // edge triggered
    const bool ph = pass && !inactive;                            // phantom (Q, R, L*, f1) (:197-198)
    created += ph;
    lanes_started += pass && inactive;                            // activate, time restored to f1 (:192)
    if constexpr (WHEEL_ENGINE) {
      if (pass && inactive) fmax = max(fmax, f1j);
#if WCSP_TREAT_AGG && !WCSP_WARP_FLUSH
      pm |= (pass ? 1u : 0u) << j;
      spm |= ((rtw >> 16) == 0xFFFFu ? 1u : 0u) << j;
#else
      const unsigned long long rec = (unsigned long long)q | ((unsigned long long)j << PH_LANE) |
                                     ((unsigned long long)(unsigned)c << PH_CAND) |
                                     ((unsigned long long)(inactive ? 1u : 0u) << 49) |
                                     ((unsigned long long)((rtw >> 16) == 0xFFFFu ? 1u : 0u) << 50);
#if WCSP_WARP_FLUSH
      ev_push_warp(s, sm, pass, rec, f1j, v.t, v.region);
#else
      ev_push(s, sm, pass, rec, f1j, v.t);
#endif
#endif
    } else {
      if (pass) dmin = min(dmin, f1j);
      if (pass && inactive) neww |= (LW)f1j << (8 * j);
      const unsigned long long prec = (unsigned long long)q | ((unsigned long long)j << PH_LANE) |
                                      ((unsigned long long)(unsigned)c << PH_CAND) |
                                      ((unsigned long long)f1j << PH_RES);
      qpush<unsigned long long>(sm.qp, QP_CAP, &sm.np, ph, prec, &acc->n_pool, s.pool[v.cur ^ 1], s.pool_cap);
    }
  }
#if WCSP_TREAT_AGG && !WCSP_WARP_FLUSH
  if constexpr (WHEEL_ENGINE) {
    // one staging reservation per warp for all its vertices' events (an exclusive scan of the
    // per-thread counts) instead of one ballot + shared atomic per lane direction
    const unsigned lane = threadIdx.x & 31u;
    const unsigned cnt = __popc(pm);
    unsigned x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if ((int)lane >= o) x += y;
    }
    const unsigned tot = __shfl_sync(0xFFFFFFFFu, x, 31);
    if (tot) {                       // warp-uniform
      unsigned base = 0;
      if (lane == 31) base = atomicAdd(&sm.np, tot);
      base = __shfl_sync(0xFFFFFFFFu, base, 31);
      unsigned idx = base + x - cnt;
#pragma unroll
      for (int j = 0; j < 2 * D; ++j) {
        if ((pm >> j) & 1u) {
          const unsigned f1j = (unsigned)(wr.f1 >> (8 * j)) & 0xFFu;
          const unsigned f2j = s.minf ? 0u : (unsigned)(wr.f2 >> (8 * j)) & 0xFFu;
          const unsigned long long rec = (unsigned long long)q | ((unsigned long long)j << PH_LANE) |
                                         ((unsigned long long)(unsigned)(lstar - (int)f2j) << PH_CAND) |
                                         ((unsigned long long)(inactive ? 1u : 0u) << 49) |
                                         ((unsigned long long)((spm >> j) & 1u) << 50);
          ev_stage(s, sm, idx++, rec, f1j, v.t);
        }
      }
    }
  }
#endif
  if (inactive) {                                                 // Step 8.1
    relabels += 1;
    if constexpr (WHEEL_ENGINE) {
      const unsigned nt = (unsigned)((fmax ? v.t + fmax : v.t) & 0xFFFF);
      *lbl_ptr(s.sw, q) = (unsigned)lstar | (nt << 16);
    } else {
      *lbl_ptr(s.sw, q) = (unsigned)lstar;
      if (neww) __stcg(reinterpret_cast<LW*>(s.res) + q, neww);
    }
  }
  if constexpr (!WHEEL_ENGINE)
    qpush<unsigned>(sm.qa, QA_CAP, &sm.na, inactive && neww != 0, q, &acc->n_act, s.act[v.cur ^ 1], 0xFFFFFFFFull);
}

// Flush hook of the wheel (defined in wcsp_wheel.cuh).
__device__ void ev_flush(const Dev& s, Smem& sm, long long t, unsigned region, bool final_flush);

// The treat windows of block vb: [wlo, whi) in `rounds` rounds of WARPS windows (the last may be
// partial): WARPS * ceil(nwin / (G * WARPS)) windows per block from the start (the tail blocks may
// get none), or balanced slabs [b * nwin / G, (b + 1) * nwin / G) (s.wbal, A/B option).  The
// fire's block-local bitmap (wheel_fire) covers the same slab.  ileave: round-robin chunks instead.
__host__ __device__ __forceinline__ void block_windows(const Dev& s, unsigned vb, unsigned nwin, unsigned& wlo,
                                                       unsigned& whi, unsigned& rounds) {
  const unsigned G = s.nblocks;
  if (s.ileave) {
    rounds = (nwin + G * WARPS - 1) / (G * WARPS);
    wlo = 0;
    whi = nwin;
  } else if (s.wbal) {
    wlo = (unsigned)((unsigned long long)nwin * vb / G);
    whi = (unsigned)((unsigned long long)nwin * (vb + 1) / G);
    rounds = (whi - wlo + WARPS - 1) / WARPS;
  } else {
    const unsigned r0 = (nwin + G * WARPS - 1) / (G * WARPS);
    wlo = min(nwin, vb * r0 * WARPS);
    whi = min(nwin, wlo + r0 * WARPS);
    rounds = r0;
  }
}

template <int D, bool WHEEL_ENGINE, bool PEER = false, bool W = false>
__device__ void phase_treat(const Dev& s, const View& v, Smem& sm) {
  Acc* acc = &s.ctl->acc[v.c % NACC];
  const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const unsigned nwin = (s.nwords + s.win_words - 1) / s.win_words;
  // every block owns one contiguous slab of windows: its phantoms / events come from a
  // compact region of the grid, so a run's destinations share sectors and L2 lines (block_windows;
  // the balanced split, which gives every block work on C2, measured neutral on C3 and 1.5 % slower
  // on C2, is an A/B option).
  const unsigned vb = blockIdx.x - s.blk0;
  unsigned wlo, whi, rounds;
  block_windows(s, vb, nwin, wlo, whi, rounds);
  // first window of round r: the block's slab, or (s.ileave, A/B option) round r of every block
  // inside one chunk of nblocks * WARPS windows
  auto rwin = [&](unsigned r) -> unsigned { return s.ileave ? (r * s.nblocks + vb) * WARPS : wlo + r * WARPS; };
  unsigned dmin = 0xFFFFFFFFu;
  unsigned created = 0, relabels = 0, triggered = 0, lanes_started = 0, tested = 0;   // per thread, this cycle
#if WCSP_TREAT_STAGE
  if (threadIdx.x == 0) sm.stg_n = 0;   // nothing staged until a dense round stages its band
#endif
  if constexpr (WHEEL_ENGINE) {
    for (unsigned d = threadIdx.x; d < WHEEL; d += THREADS) {
      sm.rcap[d] = 0; sm.rfill[d] = 0; sm.ofill[d] = 0;
#if WCSP_WARP_FLUSH
      sm.rlock[d] = 0;
#endif
    }
#if WCSP_WARP_FLUSH
    if (threadIdx.x < WARPS) sm.wnp[threadIdx.x] = 0;
#endif
    __syncthreads();
  }
  bool scan = true;
  if constexpr (WHEEL_ENGINE) {
    if (!s.slab && v.lmode) {      // sparse cycle: the cycle's triggered list, then the bitmap if needed
      // batch k (32 vertices) of the global list goes to warp k / G of block k % G: a thin front's
      // few hundred or thousand triggered vertices spread over the whole grid of blocks instead of
      // queueing in the blocks whose fire found them (C4 cycles: one batch latency)
      const unsigned total = __ldcg(&acc->tl_total);
      for (unsigned k = warp * s.nblocks + vb; k * 32u < total; k += s.nblocks * WARPS) {
        const unsigned i = k * 32u + lane;
        const unsigned q = i < total ? __ldcg(s.tlist + i) : 0xFFFFFFFFu;
        treat_one<D, WHEEL_ENGINE, PEER>(s, v, sm, acc, q, dmin, created, relabels, triggered, lanes_started, tested);
      }
      scan = __ldcg(&acc->tl_over) != 0;
#if WCSP_FLUSH_LAZY > 0 && !WCSP_WARP_FLUSH
      __syncthreads();
      if (sm.np > (unsigned)WCSP_FLUSH_LAZY) ev_flush(s, sm, v.t, v.region, false);
#endif
    }
  }
#if WCSP_ROUND_SHARE && WCSP_FLUSH_LAZY > 0 && !WCSP_WARP_FLUSH
  if constexpr (WHEEL_ENGINE) {
    unsigned short* flat = &sm.wl[0][0];
    const unsigned ww = s.win_words;
#if WCSP_WIN_PREFETCH
    unsigned raw = scan && rounds > 0 ? window_load(s, rwin(0) + warp, whi) : 0u;
#else
    unsigned bits = scan && rounds > 0 ? window_bits(s, rwin(0) + warp, whi) : 0u;
#endif
    for (unsigned r = 0; scan && r < rounds; ++r) {
#if WCSP_WIN_PREFETCH
      const unsigned bits = window_use(s, rwin(r) + warp, raw);
#endif
      const unsigned cnt = __reduce_add_sync(0xFFFFFFFFu, (unsigned)__popc(bits));
      if (lane == 0) sm.wtot[warp] = cnt;
      __syncthreads();
      if (sm.np > (unsigned)WCSP_FLUSH_LAZY) ev_flush(s, sm, v.t, v.region, false);   // uniform
      unsigned base = 0, T = 0;
#pragma unroll
      for (unsigned i = 0; i < (unsigned)WARPS; ++i) {
        const unsigned t = sm.wtot[i];
        base += i < warp ? t : 0u;
        T += t;
      }
      window_emit(s, bits, base, flat, warp * ww * 32u);
#if WCSP_CLAIM
      if (threadIdx.x == 0) sm.claim = WARPS * 32u;   // batch w goes to warp w first, then first come
#endif
#if WCSP_TREAT_STAGE
      if constexpr (!PEER) {
        if (threadIdx.x == 0) {          // the round's band (+ one axis-1 stride each side), if it fits
          const unsigned rb = rwin(r) * ww * 32u, H = s.NL >= 4 ? s.off[2] : 1u;
          const unsigned lo = (rb >= H ? rb - H : 0u) & ~1u;
          const unsigned hi = (unsigned)min((unsigned long long)s.N, (unsigned long long)rb + ww * 32u * WARPS + H);
          const unsigned n = (hi - lo + 1u) & ~1u;
          const bool ok = T > 0 && n <= (unsigned)WCSP_STAGE_WORDS && lo + n <= ((s.N + 1u) & ~1u);
          sm.stg_lo = lo;
          sm.stg_n = ok ? min(n, s.N - lo) : 0u;
          if (ok) stage_issue(s, sm, lo, n);
        }
      }
#endif
      __syncthreads();
#if WCSP_TREAT_STAGE
      if constexpr (!PEER) {
        if (sm.stg_n) { stage_wait(sm, sm.stg_phase & 1u); }
        __syncthreads();
        if (threadIdx.x == 0 && sm.stg_n) sm.stg_phase += 1;
      }
#endif
#if WCSP_WIN_PREFETCH
      if (r + 1 < rounds) raw = window_load(s, rwin(r + 1) + warp, whi);   // next round in flight
#else
      if (r + 1 < rounds) bits = window_bits(s, rwin(r + 1) + warp, whi);
#endif
      const unsigned rbase = rwin(r) * ww * 32u;
#if WCSP_CLAIM
      // a warp that finishes its batch takes the next unclaimed one (shared-memory counter), so the
      // round ends when the work does rather than when the unluckiest warp's fixed share does
      for (unsigned b = warp * 32; b < T;) {
        const unsigned q = b + lane < T ? rbase + flat[b + lane] : 0xFFFFFFFFu;
        treat_one<D, WHEEL_ENGINE, PEER>(s, v, sm, acc, q, dmin, created, relabels, triggered, lanes_started, tested);
        unsigned nb = 0;
        if (lane == 0) nb = atomicAdd(&sm.claim, 32u);
        b = __shfl_sync(0xFFFFFFFFu, nb, 0);
      }
#else
      for (unsigned b = warp * 32; b < T; b += WARPS * 32) {
        const unsigned q = b + lane < T ? rbase + flat[b + lane] : 0xFFFFFFFFu;
#if WCSP_TREAT_PF
        {   // the warp's next batch: its first dependent loads start now, one batch ahead
          const unsigned bn = b + WARPS * 32 + lane;
          if (bn < T) {
            const unsigned qn = rbase + flat[bn];
            asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(s.sw + qn));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(reinterpret_cast<const char*>(s.wt) +
                                                      (size_t)qn * 2 * sizeof(typename Tr<D>::LW)));
          }
        }
#endif
        treat_one<D, WHEEL_ENGINE, PEER>(s, v, sm, acc, q, dmin, created, relabels, triggered, lanes_started, tested);
      }
#endif
    }
    scan = false;
  }
#endif
  for (unsigned r = 0; scan && r < rounds; ++r) {
    const unsigned win = rwin(r) + warp;
    const unsigned total = win < whi ? window_take(s, win, sm.wl[warp]) : 0u;
    for (unsigned b = 0; b < total; b += 32) {
      const unsigned q = b + lane < total ? win * s.win_words * 32u + sm.wl[warp][b + lane] : 0xFFFFFFFFu;
      treat_one<D, WHEEL_ENGINE, PEER, W>(s, v, sm, acc, q, dmin, created, relabels, triggered, lanes_started, tested);
    }
    if constexpr (WHEEL_ENGINE) {
#if WCSP_WARP_FLUSH
      // nothing: every warp files its own events as its staging fills
#elif WCSP_FLUSH_LAZY > 0
      __syncthreads();             // flush only when the staging is half full (fewer block-wide sorts)
      if (sm.np > (unsigned)WCSP_FLUSH_LAZY) ev_flush(s, sm, v.t, v.region, false);
#elif WCSP_FLUSH_LAZY == 0
      ev_flush(s, sm, v.t, v.region, false);
#endif                             // < 0: no block barrier between rounds; overflow spills, one flush at the end
    } else if constexpr (W) {
      qflush<PhW>(sm, &acc->n_act, s.act[v.cur ^ 1], &acc->n_pool, reinterpret_cast<PhW*>(s.pool[v.cur ^ 1]), s.pool_cap);
    } else {
      qflush(sm, &acc->n_act, s.act[v.cur ^ 1], &acc->n_pool, s.pool[v.cur ^ 1], s.pool_cap);
    }
  }
  if constexpr (WHEEL_ENGINE) {
#if WCSP_WARP_FLUSH
    warp_flush(s, sm, v.t, v.region);
    regions_close(s, sm, v.t);
#else
    ev_flush(s, sm, v.t, v.region, true);
#endif
  }
  block_reduce_commit(sm, dmin, 0, 0, created, relabels, triggered, acc, lanes_started, tested);
}

// ---------------------------------------------------------------------------
// decide (sweep engine): Step 6 + time skipping.  One thread; writes ctl if writer.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void reset_acc(Acc* a) {
  a->n_act = 0; a->n_pool = 0; a->tl_over = 0; a->tl_total = 0; a->dmin = 0xFFFFFFFFu;
  a->bhit = 0; a->live = 0; a->arrivals = 0; a->created = 0; a->relabels = 0; a->triggered = 0;
  a->started = 0; a->tested = 0; a->pend_lanes = 0; a->pend_phantoms = 0;
  a->nfire = 0;
}

__device__ __forceinline__ void resolve_hit(const Dev& s, unsigned long long bhit, long long t, unsigned c) {
  Ctl* C = s.ctl;
  const unsigned q = (unsigned)(bhit >> 32);
  const unsigned X = 0xFFFFFFFFu - (unsigned)bhit;
  // Y = smallest source among cycle c's arrivals at X carrying q; a regular edge wins over a phantom (R5)
  const unsigned par = c & 1u;
  const unsigned nb = min(__ldcg(&C->n_barr2[par]), s.barr_cap);
  unsigned long long best = ~0ull;
  for (unsigned k = 0; k < nb; ++k) {
    const BArr b = s.barr[(size_t)par * s.barr_cap + k];
    if (b.D == X && b.cand == q) best = min(best, ((unsigned long long)b.src << 1) | b.via);
  }
  C->F1 = t;
  C->F2 = s.minf ? -1 : (long long)s.M - q;
  C->X = X;
  C->ybest = best;                 // slab engine: the host takes the min over slabs
  C->Y = best == ~0ull ? -1 : (long long)(best >> 1);
  C->via = (long long)(best & 1);
}

__device__ void decide(const Dev& s, View& v, bool writer) {
  Acc* a = &s.ctl->acc[v.c % NACC];
  const unsigned long long bhit = __ldcg(&a->bhit);
  const unsigned n_act = __ldcg(&a->n_act), n_pool = __ldcg(&a->n_pool), dmin = __ldcg(&a->dmin);
  View nv = v;
  Ctl* C = s.ctl;
  if (writer) {
    const unsigned long long live = __ldcg(&a->live), arrivals = __ldcg(&a->arrivals);
    const unsigned long long created = __ldcg(&a->created), relabels = __ldcg(&a->relabels);
    const unsigned long long triggered = __ldcg(&a->triggered);
    C->started += (long long)__ldcg(&a->started);
    if (v.c > 0) {
      C->cycles += 1;
      C->edge_updates += (long long)(live + v.n_pool);
      if ((long long)v.c - 1 < s.trace_cap) {
        const unsigned long long t2 = globaltimer_ns();
        TraceRec r{v.t, (long long)v.delta, (long long)v.n_act, (long long)live, (long long)v.n_pool,
                   (long long)triggered, (long long)arrivals, (long long)created, (long long)relabels,
                   (long long)__ldcg(&a->tested), (long long)(C->ts1 - C->ts0), (long long)(t2 - C->ts1), 0, 0};
        s.trace[v.c - 1] = r;
      }
    }
    C->arrivals += arrivals; C->triggered += triggered; C->created += created; C->relabels += relabels;
  }
  if (bhit) {
    nv.status = 0;  // WCSP_REACHED
    if (writer) resolve_hit(s, bhit, v.t, v.c);
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
// grid barrier for the cooperative persistent kernels (monotone counter)
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Returns false if the barrier was abandoned (watchdog: a block missing for
// BARRIER_TIMEOUT_NS sets ctl->abort; every waiting block then gives up).
constexpr unsigned long long BARRIER_TIMEOUT_NS = 20ull * 1000000000ull;

#ifndef WCSP_BAR_SLEEP
#define WCSP_BAR_SLEEP 32          // ns between polls of the grid barrier
#endif
#ifndef WCSP_BAR_RELEASE
#define WCSP_BAR_RELEASE 0         // 1: the last arriver releases a flag on its own line (measured: C2 +8 %; off)
#endif
__device__ __forceinline__ void st_release_gpu(unsigned long long* p, unsigned long long x) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(x) : "memory");
}
__device__ __forceinline__ bool grid_sync(Ctl* ctl, unsigned long long target, Smem& sm,
                                          unsigned long long* fin = nullptr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (fin) {                     // block busy time in this phase: max and sum over blocks
      const unsigned long long busy = globaltimer_ns() - sm.tphase;
      atomicMax(fin, busy);
      atomicAdd(fin + 1, busy);
    }
    __threadfence();
#if WCSP_BAR_RELEASE
    // arrivals count on ctl->bar; the last one publishes the release on a line of its own
    if (atomicAdd(&ctl->bar, 1ull) == target - 1) {
      __threadfence();
      st_release_gpu(&ctl->grel, target);
    }
    unsigned long long* const poll = &ctl->grel;
#elif WCSP_BAR_GROUPS > 1
    // two-level arrival: blocks count on one of WCSP_BAR_GROUPS lines; the last of each group adds
    // the group's size to ctl->bar (fewer same-address atomics serialised at one L2 slice)
    {
      const unsigned NGp = WCSP_BAR_GROUPS, G = gridDim.x, g = blockIdx.x % NGp;
      const unsigned long long gk = (G - g + NGp - 1) / NGp;          // blocks in group g
      const unsigned long long epoch = target / G;
      if (atomicAdd(&ctl->bsub[g][0], 1ull) == epoch * gk - 1) {
        __threadfence();
        atomicAdd(&ctl->bar, gk);
      }
    }
    unsigned long long* const poll = &ctl->bar;
#else
    atomicAdd(&ctl->bar, 1ull);
    unsigned long long* const poll = &ctl->bar;
#endif
    const unsigned long long t0 = globaltimer_ns();
    unsigned ok = 1;
    while (ld_acquire(poll) < target) {
      if (WCSP_BAR_SLEEP > 0) __nanosleep(WCSP_BAR_SLEEP);
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
    x.n_pool = g->n_pool; x.cur = g->cur; x.status = g->status; x.region = g->region; x.lmode = g->lmode;
    x.ncount = g->ncount; x.pad_ = g->pad_;
    sm.view = x;
  }
  __syncthreads();
  v = sm.view;
}

__device__ __forceinline__ void init_smem(Smem& sm) {
  if (threadIdx.x == 0) { sm.na = 0; sm.np = 0; sm.nspill = 0; sm.ovf = 0; sm.alloc_lim = ~0ull; sm.f_prep = 0; sm.f_nd = 0; }
#if WCSP_TREAT_STAGE
  if (threadIdx.x == 0) {
    sm.stg_n = 0; sm.stg_lo = 0; sm.stg_phase = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sm.stg_bar)) : "memory");
  }
#endif
  __syncthreads();
}

// Forget every temp (keeps the target / removed sentinels): used when the
// 16-bit cycle stamps wrap.
template <bool W = false>
__device__ __forceinline__ void clear_temps(const Dev& s) {
  for (unsigned long long i = (unsigned long long)blockIdx.x * THREADS + threadIdx.x; i < s.N;
       i += (unsigned long long)gridDim.x * THREADS) {
    if constexpr (W) {
      if ((s.sw[i] >> 32) != 0xFFFFFFFFull) s.sw[i] = 0ull;
    } else {
      unsigned* t = tmp_ptr(s.sw, (unsigned)i);
      if ((*t >> 16) != 0xFFFFu) *t = 0u;
    }
  }
}

// ---------------------------------------------------------------------------
// kernels (sweep engine)
// ---------------------------------------------------------------------------
template <int D, bool W = false>   // W: wide labels (M > WCSP_M_MAX)
__global__ void __launch_bounds__(THREADS, WCSP_MINB_SWEEP) k_persistent(Dev s) {
  Smem& sm = smem();
  init_smem(sm);
  View v;
  load_view(s, sm, v);
  const unsigned long long G = gridDim.x;
  unsigned long long target = 0;
  while (v.status == ST_RUNNING) {
    if (v.c > 0) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        reset_acc(&s.ctl->acc[(v.c + 1) % NACC]);
        s.ctl->ts0 = globaltimer_ns();
      }
      phase_sweep<D, W>(s, v, sm);
      target += G;
      if (!grid_sync(s.ctl, target, sm)) return;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) s.ctl->ts1 = globaltimer_ns();
    if (threadIdx.x == 0) sm.bhit = __ldcg(&s.ctl->acc[v.c % NACC].bhit);
    __syncthreads();
    const unsigned long long bhit = sm.bhit;
    __syncthreads();
    if (!bhit) {                                   // S5 precedes S6: the final cycle skips the treat
      phase_treat<D, false, false, W>(s, v, sm);
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
      clear_temps<W>(s);
      target += G;
      if (!grid_sync(s.ctl, target, sm)) return;
    }
  }
}

template <int D, bool W = false>
__global__ void __launch_bounds__(THREADS, WCSP_MINB_SWEEP) k_sweep(Dev s) {
  Smem& sm = smem();
  init_smem(sm);
  View v;
  load_view(s, sm, v);
  if (v.status != ST_RUNNING || v.c == 0) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    reset_acc(&s.ctl->acc[(v.c + 1) % NACC]);
    s.ctl->ts0 = globaltimer_ns();
  }
  phase_sweep<D, W>(s, v, sm);
}

template <int D, bool W = false>
__global__ void __launch_bounds__(THREADS, WCSP_MINB_SWEEP) k_treat(Dev s) {
  Smem& sm = smem();
  init_smem(sm);
  View v;
  load_view(s, sm, v);
  if (v.status != ST_RUNNING) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) s.ctl->ts1 = globaltimer_ns();
  if (__ldcg(&s.ctl->acc[v.c % NACC].bhit)) return;
  phase_treat<D, false, false, W>(s, v, sm);
}

__global__ void k_decide(Dev s) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  View v = s.ctl->view;
  if (v.status != ST_RUNNING) return;
  decide(s, v, true);
  if (v.status == ST_RUNNING && v.stamp == 1u) s.ctl->view.status = ST_WRAP;
}

template <bool W = false>
__global__ void __launch_bounds__(THREADS) k_clear_temps(Dev s) { clear_temps<W>(s); }

// Initial state (reading R20): L = 0 everywhere, target /
// removed sentinels, no live lane, A triggered with temp M (the treat of
// c = 0 then sets L = M on A and starts its lanes).
__global__ void __launch_bounds__(THREADS) k_init(Dev s, const uint8_t* maskA, const uint8_t* maskB,
                                                  const uint8_t* present, const uint8_t* ghost, int lblA,
                                                  int d) {
  const unsigned N = s.N;
  for (unsigned long long i = (unsigned long long)blockIdx.x * THREADS + threadIdx.x; i < N;
       i += (unsigned long long)gridDim.x * THREADS) {
    const bool p = present ? present[i] != 0 : true;
    const bool a = p && maskA[i] && !(ghost && ghost[i]);
    const bool b = p && maskB[i];
    if (s.wide) {                   // wide labels: L in lab[], temp = stamp:32 | cand:32 in sw[]
      s.lab[i] = p ? 0u : LBL_REMOVED_W;
      s.sw[i] = !p ? TMPW_REMOVED : b ? TMPW_B : a ? (((unsigned long long)stamp_of(0) << 32) | (unsigned)lblA) : 0ull;
    } else {
      unsigned lbl = 0, tmp = 0;
      if (!p) { lbl = LBL_REMOVED; tmp = TMP_REMOVED; }
      else if (ghost && ghost[i]) { lbl = 0; tmp = ghost[i] == 2 ? TMP_GHOST_B : TMP_GHOST; }   // slab engine
      else if (b) { lbl = 0; tmp = TMP_B; }
      else if (a) { lbl = 0; tmp = (stamp_of(0) << 16) | (unsigned)lblA; }
      s.sw[i] = ((unsigned long long)tmp << 32) | lbl;
    }
    if (s.res) {
      if (d <= 2) reinterpret_cast<uint32_t*>(s.res)[i] = 0u;
      else reinterpret_cast<unsigned long long*>(s.res)[i] = 0ull;
    }
  }
  // triggered bitmap = A
  for (unsigned long long w = (unsigned long long)blockIdx.x * THREADS + threadIdx.x; w < s.nwords;
       w += (unsigned long long)gridDim.x * THREADS) {
    unsigned bits = 0;
    for (unsigned b = 0; b < 32; ++b) {
      const unsigned long long i = w * 32 + b;
      if (i < N && maskA[i] && (present ? present[i] != 0 : true) && !maskB[i] && !(ghost && ghost[i]))
        bits |= 1u << b;
    }
    s.tbits[w] = bits;
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

// Validation counters (wcsp.h rules): [0] |A|, [1] |B|, [2] |A n B|, [3] present edges with f2 = 0,
// [4] max f1 over present edges.
__global__ void __launch_bounds__(THREADS) k_validate(unsigned long long N, int d, long long n0, long long n1,
                                                      long long n2, long long n3, const uint8_t* f1,
                                                      const uint8_t* f2, const uint8_t* maskA,
                                                      const uint8_t* maskB, const uint8_t* present,
                                                      unsigned long long* out) {
  const long long n[4] = {n0, n1, n2, n3};
  unsigned long long c[4] = {0, 0, 0, 0};
  unsigned fmax = 0;
  for (unsigned long long v = (unsigned long long)blockIdx.x * THREADS + threadIdx.x; v < N;
       v += (unsigned long long)gridDim.x * THREADS) {
    const bool p = present ? present[v] != 0 : true;
    const bool a = p && maskA[v], b = p && maskB[v];
    c[0] += a; c[1] += b; c[2] += a && b;
    unsigned long long stride = 1;
    for (int k = 0; k < d; ++k) {
      const unsigned long long xk = (v / stride) % (unsigned long long)n[k];
      if (xk + 1 < (unsigned long long)n[k]) {
        c[3] += (f1[k * N + v] != 0 && f2[k * N + v] == 0);
        fmax = max(fmax, (unsigned)f1[k * N + v]);
      }
      stride *= (unsigned long long)n[k];
    }
  }
  for (int i = 0; i < 4; ++i)
    if (c[i]) atomicAdd(out + i, c[i]);
  if (fmax) atomicMax(out + 4, (unsigned long long)fmax);
}

}  // namespace wcspk
