// sim.cu — device-resident lockstep event loop (north-star kernel 4).
//
// Reference: oracle.simulate / _plan (pkg/src/timewarp/oracle.py:49-180), the exact
// CPU timeline the live stack must match event-for-event
// (pkg/tests/test_harness_integration.py:77-83).
//
// Design:
//  * persistent kernel; each warp pulls whole configs from a device work counter in
//    host-sorted (largest-first) order and runs that config's loop to completion;
//  * the config's active list lives in the warp's slice of shared memory as SoA
//    int32 arrays (request index, prompt, output, done_prefill, emitted, plan), in
//    admission order; lane i of round r owns slot 32r+i;
//  * _plan's order-sensitive budget rules become warp scans: decode cutoff = ballot
//    rank, chunk takes = exclusive int64 scan of min(chunk, remaining), FCFS
//    admission with head-of-line blocking = count of leading lanes whose running
//    (budget, KV, slot) constraints hold;
//  * features P/D/C are REDUX sums, the prediction is the warp-uniform exact-fp64
//    predictor over the TMA-staged calibration blob in shared memory;
//  * virtual time advances through the config's Timekeeper min-advance (dispatcher +
//    TP x PP workers, BarrierCore rules on a FakeClock);
//  * decode-only runs are macro-stepped: while no request finishes and no arrival
//    can be admitted, every step decodes the same D requests with the same predicted
//    duration, so the run length is closed-form (min remaining outputs, first
//    arrival crossing) and the run's K*D token events are hashed in parallel across
//    the lanes instead of K serial plan/apply passes ("macro steps");
//  * every token event is hashed into a position-bound digest (tw_event_hash, linear in
//    position/time/step per request, so a run's body sums in closed form) and
//    FIRST_TOKEN / FINISHED stamps are stored per request; full event dumps only
//    for audited configs.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace twb {

// Phase boundaries of the event loop. With -DTWB_PROFILE_PHASES they read the SM clock
// (scripts/prof_sim.py); otherwise they are compiler memory barriers: keeping ptxas from
// moving shared/global accesses across phases measured 14% faster on the 1,024-config
// sweep than letting it schedule freely (15.6 -> 13.4 ms; profiles/README.md).
#if defined(TWB_PROFILE_PHASES)
#define TWB_CLK() clock64()
#else
__device__ __forceinline__ long long twb_phase_barrier() {
  asm volatile("" ::: "memory");
  return 0LL;
}
#define TWB_CLK() twb_phase_barrier()
#endif

// Code placement: the event loop's SASS (~4.5 k instructions) exceeds the instruction
// caches, but moving the rare or duplicated paths (prediction-cache misses, the
// Timekeeper walk) out of line measured slower (A/B 13.4 ms inline vs 14.2 / 15.5 ms;
// profiles/README.md), so they stay inlined unless these switches are set.
#ifdef TWB_SIM_OUTLINE_PRED
#define TWB_PRED_FN static __device__ __noinline__
#else
#define TWB_PRED_FN __device__ __forceinline__
#endif
#ifdef TWB_SIM_OUTLINE_TK
#define TWB_TK_FN static __device__ __noinline__
#else
#define TWB_TK_FN __device__ __forceinline__
#endif

#ifndef TWB_SIM_WARPS
#define TWB_SIM_WARPS 4
#endif
constexpr int kSimThreads = 32 * TWB_SIM_WARPS;  // warps per CTA (one config per warp at a time)
constexpr int kSimWarps = kSimThreads / 32;
constexpr int kMaxSlotCap = 4096;
constexpr int kLatencyConfigsPerSm = 8;  // tw_sim_many: up to 8 configs per SM -> latency variant

struct SimParams {
  const void* pset;
  uint32_t pset_bytes;
  uint32_t pset_smem;  // bytes reserved for the blob (multiple of 128)
  const tw_sim_cfg* cfgs;
  int32_t n_cfg;
  const int32_t* order;
  const int64_t* wl_off;
  const int64_t* ts;
  const int32_t* prompt;
  const int32_t* output;
  tw_sim_result* res;
  const int64_t* req_base;
  int64_t* first;
  int64_t* finish;
  const int64_t* ev_off;
  tw_event* ev;
  int32_t* counter;
  int32_t cap;
  int64_t* prof;  // optional: 16 int64 per config (tw_sim_set_profile)
  int32_t* gslots;  // slot state in global memory (capacities above kMaxSlotCap; sim_big.cu)
  int32_t* checks;  // sim_check.cu only: 8 invariant counters per config (tw_sim_set_checks)
};

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// int64 warp sum of non-negative values < 2^50 per lane, with two REDUX ops
__device__ __forceinline__ int64_t warp_sum_i64_redux(int64_t v) {
  const unsigned lo = (unsigned)(v & 0xffffff);
  const unsigned hi = (unsigned)(v >> 24);
  const unsigned sl = __reduce_add_sync(kFull, lo);
  const unsigned sh = __reduce_add_sync(kFull, hi);
  return ((int64_t)sh << 24) + (int64_t)sl;
}
// Inclusive saturating scan of non-negative int32 counts (token takes, KV blocks):
// partial sums clamp at INT32_MAX. Every decision compares an exclusive prefix against a
// budget or free-block count <= INT32_MAX, and a clamped prefix is >= that bound exactly
// when the true one is, so the decisions equal the exact 64-bit scan's (and totals of
// admitted prefixes, which stay below the bound, are exact). 32-bit shuffles, less code.
__device__ __forceinline__ int32_t warp_incl_scan_sat(int32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t w = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v = (int32_t)min((uint32_t)v + (uint32_t)w, 0x7fffffffu);
  }
  return v;
}
__device__ __forceinline__ int32_t warp_excl_from_incl(int32_t incl) {
  const int32_t e = __shfl_up_sync(kFull, incl, 1);
  return (threadIdx.x & 31) ? e : 0;
}

// a / b for a >= 0, b > 0. (A hand-made 32-bit fast path measured 13% slower than
// the compiler's 64-bit routine, which already short-cuts small operands; a variant
// that moved the Timekeeper rounds to a partner warp behind a shared-memory ring
// measured 10-18% slower than keeping them inline — see profiles/README.md.)
__device__ __forceinline__ int64_t div_nn(int64_t a, int64_t b) { return a / b; }

// Cold paths kept out of line: the loop's SASS is larger than the instruction caches
// and the kernel is fetch-sensitive (adding inline code to the hot loop measured
// slower even when it removed work), so rarely taken code should not sit inside it.
#ifdef TWB_SIM_INLINE_COLD
#define TWB_COLD static __device__ __forceinline__
#else
#define TWB_COLD static __device__ __noinline__  // static: sim.cu is compiled twice (sim_tput.cu)
#endif
TWB_COLD int64_t cold_div(int64_t a, int64_t b) { return a / b; }
TWB_COLD int64_t cold_fake_sleep(int64_t wait_ns) { return fake_sleep_ns(wait_ns); }
#ifdef TWB_SIM_COLD_DIV_ALL
#define HOT_DIV cold_div
#else
#define HOT_DIV div_nn
#endif

// floor(a / b) for 0 <= a < 2^52 and b > 0 given rb ~= 1/b (any fp64 approximation):
// the fp64 estimate is within 2 of the quotient, fixed up with exact int64 checks.
__device__ __forceinline__ int64_t div_rcp(int64_t a, int64_t b, double rb) {
  if (a >= (1LL << 52)) return cold_div(a, b);
  int64_t q = (int64_t)__dmul_rz(__ll2double_rn(a), rb);
  int64_t r = a - q * b;
  while (r < 0) { q--; r += b; }
  while (r >= b) { q++; r -= b; }
  return q;
}

// ceil(t / bk) for 0 <= t < 2^31 with a per-config magic reciprocal (no IDIV chain):
// q0 = umulhi(t, floor((2^32-1)/bk)) is at most 2 below floor(t/bk).
struct Blocks {
  uint32_t bk, magic;
  __device__ __forceinline__ void init(uint32_t b) {
    bk = b;
    magic = 0xffffffffu / b;
  }
  __device__ __forceinline__ int32_t ceil_div(int32_t t) const {  // oracle.py:39-40
    if (t <= 0) return 0;
    uint32_t q = __umulhi((uint32_t)t, magic);
    uint32_t r = (uint32_t)t - q * bk;
    if (r >= bk) { q++; r -= bk; }
    if (r >= bk) { q++; r -= bk; }
    return (int32_t)(q + (r != 0u));
  }
};

struct Slots {
  int32_t* req;
  int32_t* prompt;
  int32_t* output;
  int32_t* done;
  int32_t* emit;
  int32_t* plan;   // >= 0 chunk tokens, -1 decode, -2 idle (this step)
  int32_t* dlist;  // this step's decode slots in order (rank -> slot)
};

// Lane-distributed window over a workload's arrival offsets: lane l holds
// epoch + ts[base + l] (INT64_MAX past the end); one coalesced load per 32 arrivals.
struct ArrWindow {
  int32_t base;
  int64_t v;
  __device__ __forceinline__ void load(const int64_t* __restrict__ ts, int32_t n, int64_t epoch, int32_t b) {
    const int lane = threadIdx.x & 31;
    base = b;
    v = (b + lane < n) ? epoch + __ldg(ts + b + lane) : INT64_MAX;
  }
  // uniform idx < n
  __device__ __forceinline__ int64_t get(const int64_t* __restrict__ ts, int32_t n, int64_t epoch, int32_t idx) {
    if (idx - base >= 32) load(ts, n, epoch, idx);
    return __shfl_sync(kFull, v, idx - base);
  }
};

// Per-config Timekeeper actor grid: actor 0 is the dispatcher,
// actors 1..TP*S the WorkerGrid cells; BarrierCore rules on a FakeClock. Each round's
// t_min is the min over the eligible actors' pending targets, which reduces to
// min(dispatcher's next arrival, current stage deadline) because the TP ranks of a
// stage share its deadline and parked workers are exempt.
struct TkGrid {
  int64_t wall, offset, seq, last_bcast, V, cooldown, conv_cooldown;
  double rcp_cooldown;
  int64_t disp_ts;
  int32_t disp;
  ArrWindow win;
  // speculative segments (kSpec): the run started from a guessed wall clock; a true run
  // whose wall is this one's + delta takes the same decisions iff d_lo <= delta < d_hi
  int64_t d_lo, d_hi;
#ifdef TWB_PROFILE_PHASES
  int64_t prof_calls, prof_fast, prof_loops;
#endif
};

// The Timekeeper's decisions depend on its FakeClock wall only through `wall < t_min` and
// `offset >= cJ` (sleeps use last_bcast - wall, broadcasts set offset = t_min - wall, so
// V = wall + offset and everything else move with V alone). A speculative segment records,
// for each such comparison, the range of wall shifts delta that keep its outcome.
template <bool kSpec>
__device__ __forceinline__ bool tk_wall_lt(TkGrid& g, int64_t t) {
  const bool r = g.wall < t;
  if constexpr (kSpec) {  // wall + delta < t  <=>  delta < t - wall
    const int64_t m = t - g.wall;
    if (r) g.d_hi = min(g.d_hi, m);
    else g.d_lo = max(g.d_lo, m);
  }
  return r;
}
template <bool kSpec>
__device__ __forceinline__ bool tk_off_ge(TkGrid& g, int64_t cj) {
  const bool r = g.offset >= cj;
  if constexpr (kSpec) {  // offset - delta >= cj  <=>  delta < offset - cj + 1
    const int64_t m = g.offset - cj + 1;
    if (r) g.d_hi = min(g.d_hi, m);
    else g.d_lo = max(g.d_lo, m);
  }
  return r;
}

template <bool kSpec = false>
__device__ __forceinline__ void tk_resolve(TkGrid& g, int64_t t_min) {
  // timekeeper.py:326-366 with FakeClock sleep (pkg/tests/_support.py:33-34)
  if (tk_wall_lt<kSpec>(g, t_min) && g.last_bcast != INT64_MIN && g.cooldown > 0) {
    const int64_t wait = g.last_bcast + g.cooldown - g.wall;
    if (wait > 0) g.wall += (wait == g.cooldown) ? g.conv_cooldown : cold_fake_sleep(wait);
  }
  if (tk_wall_lt<kSpec>(g, t_min)) {
    const int64_t cand = t_min - g.wall;
    if (cand > g.offset) g.offset = cand;
    g.seq++;
    g.last_bcast = g.wall;
  }
  g.V = g.wall + g.offset;
}

__device__ __forceinline__ void tk_dispatch(TkGrid& g, const int64_t* __restrict__ ts, int32_t n, int64_t epoch) {
  while (g.disp_ts <= g.V) {  // the dispatcher passes every arrival <= V (runner.py:94-124)
    g.disp++;
    g.disp_ts = g.disp < n ? g.win.get(ts, n, epoch, g.disp) : INT64_MAX;
  }
}

// K consecutive steps of duration d from now0 through the Timekeeper (a macro run, or
// K = 1 for a normal step). The deadlines form a fixed pattern per step (stage s ends
// at base + per*(s+1), the last at base + d), so the walk keeps (step k, stage s) and
// only resolves targets beyond V; a V that jumped several steps ahead (the FakeClock
// wall outrunning short steps) is skipped in O(1). Each resolve is one BarrierCore
// round with t_min = min(dispatcher's next arrival, the stage deadline).
template <bool kSpec = false>
TWB_TK_FN void tk_run(TkGrid& g, const int64_t* __restrict__ ts, int32_t n, int64_t epoch,
                                       int S, int64_t now0, int64_t d, int64_t K) {
  // deadline m (m >= 1) of this run: now0 + (m / S) * d + per * (m % S); m = 0 is now0
#ifdef TWB_PROFILE_PHASES
  g.prof_calls++;
#endif
#if !defined(TWB_SIM_TPUT_TU) || defined(TWB_TPUT_TK_FAST)
  // One or two stages, steady state on the run's start (every stage gap > cJ), no
  // dispatcher target inside the run: the K*S deadlines each resolve as sleep cJ +
  // broadcast, which is the loop's steady-state closed form with R = K*S, without the
  // walk (latency variant only: 1,024 configs 8.57 -> 8.31 ms for S = 1, 8.37 -> 8.08 ms
  // with S = 2; in the throughput variant the extra code measured 289 -> 296 ms).
  if (S <= 2 && g.V == now0 && g.last_bcast == g.wall && (S == 1 ? d : d >> 1) > g.conv_cooldown &&
      g.disp_ts > now0 + K * d) {
    const int64_t end1 = now0 + K * d, R = K * S;
    g.wall += R * g.conv_cooldown;
    g.seq += R;
    g.last_bcast = g.wall;
    g.offset = end1 - g.wall;
    g.V = end1;
#ifdef TWB_PROFILE_PHASES
    g.prof_fast++;
#endif
    return;
  }
  // Wall-bound state (every stage gap <= cJ <= offset): the loop's first closed form,
  // then the dispatcher catches up (the walk's second pass).
  if (S <= 2 && g.last_bcast == g.wall && g.conv_cooldown > 0 && d > 0 && tk_off_ge<kSpec>(g, g.conv_cooldown) &&
      (S == 1 ? d : d - (d >> 1)) <= g.conv_cooldown && g.V < now0 + K * d) {
    const int64_t cj1 = g.conv_cooldown;
    const int64_t R = div_rcp(now0 + K * d - g.V + cj1 - 1, cj1, g.rcp_cooldown);
    g.wall += R * cj1;
    g.seq += R;
    g.last_bcast = g.wall;
    g.V += R * cj1;
    tk_dispatch(g, ts, n, epoch);
#ifdef TWB_PROFILE_PHASES
    g.prof_fast++;
#endif
    return;
  }
#endif
  int64_t per = d;
  if (S == 2) per = d >> 1;
  else if (S > 2) per = cold_div(d, S);
  const int64_t end_all = now0 + K * d;
  const int64_t cj = g.conv_cooldown;  // 0 when the cooldown is 0
  const int64_t gap = (S > 1) ? min(per, d - per * (S - 1)) : d;
  const int64_t maxgap = (S > 1) ? max(per, d - per * (S - 1)) : d;
  const bool steady_ok = gap > cj && (S == 1 || per > 0);
  const bool wallbound_ok = cj > 0 && d > 0 && maxgap <= cj;
  int64_t base = now0;  // walk position: deadline (base, s) is index m_walk
  int s = 0;
  int64_t m_walk = 1;
  int64_t tgt = (S == 1) ? now0 + d : now0 + per;
  int64_t m_on = g.V == now0 ? 0 : -1;  // index of the deadline V sits on, or -1
  for (;;) {
#ifdef TWB_PROFILE_PHASES
    g.prof_loops++;
#endif
    tk_dispatch(g, ts, n, epoch);
    if (g.V >= end_all) return;
    if (g.last_bcast == g.wall) {
      // Wall-bound state: consecutive deadlines are at most cJ apart and the offset is
      // at least cJ. Every round then sleeps cJ, broadcasts without growing the offset
      // (the next deadline lies within V + cJ) and moves V by exactly cJ, so the rounds
      // up to end_all are R = ceil((end_all - V) / cJ): wall += R*cJ, seq += R.
      // Dispatcher targets inside that window change no clock value, only which
      // arrivals have been passed (tk_dispatch).
      if (wallbound_ok && tk_off_ge<kSpec>(g, cj)) {
        const int64_t R = div_rcp(end_all - g.V + cj - 1, cj, g.rcp_cooldown);
        g.wall += R * cj;
        g.seq += R;
        g.last_bcast = g.wall;
        g.V += R * cj;
        continue;
      }
      // Steady state: V sits on deadline m_on and the stage gaps exceed cJ, so every
      // later deadline below the dispatcher's target resolves the same way (sleep cJ,
      // broadcast, V := deadline): R of them are closed-form: wall += R*cJ, seq += R,
      // offset = t_R - wall, V = t_R.
      if (steady_ok && m_on >= 0) {
        int64_t m_x = K * S;  // last deadline we may cover: end_all, or below the target
        if (g.disp_ts <= end_all) {
          const int64_t x = g.disp_ts - 1 - now0;
          const int64_t fx = HOT_DIV(x, d);
          const int64_t px = (S > 1) ? min((int64_t)(S - 1), HOT_DIV(x - fx * d, per)) : 0;
          m_x = fx * S + px;
        }
        const int64_t R = m_x - m_on;
        if (R > 0) {
          const int64_t fx = (S == 1) ? m_x : (S == 2 ? (m_x >> 1) : m_x / S);
          const int64_t tR = now0 + fx * d + per * (m_x - fx * S);
          g.wall += R * cj;
          g.seq += R;
          g.last_bcast = g.wall;
          g.offset = tR - g.wall;
          g.V = tR;
          m_on = m_x;
          // the walk resumes at deadline m_x + 1 (no catch-up through the skipped ones)
          base = now0 + fx * d;
          s = (int)(m_x - fx * S);
          m_walk = m_x + 1;
          tgt = (s == S - 1) ? base + d : base + per * (s + 1);
          // below the dispatcher's target (m_x < K*S): the next pass would find R = 0 and
          // resolve the round at min(target, next deadline); do that round now (latency
          // variant: with the wall-bound fast path, 8.10 -> 7.94 ms; throughput variant, round
          // 2: 241.3 -> 239.7 ms)
          if (g.V >= end_all) continue;
        }
      }
    }
    // one round, resolved at min(dispatcher's next arrival, first deadline beyond V)
    if (tgt <= g.V) {
      if (d > 0 && g.V - base >= 4 * d) {  // V far ahead: skip whole steps at once
        const int64_t jump = cold_div(g.V - base, d);
        base += jump * d;
        m_walk += jump * S - s;
        s = 0;
      }
      for (;;) {
        tgt = (s == S - 1) ? base + d : base + per * (s + 1);
        if (tgt > g.V) break;
        m_walk++;
        if (++s == S) {
          s = 0;
          base += d;
        }
      }
    }
    const int64_t t_min = g.disp_ts < tgt ? g.disp_ts : tgt;
    tk_resolve<kSpec>(g, t_min);
    m_on = g.V == tgt ? m_walk : -1;
  }
}

#ifdef TWB_SIM_OUTLINE_IDLE
#define TWB_IDLE_FN static __device__ __noinline__
#else
#define TWB_IDLE_FN TWB_TK_FN
#endif
template <bool kSpec = false>
TWB_IDLE_FN void tk_idle(TkGrid& g, const int64_t* __restrict__ ts, int32_t n, int64_t epoch,
                                        int64_t end) {
  // idle jump: only the dispatcher drives time (its target is <= end while V < end)
  for (;;) {
    tk_dispatch(g, ts, n, epoch);
    if (g.V >= end) return;
    tk_resolve<kSpec>(g, g.disp_ts);
  }
}

// Prediction cache: 32 entries held one per lane (key = P << 32 | D, for predictors
// whose duration ignores C); a lookup is one compare + ballot + shuffle. Linear models
// with a context term keep a single exact (P, D, C) entry.
TWB_COLD int64_t cold_predict_scalar(const char* ps, int id, int64_t P, int64_t D, int64_t C) {
  return predict_scalar(ps, id, P, D, C);
}
TWB_COLD int64_t cold_nearest_warp(const TableView& t, int64_t P, int64_t D) { return table_nearest_warp(t, P, D); }

#define TWB_LUT_FN __device__ __forceinline__  // outlining it: 65,536 configs 345 -> 392 ms
// every lane runs the same scalar lookup (bit-length LUT bracketing, exact int lerps
// with blob reciprocals); only the rare nearest-row fallback uses the lanes
TWB_LUT_FN int64_t predict_lut(const char* ps, int id, int64_t P, int64_t D, int64_t C) {
  if (id < 0 || id >= pset_ndesc(ps)) return TW_PRED_BAD_DESC;
  const tw_pred_desc* d = pset_desc(ps, id);
  if (d->kind != TW_PRED_TABLE) return cold_predict_scalar(ps, id, P, D, C);
  const TableView t = table_view(ps, d);
  int p0, p1, d0, d1;
  int64_t P0, P1, D0, D1;
  if (bracket_lut(t.pax, t.lutp, t.np, P, p0, p1, P0, P1) && bracket_lut(t.dax, t.lutd, t.nd, D, d0, d1, D0, D1)) {
    const int64_t r = table_corners2(t, p0, p1, d0, d1, P0, P1, D0, D1, P, D);
    if (r != TW_PRED_TABLE_MISS) return r;
  }
  if (d->allow_extrapolation) return cold_nearest_warp(t, P, D);
  return TW_PRED_TABLE_MISS;
}

template <bool kTput>
TWB_PRED_FN int64_t predict_miss(const char* ps, const uint2* qh, int id, int64_t P, int64_t D, int64_t C) {
#ifdef TWB_SIM_WARP_PRED
  return predict_warp(ps, id, P, D, C);
#else
  // with the bulk-lookup section staged (latency regime): four shared-memory loads
  if (qh != nullptr && ((P | D) >> 31) == 0) {
    int64_t r;
    if (predict_fast<!kTput>(ps, qh, pset_ndesc(ps), (int32_t)P, (int32_t)D, id, r)) return r;
  }
  return predict_lut(ps, id, P, D, C);
#endif
}

// Linear models with a context term only (never in the Table sweeps): out of line
// (A/B: 1,024 configs 8.68 -> 8.63 ms, 65,536 configs 345 -> 335 ms)
#ifdef TWB_SIM_INLINE_CTXPRED
static __device__ __forceinline__
#else
static __device__ __noinline__
#endif
int64_t cold_predict_warp(const char* ps, int id, int64_t P, int64_t D, int64_t C) {
  return predict_warp(ps, id, P, D, C);
}

struct PredCache {
  int64_t misses;      // profiling only
  int64_t miss_cyc;    // profiling only
  int64_t key, val;    // this lane's entry
  int64_t P, D, C, d;  // single entry (uses_c)
  bool uses_c;
  int victim;
};

template <bool kTput>
__device__ __forceinline__ int64_t predict_cached(PredCache& pc, const char* ps, const uint2* qh, int id, int64_t P,
                                                  int64_t D, int64_t C) {
  const int lane = threadIdx.x & 31;
  if (pc.uses_c) {  // Linear models with a context term: one exact (P, D, C) entry
    if (P == pc.P && D == pc.D && C == pc.C) return pc.d;
    const int64_t d = cold_predict_warp(ps, id, P, D, C);
    pc.P = P;
    pc.D = D;
    pc.C = C;
    pc.d = d;
    return d;
  }
  const int64_t key = (P << 32) | D;
  const unsigned hit = __ballot_sync(kFull, pc.key == key);
  if (hit) return __shfl_sync(kFull, pc.val, __ffs(hit) - 1);
#ifdef TWB_PROFILE_PHASES
  const long long m0 = clock64();
#endif
  const int64_t d = predict_miss<kTput>(ps, qh, id, P, D, C);
#ifdef TWB_PROFILE_PHASES
  pc.misses++;
  pc.miss_cyc += clock64() - m0;
#endif
  if (lane == pc.victim) {
    pc.key = key;
    pc.val = d;
  }
  pc.victim = (pc.victim + 1) & 31;
  return d;
}

// full event dump (audited configs only)
// (outlining this and the Linear-with-context predictor measured slower: 11.6 -> 12.2 ms)
#ifndef TWB_SIM_OUTLINE_COLD2
__device__ __forceinline__
#else
static __device__ __noinline__
#endif
void cold_dump_event(tw_event* evp, int64_t pos, int32_t rq, int kind, int64_t ts, int64_t step) {
  tw_event e;
  e.ts_ns = ts;
  e.step = (int32_t)step;
  e.req_kind = (rq << 2) | kind;
  evp[pos] = e;
}

struct Emitter {
  uint64_t dig;   // lane-partial digest
  uint64_t msum;  // lane-partial sum of the multipliers (segments only; dead code otherwise)
  int64_t* first;
  int64_t* finish;
  tw_event* evp;
  int64_t ev_cap;
  __device__ __forceinline__ void event(int64_t pos, int32_t rq, int kind, int64_t ts, int64_t step) {
    dig += tw_event_hash((uint64_t)pos, (uint64_t)rq, (uint64_t)kind, ts, step);
    if (evp && pos < ev_cap) cold_dump_event(evp, pos, rq, kind, ts, step);
  }
  // u = tw_event_u(ts, step), the step-uniform part of the hash, computed once per step
  __device__ __forceinline__ void event_u(int64_t pos, int32_t rq, int kind, uint64_t u, int64_t ts, int64_t step) {
    const uint64_t m = tw_event_mult((uint64_t)rq, (uint64_t)kind);
    dig += m * ((uint64_t)pos * TW_DIG_A + u);
    msum += m;
    if (evp && pos < ev_cap) cold_dump_event(evp, pos, rq, kind, ts, step);
  }
};

// Plan passes over more than 32 active slots (pass 1a: decode candidates and whether any
// request is mid-prefill; the KV blocks held, oracle.py:43-46, 122). Out of line in the
// throughput variant (TWB_SIM_OUTLINE_WIDE): the hot loop's code footprint is what bounds
// it there (instruction-fetch stalls), and most steps have <= 32 active requests.
#ifdef TWB_SIM_OUTLINE_WIDE
#define TWB_WIDE_FN static __device__ __noinline__
#else
#define TWB_WIDE_FN static __device__ __forceinline__
#endif
TWB_WIDE_FN int wide_pass1a(Slots sl, int n_act) {
  const int lane = threadIdx.x & 31;
  int total_dec = 0;
  bool any_mid = false;
#pragma unroll 1
  for (int b = 0; b < n_act; b += 32) {
    const int i = b + lane;
    const bool v = i < n_act;
    const int32_t pr = v ? sl.prompt[i] : 0, dn = v ? sl.done[i] : 0;
    const int32_t e = v ? sl.emit[i] : 0, op = v ? sl.output[i] : 0;
    const bool mid = v && dn < pr;
    total_dec += __popc(__ballot_sync(kFull, v && !mid && e < op));
    any_mid |= __any_sync(kFull, mid);
  }
  return (total_dec << 1) | (any_mid ? 1 : 0);
}
TWB_WIDE_FN int64_t wide_held(Slots sl, int n_act, Blocks blk) {
  const int lane = threadIdx.x & 31;
  int64_t held_l = 0;
#pragma unroll 1
  for (int b = 0; b < n_act; b += 32) {
    const int i = b + lane;
    if (i < n_act) {
      const int32_t h0 = blk.ceil_div(sl.prompt[i]), h1 = blk.ceil_div(sl.done[i] + sl.emit[i]);
      held_l += h0 > h1 ? h0 : h1;  // _held (oracle.py:43-46)
    }
  }
  return warp_sum_i64_redux(held_l);
}

// ---- busy-period segments (sim_seg.cu, DESIGN.md §4.1 "Busy-period segments") ----------
// A config's timeline restarts from the same state whenever an arrival finds the engine
// empty (nothing running or waiting: oracle.py:78-83 jumps `now` to the arrival): from
// there on the event stream depends only on the arrivals, not on the history. Such an
// arrival is a regeneration point. The latency regime splits each config's arrivals into
// segments at likely regeneration points and simulates them speculatively in parallel
// (mode 1); a join pass (mode 2 for the rare mismatches) chains the valid pieces.
constexpr int32_t kSegOverflow = -1;  // a segment ran out of log or overrun-stamp room
constexpr int kSegLogPerReq = 8;      // Timekeeper log records per request of a segment
// Room per segment: kSegLogPerReq log records and 4 overrun stamps per own request, plus
// the same for SegParams::xtra more requests (an overrun past the segment's end needs room
// for the next busy period; xtra is set from the segment count so the total stays bounded)
struct TkLog {  // one Timekeeper call of the loop: K >= 1 tk_run(now0, d, K); K = 0 tk_idle(now0)
  int64_t now0, d, K;
};
struct TkState {                      // a Timekeeper state as the join pass needs it
  int64_t wall, seq, last_bcast, offset;
  int32_t disp, pad;
};
struct SegRegen {  // a segment's counters and speculative Timekeeper at the idle point before arrival j
  int64_t events;
  uint64_t dig;
  uint64_t msum;
  int32_t steps;
  int32_t pad;
  TkState tk;
};
struct SegSummary {  // one per (config, segment)
  int32_t j_stop;    // next arrival at the stop (n: the config's end)
  int32_t status;    // TW_SIM_* or kSegOverflow
  int32_t last_regen;  // last regeneration point recorded (a0 if none)
  int32_t adm_end;     // requests [.., adm_end) admitted at the stop
  int64_t final_now;
  int64_t events;
  uint64_t dig;
  uint64_t msum;  // sum of the event multipliers (frame shifts)
  int32_t steps;
  int32_t pred_code;
  int32_t log_len;       // Timekeeper log records of this segment
  int32_t pad;
  TkState tk;            // speculative Timekeeper at the stop
  int64_t d_lo, d_hi;    // wall shifts that keep every Timekeeper decision of this run
};
struct SegCtx {
  int32_t a0, a1;         // arrival range: own [a0, a1); mode 2: start a0, a1 = n
  TkLog* log;             // mode 1: this segment's Timekeeper calls, replayed after its run
  int32_t log_cap;
  int32_t log_len;        // mode 1: out
  int64_t* side;          // mode 1: (first, finish) of requests a1 + i admitted in the overrun
  int32_t side_cap;
  int32_t* regpos;        // per request of the config: log position at a regeneration point, else -1
  SegRegen* reg;          // per request of the config: counters at that point
  TkGrid* g;              // mode 2: the Timekeeper state (in/out)
  SegSummary out;         // mode 2: result (mode 1 writes its own summary to `sum`)
  SegSummary* sum;        // mode 1: where the summary goes
};

struct SegParams {
  int32_t wmax;          // segment slots per config
  int32_t min_req;       // requests per segment at least
  int32_t* nseg;         // [n_cfg]; 0 = not segmented (the join pass runs the config serially)
  int32_t* seg_a0;       // [n_cfg * wmax] first arrival of each segment
  SegSummary* summ;      // [n_cfg * wmax]
  int32_t* regpos;       // [r_max], -1 = not a regeneration point
  SegRegen* reg;         // [r_max]
  TkLog* log;            // [kSegLogPerReq * (r_max + xtra * n_cfg * wmax)]
  int64_t* side;         // [2 * 4 * (r_max + xtra * n_cfg * wmax)]
  int64_t r_max;
  int64_t xtra;          // extra requests of room per segment
  int32_t cap_div;       // test hook (TWB_SIM_SEG_CAPDIV): log / overrun room divided by this
  int32_t epoch;         // launch number: a segment's summary is complete when its pad == epoch
  int32_t* stats;        // optional, 8 int32 per config (tw_sim_set_seg_stats)
  int32_t* counter;      // [0..1] segment work counter (64-bit), [2] join work counter,
                         // [4..5] Timekeeper replay work counter (64-bit)
};

__device__ __forceinline__ TkState tk_state(const TkGrid& g) {
  TkState t;
  t.wall = g.wall;
  t.seq = g.seq;
  t.last_bcast = g.last_bcast;
  t.offset = g.offset;
  t.disp = g.disp;
  t.pad = 0;
  return t;
}

// kTput: the throughput variant (predictor blob read from global memory, see k_sim).
// kMode: 0 the whole config (k_sim); 1 one speculative segment (k_sim_seg: local frame,
// Timekeeper calls logged for the segment's replay, stops at the first idle point at or
// past a1); 2 the join pass's serial piece (k_sim_join: the true Timekeeper inline, stops at
// the first idle point that its owner segment also recorded as a regeneration point).
template <bool kTput, int kMode = 0>
__device__ void run_config(const SimParams& p, const char* ps, Slots sl, int c, SegCtx* sx = nullptr) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  const long long t_start = clock64();  // per-config cycles (always on: 2 reads)
  int64_t n_normal = 0, n_runs = 0, n_run_steps = 0, tk_cyc = 0, ev_cyc = 0;
  int64_t plan_cyc = 0, pred_cyc = 0, apply_cyc = 0, arr_cyc = 0, adm_cyc = 0;
#ifdef TWB_SIM_CHECK
  // invariant counters (sim_check.cu): [0] iterations checked, [1] virtual time went back,
  // [2] a slot overran its prompt / output, [3] the incremental KV-block counter differs from
  // the recomputation (engine.py:359-369), [4] Timekeeper offset / seq / wall went back,
  // [5] V != wall + offset or V short of the step end, [6] last broadcast after the wall,
  // [7] event count at the end differs from sum(max(output, 1) + 1)
  int32_t chk[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int64_t chk_kv = 0, chk_now = 0, chk_off = 0, chk_seq = 0, chk_wall = 0;
#endif
#ifdef TWB_PROFILE_PHASES
  // TWB_PROFILE_PHASES builds write 32 int64 per config (tw_sim_set_profile stride 32)
  int64_t x_walk_cyc = 0, x_fast_cyc = 0, x_it_adm = 0, x_it_wait = 0, x_it_wide = 0, x_body_cyc = 0;
  int64_t x_it_chunk = 0, x_it_k1 = 0, x_it_idle = 0, x_idle_cyc = 0;
#endif
  const tw_sim_cfg cfg = p.cfgs[c];
  tw_sim_result r;
  r.final_now_ns = cfg.epoch_ns;
  r.steps = 0;
  r.events = 0;
  r.digest = 0;
  r.tk_seq = 0;
  r.tk_offset_ns = 0;
  r.tk_wall_ns = 0;
  r.status = TW_SIM_OK;
  r.pred_code = 0;

  const int S = cfg.pp_stages, TP = cfg.workers_per_replica;
  const bool tk_on = (cfg.flags & TW_SIM_TIMEKEEPER) != 0;
  if (cfg.chunk_size < 1 || cfg.max_batch_tokens < cfg.chunk_size || cfg.kv_block_tokens < 1 ||
      cfg.kv_capacity_blocks < 1 || TP < 1 || S < 1 || (cfg.policy != 0 && cfg.policy != 1)) {
    r.status = TW_SIM_BAD_CONFIG;  // engine.py:109-120
  } else if (cfg.max_running > p.cap) {
    r.status = TW_SIM_CAPACITY;
  }
  if (r.status != TW_SIM_OK) {
    if constexpr (kMode == 0) {
      if (lane == 0) p.res[c] = r;
    } else {
      SegSummary o = {};
      o.j_stop = sx->a0;
      o.status = r.status;
      o.last_regen = sx->a0;
      o.adm_end = sx->a0;
      o.final_now = cfg.epoch_ns;
      if constexpr (kMode == 1) {
        if (lane == 0) *sx->sum = o;
      } else {
        sx->out = o;
      }
    }
    return;
  }

  const int64_t wl0 = p.wl_off[cfg.workload_id];
  const int32_t n = (int32_t)(p.wl_off[cfg.workload_id + 1] - wl0);
  const int64_t* __restrict__ ts = p.ts + wl0;
  const int32_t* __restrict__ prm = p.prompt + wl0;
  const int32_t* __restrict__ outp = p.output + wl0;
  const int64_t epoch = cfg.epoch_ns;
  const int32_t chunk = cfg.chunk_size;
  const int32_t mbt = cfg.max_batch_tokens;
  const int32_t max_running = cfg.max_running;
  Blocks blk;
  blk.init((uint32_t)cfg.kv_block_tokens);

  Emitter em;
  em.dig = 0;
  em.msum = 0;
  em.first = p.first ? p.first + p.req_base[c] : nullptr;
  em.finish = p.finish ? p.finish + p.req_base[c] : nullptr;
  em.evp = nullptr;
  em.ev_cap = 0;
  if (p.ev && p.ev_off[c + 1] > p.ev_off[c]) {  // audited config: full event dump
    em.evp = p.ev + p.ev_off[c];
    em.ev_cap = p.ev_off[c + 1] - p.ev_off[c];
  }

  // predictor: cache + whether a decode-only run has a constant duration
  const tw_pred_desc* pd = pset_desc(ps, cfg.pred_id < pset_ndesc(ps) ? cfg.pred_id : 0);
  PredCache pc;
  pc.misses = 0;
  pc.miss_cyc = 0;
  pc.key = -1;
  pc.val = 0;
  pc.victim = 0;
  pc.P = -1;
  pc.D = -1;
  pc.C = -1;
  pc.d = 0;
  pc.uses_c = pd->kind == TW_PRED_LINEAR && pd->per_context_token_us != 0.0;
  // the blob holds the bulk-lookup section: staged in shared memory (latency variant) or
  // read from global memory (throughput variant)
  const tw_pset_header* hdr = reinterpret_cast<const tw_pset_header*>(ps);
  const uint2* qh = (hdr->fast_off > 0 && p.pset_bytes >= (uint32_t)hdr->total_bytes) ? pset_qhdr(ps) : nullptr;
  const bool macro_ok = !pc.uses_c && cfg.pred_id >= 0 && cfg.pred_id < pset_ndesc(ps);

  TkGrid g_own;
  TkGrid& g = (kMode == 2) ? *sx->g : g_own;  // mode 2 continues the join pass's Timekeeper
  g.d_lo = INT64_MIN;
  g.d_hi = INT64_MAX;
  if constexpr (kMode != 2) {
  g.wall = epoch;
  g.offset = 0;
  g.seq = 0;
  g.last_bcast = INT64_MIN;
  g.V = epoch;
  g.cooldown = cfg.tk_cooldown_ns;
  g.conv_cooldown = g.cooldown > 0 ? cold_fake_sleep(g.cooldown) : 0;
  g.rcp_cooldown = g.conv_cooldown > 0 ? __drcp_rn(__ll2double_rn(g.conv_cooldown)) : 0.0;
  g.disp = 0;
#ifdef TWB_PROFILE_PHASES
  g.prof_calls = g.prof_fast = g.prof_loops = 0;
#endif
  g.win.load(ts, n, epoch, 0);
  g.disp_ts = n > 0 ? __shfl_sync(kFull, g.win.v, 0) : INT64_MAX;
  }

  // segments start at arrival a0 (the engine empty, `now` jumping to it); mode 0 at 0
  const int32_t a0 = kMode != 0 ? sx->a0 : 0;
  const int32_t a1 = kMode == 1 ? sx->a1 : n;
  ArrWindow arr;
  arr.load(ts, n, epoch, a0);
  int64_t now = epoch, n_events = 0;
  int32_t step = 0, fut = a0, w_head = a0, n_act = 0;  // waiting = [w_head, fut), future = [fut, n)
  int64_t next_arr = a0 < n ? __shfl_sync(kFull, arr.v, 0) : INT64_MAX;
  // waiting-queue window: lane l holds prompt/output of request w_head + l, reloaded
  // (prefetched) right after every admission so the next admission finds it in registers
  int32_t qbase = a0;
  int32_t q_pr = (a0 + lane < n) ? __ldg(prm + a0 + lane) : 0;
  int32_t q_op = (a0 + lane < n) ? __ldg(outp + a0 + lane) : 0;
  int overflow = 0;
  int32_t last_regen = a0, j_stop = n, log_len = 0;
  if constexpr (kMode != 0) {
    // (a0 < n: an empty workload's slot 0 is the next config's first request)
    if (kMode == 1 && lane == 0 && a0 < n) {  // the segment's start is its first regeneration point
      sx->reg[a0] = SegRegen{0, 0, 0, 0, 0, TkState{}};
      sx->regpos[a0] = 0;
    }
    if (a0 > 0 && a0 < n) {  // the idle jump to the first arrival (oracle.py:81-83)
      now = next_arr;
      if constexpr (kMode == 1) {
        if (tk_on) {
          if (lane == 0) sx->log[0] = TkLog{now, 0, 0};
          log_len = 1;
        }
      } else if (tk_on) {
        tk_idle(g, ts, n, epoch, now);
      }
    }
  }

  while (fut < n || w_head < fut || n_act > 0) {
    // ---- arrivals with epoch + offset <= now join the waiting queue (oracle.py:73-75)
    const long long q0 = TWB_CLK();
    while (next_arr <= now) {
      fut++;
      next_arr = fut < n ? arr.get(ts, n, epoch, fut) : INT64_MAX;
    }
    const bool waiting = w_head < fut;
    if constexpr (kMode == 1) {  // room for this iteration's log record and overrun stamps
      if (log_len + 2 > sx->log_cap || fut - a1 > sx->side_cap) {
        r.status = kSegOverflow;
        break;
      }
    }
    const long long q1 = TWB_CLK();
    arr_cyc += q1 - q0;

    // ---- _plan (oracle.py:117-180), pass 1a (only needed with > 32 active)
    int total_dec = 0;
    bool any_mid = false;
    if (n_act > 32) {
      const int v = wide_pass1a(sl, n_act);
      total_dec = v >> 1;
      any_mid = v & 1;
    }
    // KV: free = cap - sum(_held) (oracle.py:122), only needed when a queue head is probed
    int64_t free0 = 0;
    const bool need_free = waiting && n_act > 32;  // <= 32 active: summed in pass 1b below
    if (need_free) free0 = (int64_t)cfg.kv_capacity_blocks - wide_held(sl, n_act, blk);

    // ---- pass 1b: decode cutoff, chunk takes, features
    bool do_dec = true, do_chunks = true;
    int64_t p_l = 0, c_l = 0;  // lane partial P and C
    int n_chunk = 0, chunk_ev = 0, n_dec = 0;
    int dec_before = 0;
    int64_t want_before = 0, budget = mbt;
    int min_rem = 0x7fffffff;  // macro-step horizon: decoders' remaining outputs, chunks' repeats
#pragma unroll 1
    for (int b = 0; b < (n_act > 0 ? n_act : 1); b += 32) {
      const int i = b + lane;
      const bool v = i < n_act;
      const int32_t pr = v ? sl.prompt[i] : 0, dn = v ? sl.done[i] : 0;
      const int32_t e = v ? sl.emit[i] : 0, op = v ? sl.output[i] : 0;
      const bool mid = v && dn < pr;
      const bool dcand = v && !mid && e < op;
      const unsigned dm = __ballot_sync(kFull, dcand);
      if (b == 0) {
        if (n_act <= 32) {
          total_dec = __popc(dm);
          any_mid = __any_sync(kFull, mid);
          if (waiting) {  // free KV blocks from this pass's loads (oracle.py:122)
            const int32_t h0 = blk.ceil_div(pr), h1 = blk.ceil_div(dn + e);  // 0 for idle lanes
            free0 = (int64_t)cfg.kv_capacity_blocks - warp_sum_i64_redux(h0 > h1 ? h0 : h1);
          }
        }
        if (cfg.policy == TW_POLICY_PREFILL_PRIORITIZED) {  // oracle.py:168-178
          bool have_prefill = any_mid;
          if (!have_prefill && waiting) {
            const int32_t hp = __shfl_sync(kFull, q_pr, 0);  // qbase == w_head
            have_prefill = n_act < max_running && blk.ceil_div(hp) <= free0;
          }
          do_chunks = have_prefill;
          do_dec = !have_prefill;
        }
        n_dec = do_dec ? min(total_dec, mbt) : 0;
        budget = (int64_t)mbt - n_dec;
      }
      const int rank = dec_before + __popc(dm & lt);
      const bool is_dec = do_dec && dcand && rank < mbt;
      dec_before += __popc(dm);
      int32_t plan = is_dec ? -1 : -2;
      if (is_dec) {
        c_l += (int64_t)pr + e;  // DecodeSlot.context_len = prompt + emitted
        min_rem = min(min_rem, op - e);
        sl.dlist[rank] = i;
      }
      if (do_chunks && __any_sync(kFull, mid)) {
        const int64_t want = mid ? min((int64_t)chunk, (int64_t)(pr - dn)) : 0;
        const int32_t incl = warp_incl_scan_sat((int32_t)want);
        const int64_t E = want_before + warp_excl_from_incl(incl);  // tokens taken by earlier chunks
        const bool chosen = mid && budget - E > 0;
        if (chosen) {
          const int64_t take = min(want, budget - E);
          plan = (int32_t)take;
          p_l += take;
          c_l += dn;  // PrefillChunk.context_len_before = done_prefill
          if (dn + take >= pr) chunk_ev += (op <= 1) ? 2 : 1;
          // steps this chunk repeats with the same take before the one that completes
          // the prompt: ceil(rem / take) - 1
          min_rem = min(min_rem, (int)((uint32_t)(pr - dn - 1) / (uint32_t)take));
        }
        n_chunk += __popc(__ballot_sync(kFull, chosen));
        want_before += __shfl_sync(kFull, incl, 31);
      }
      if (v) sl.plan[i] = plan;
    }
    // tokens the chunks consumed: every chosen chunk took `want` except possibly the last
    budget -= min(want_before, budget > 0 ? budget : (int64_t)0);

    // ---- admission from the waiting head: strict FCFS, KV + slot + budget gates
    const long long q2 = TWB_CLK();
    plan_cyc += q2 - q1;
    int n_adm = 0;
    if (do_chunks && budget > 0 && waiting) {
      int64_t free_l = free0, slots = (int64_t)max_running - n_act;
      while (budget > 0 && slots > 0 && w_head + n_adm < fut) {
        const int32_t idx = w_head + n_adm + lane;
        const bool cand = idx < fut && lane < slots;
        const bool inwin = n_adm == 0;  // qbase == w_head: the window is this round
        const int32_t pr = cand ? (inwin ? q_pr : __ldg(prm + idx)) : 0;
        const int64_t need = blk.ceil_div(pr);
        const int64_t want = min((int64_t)chunk, (int64_t)pr);
        const int32_t NEi = warp_incl_scan_sat(cand ? (int32_t)need : 0);
        const int32_t WEi = warp_incl_scan_sat(cand ? (int32_t)want : 0);
        const int64_t NE = warp_excl_from_incl(NEi), WE = warp_excl_from_incl(WEi);
        const bool ok = cand && (budget - WE > 0) && (need <= free_l - NE);
        const unsigned bad = __ballot_sync(kFull, !ok);
        const int k = bad ? __ffs(bad) - 1 : 32;
        if (lane < k) {
          const int slot = n_act + n_adm + lane;
          const int64_t take = min(want, budget - WE);
          sl.req[slot] = idx;
          if constexpr (kMode == 1) {
            if (idx >= a1) {  // overrun: its stamps go to the side buffer (unset = -1)
              sx->side[2 * (int64_t)(idx - a1)] = -1;
              sx->side[2 * (int64_t)(idx - a1) + 1] = -1;
            }
          } else if constexpr (kMode == 2) {
            // a serial piece crosses other segments' ranges, whose speculative stamps of a
            // request still running when the config stops must not survive
            if (em.first) em.first[idx] = -1;
            if (em.finish) em.finish[idx] = -1;
          }
          sl.prompt[slot] = pr;
          const int32_t op = inwin ? q_op : __ldg(outp + idx);
          sl.output[slot] = op;
          sl.done[slot] = 0;
          sl.emit[slot] = 0;
          sl.plan[slot] = (int32_t)take;
          p_l += take;
#ifdef TWB_SIM_CHECK
          chk_kv += blk.ceil_div(pr);  // held at admission: the prompt's reservation (lane partial)
#endif
          if (take >= pr) chunk_ev += (op <= 1) ? 2 : 1;
          // repeats of this first take before the completing chunk (macro horizon)
          min_rem = min(min_rem, take > 0 ? (int)((uint32_t)(pr - 1) / (uint32_t)take) : 0);
        }
        if (k == 0) break;
        const int64_t tot_need = __shfl_sync(kFull, NEi, k - 1);  // <= free: exact
        const int64_t last_want = __shfl_sync(kFull, want, k - 1);
        const int64_t last_we = __shfl_sync(kFull, WE, k - 1);    // < budget: exact
        const int64_t last_take = min(last_want, budget - last_we);
        budget -= last_we + last_take;
        free_l -= tot_need;
        slots -= k;
        n_adm += k;
        if (k < 32) break;
      }
      n_chunk += n_adm;
    }
    __syncwarp();

    if (n_dec == 0 && n_chunk == 0) {
      if (n_act > 0 || waiting) {  // oracle.py:78-80 -> _diagnose_stall
        r.status = n_act > 0 ? TW_SIM_STALLED_ACTIVE : TW_SIM_STALLED_KV;
        break;
      }
      if constexpr (kMode == 1) {  // the engine is empty and arrival fut is next
        if (fut >= a1) {             // past this segment's arrivals: stop here
          j_stop = fut;
          break;
        }
        uint64_t dg = em.dig, ms = em.msum;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          dg += __shfl_xor_sync(kFull, dg, o);
          ms += __shfl_xor_sync(kFull, ms, o);
        }
        if (lane == 0) {  // a regeneration point of this segment's run
          sx->reg[fut] = SegRegen{n_events, dg, ms, step, 0, TkState{}};
          sx->regpos[fut] = log_len;
        }
        last_regen = fut;
      } else if constexpr (kMode == 2) {  // converged with the owner segment's run
        if (sx->regpos && fut > a0 && __ldg(sx->regpos + fut) >= 0) {
          j_stop = fut;
          break;
        }
      }
      now = next_arr;  // idle until the next arrival (oracle.py:81-83)
#ifdef TWB_PROFILE_PHASES
      const long long i0 = clock64();
      x_it_idle++;
#endif
      if constexpr (kMode == 1) {
        if (tk_on) {
          if (lane == 0) sx->log[log_len] = TkLog{now, 0, 0};
          log_len++;
        }
      } else {
        if (tk_on) tk_idle(g, ts, n, epoch, now);
      }
#ifdef TWB_PROFILE_PHASES
      x_idle_cyc += clock64() - i0;
#endif
      continue;
    }

    // ---- predict (oracle.py:85-86)
    const long long q3 = TWB_CLK();
    adm_cyc += q3 - q2;
    const int64_t P = (int64_t)__reduce_add_sync(kFull, (unsigned)p_l);  // P <= max_batch_tokens
    const int64_t C = pc.uses_c ? warp_sum_i64_redux(c_l) : 0;
    const int64_t d = predict_cached<kTput>(pc, ps, qh, cfg.pred_id, P, n_dec, C);
    pred_cyc += TWB_CLK() - q3;
    if (d < 0) {
      r.status = TW_SIM_PRED_ERROR;
      r.pred_code = (d % 1000 != 0) ? (int32_t)d : TW_PRED_NEGATIVE;  // a negative table row: engine limit
      if constexpr (kMode != 0) w_head += n_adm;  // admitted (unstamped) before the error
      break;
    }

    // ---- macro step: a run of K steps with an identical plan.
    // After this step's admissions (the admitted become mid-prefill chunk slots with the
    // same take), the same decoders decode and the same chunks take
    // the same tokens until a decoder finishes (min remaining output, finishing step
    // included), a chunk reaches its prompt's last chunk (excluded), or a new arrival
    // becomes visible to an empty queue; a blocked queue head stays blocked (slots and
    // budget constant, KV free non-increasing). P and D are constant, so is d.
    // One code path for both: a normal step is the K = 1 case (the loop is fetch-bound,
    // so a single Timekeeper walk and a single apply block beat specialised copies).
    int64_t K = 1;
    if (macro_ok) {
      K = __reduce_min_sync(kFull, min_rem);
      // an emptied queue can admit the next arrival; a non-empty one stays blocked
      if (w_head + n_adm == fut && fut < n && d > 0 && next_arr - now <= (K - 1) * d) {
        // the plan after step j sees arrivals <= now + j*d: stop at the first crossing
        const int64_t ka = div_rcp(next_arr - now + d - 1, d, __drcp_rn(__ll2double_rn(d)));
        if (ka < K) K = ka;
      }
      if (K < 1) K = 1;
    }
    const int64_t now0 = now;
    const int32_t step0 = step;
    {
#ifdef TWB_PROFILE_PHASES
      const int64_t prof_fast0 = g.prof_fast;
      x_it_adm += n_adm > 0;
      x_it_wait += waiting;
      x_it_wide += n_act > 32;
      x_it_chunk += n_chunk > 0;
      x_it_k1 += K == 1;
#endif
      const long long c0 = TWB_CLK();
      if constexpr (kMode == 1) {  // logged, replayed after the segment's run (k_sim_seg)
        if (tk_on) {
          if (lane == 0) sx->log[log_len] = TkLog{now0, d, K};
          log_len++;
        }
      } else {
        if (tk_on) tk_run(g, ts, n, epoch, S, now0, d, K);  // WorkerGrid stage deadlines
      }
      tk_cyc += TWB_CLK() - c0;
#ifdef TWB_PROFILE_PHASES
      if (tk_on) {
        if (g.prof_fast != prof_fast0) x_fast_cyc += TWB_CLK() - c0;
        else x_walk_cyc += TWB_CLK() - c0;
      }
#endif
    }
    const long long q4 = TWB_CLK();
    // events of steps 1..K-1 (decodes only), flattened over the lanes: e -> (step j, rank i)
    const int64_t body = (K - 1) * (int64_t)n_dec;
#ifdef TWB_PROFILE_PHASES
    const long long b0 = clock64();
#endif
    if (body > 0) {
      const int D = n_dec;
      // digest v2 is linear in (position, ts, step) per request: decoder i's K-1 body
      // events sum to M_i * (U + (K-1)*A*i) (twb200.h tw_event_run_sum), one term per
      // decoder instead of one hash per event
      const uint64_t m = (uint64_t)(K - 1);
      const uint64_t U = tw_event_run_sum(m, (uint64_t)n_events, (uint64_t)D, now0, d, step0);
      const uint64_t mA = m * TW_DIG_A;
#pragma unroll 1
      for (int i = lane; i < D; i += 32)
      {
        const uint64_t mi = tw_event_mult((uint64_t)sl.req[sl.dlist[i]], TW_EV_OUTPUT_TOKEN);
        em.dig += mi * (U + mA * (uint64_t)i);
        em.msum += mi * m;
      }
      if (em.evp) {  // audited config: the body's events themselves, flattened over the lanes
        const int q32 = 32 / D, r32 = 32 % D;
        int64_t j = lane / D;
        int i = lane - (int)j * D;
#pragma unroll 1
        for (int64_t e = lane; e < body && n_events + e < em.ev_cap; e += 32) {
          cold_dump_event(em.evp, n_events + e, sl.req[sl.dlist[i]], TW_EV_OUTPUT_TOKEN, now0 + (j + 1) * d,
                          step0 + j + 1);
          i += r32;
          j += q32;
          if (i >= D) { i -= D; j++; }
        }
      }
    }
#ifdef TWB_PROFILE_PHASES
    x_body_cyc += clock64() - b0;
#endif
    if (K >= 2) {
      n_runs++;
      n_run_steps += K;
    } else {
      n_normal++;
    }
    now = now0 + K * d;
    step = step0 + (int32_t)K;

    // ---- apply step K (oracle.py:88-112): chunks' events first, then decodes', in slot
    // order. Chunks advance K takes; in a run (K >= 2) none completes (run horizon), so
    // chunk events only occur when K == 1.
    const int n_tot = n_act + n_adm;
    const int chunk_ev_total = __reduce_add_sync(kFull, (unsigned)chunk_ev);
    int64_t pos_c = n_events + body, pos_d = pos_c + chunk_ev_total;
    int kept = 0;
    const uint64_t u_now = tw_event_u(now, step);
#pragma unroll 1
    for (int b = 0; b < n_tot; b += 32) {
      const int i = b + lane;
      const bool v = i < n_tot;
      int32_t rq = 0, pr = 0, op = 0, dn = 0, e = 0, plan = -2;
      if (v) {
        rq = sl.req[i];
        pr = sl.prompt[i];
        op = sl.output[i];
        dn = sl.done[i];
        e = sl.emit[i];
        plan = sl.plan[i];
      }
      int nev = 0, k0 = 0;
      bool fin = false;
      const bool is_chunk = plan >= 0, is_dec = plan == -1;
#ifdef TWB_SIM_CHECK
      const int32_t held0 = v ? max(blk.ceil_div(pr), blk.ceil_div(dn + e)) : 0;
#endif
      if (is_chunk) {
        dn += plan * (int32_t)K;
        if (dn >= pr) {
          e = 1;
          nev = 1;
          k0 = TW_EV_FIRST_TOKEN;
          if (e >= op) { nev = 2; fin = true; }
        }
      } else if (is_dec) {
        e += (int32_t)K;
        nev = 1;
        k0 = TW_EV_OUTPUT_TOKEN;
        if (e >= op) { nev = 2; fin = true; }
      }
      const unsigned c1 = __ballot_sync(kFull, is_chunk && nev >= 1);
      const unsigned c2 = __ballot_sync(kFull, is_chunk && nev == 2);
      const unsigned d1 = __ballot_sync(kFull, is_dec && nev >= 1);
      const unsigned d2 = __ballot_sync(kFull, is_dec && nev == 2);
      if (nev) {
        const int64_t ps0 = is_chunk ? pos_c + __popc(c1 & lt) + __popc(c2 & lt)
                                     : pos_d + __popc(d1 & lt) + __popc(d2 & lt);
#pragma unroll 1
        for (int t = 0; t < nev; t++) em.event_u(ps0 + t, rq, t ? TW_EV_FINISHED : k0, u_now, now, step);
        if (kMode == 1 && rq >= a1) {  // overrun request: side buffer
          int64_t* sp = sx->side + 2 * (int64_t)(rq - a1);
          if (k0 == TW_EV_FIRST_TOKEN) sp[0] = now;
          if (nev == 2) sp[1] = now;
        } else {
          if (k0 == TW_EV_FIRST_TOKEN && em.first) em.first[rq] = now;
          if (nev == 2 && em.finish) em.finish[rq] = now;
        }
      }
      pos_c += __popc(c1) + __popc(c2);
      pos_d += __popc(d1) + __popc(d2);
#ifdef TWB_SIM_CHECK
      if (v) {
        const int32_t held1 = max(blk.ceil_div(pr), blk.ceil_div(dn + e));
        chk_kv += (int64_t)held1 - held0 - (fin ? held1 : 0);  // _finish frees the final hold
        if (dn > pr || e > op) chk[2]++;
      }
#endif
      // stable removal of finished requests (oracle.py:111-112)
      const bool keep = v && !fin;
      const unsigned km = __ballot_sync(kFull, keep);
      __syncwarp();
      if (keep) {
        const int np = kept + __popc(km & lt);
        sl.req[np] = rq;
        sl.prompt[np] = pr;
        sl.output[np] = op;
        sl.done[np] = dn;
        sl.emit[np] = e;
      }
      kept += __popc(km);
      __syncwarp();
    }
    n_events = pos_d;
    n_act = kept;
#ifdef TWB_SIM_CHECK
    {
      // recompute the blocks the active set holds and compare with the incremental counter
      int64_t held_l = 0;
      for (int b = 0; b < n_act; b += 32) {
        const int i = b + lane;
        if (i < n_act) held_l += max(blk.ceil_div(sl.prompt[i]), blk.ceil_div(sl.done[i] + sl.emit[i]));
      }
      __syncwarp();
      int64_t kv = chk_kv;  // lane partials can be negative (finishes): plain shuffle sum
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) kv += __shfl_xor_sync(kFull, kv, o);
      if (warp_sum_i64_redux(held_l) != kv) chk[3]++;
      chk[0]++;
      if (now < chk_now) chk[1]++;
      chk_now = now;
      if (tk_on) {
        if (g.offset < chk_off || g.seq < chk_seq || g.wall < chk_wall) chk[4]++;
        if (g.V != g.wall + g.offset || g.V < now) chk[5]++;
        if (g.last_bcast != INT64_MIN && g.last_bcast > g.wall) chk[6]++;
        chk_off = g.offset;
        chk_seq = g.seq;
        chk_wall = g.wall;
      }
    }
#endif
    if (n_adm) {
      w_head += n_adm;
      qbase = w_head;
      q_pr = (qbase + lane < n) ? __ldg(prm + qbase + lane) : 0;
      q_op = (qbase + lane < n) ? __ldg(outp + qbase + lane) : 0;
    }
    apply_cyc += TWB_CLK() - q4;
  }

  if (em.evp && n_events > em.ev_cap) overflow = 1;
#ifdef TWB_SIM_CHECK
  if (r.status == TW_SIM_OK) {
    int64_t want_l = 0;
    for (int i = lane; i < n; i += 32) want_l += (int64_t)max(__ldg(outp + i), 1) + 1;
    if (warp_sum_i64_redux(want_l) != n_events) chk[7]++;
  }
  if (p.checks && lane == 0)
    for (int k = 0; k < 8; k++) p.checks[8 * (int64_t)c + k] = chk[k];
#endif

  // digest: sum of lane partials mod 2^64
  uint64_t dig = em.dig;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dig += __shfl_xor_sync(kFull, dig, o);
  if constexpr (kMode != 0) {
    uint64_t ms = em.msum;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ms += __shfl_xor_sync(kFull, ms, o);
    SegSummary o;
    o.j_stop = (r.status == TW_SIM_OK) ? j_stop : fut;
    o.status = r.status;
    o.last_regen = last_regen;
    o.adm_end = w_head;
    o.final_now = now;
    o.events = n_events;
    o.dig = dig;
    o.msum = ms;
    o.steps = step;
    o.pred_code = r.pred_code;
    o.log_len = log_len;
    o.pad = 0;
    o.tk = tk_state(g);  // mode 1: filled in by the replay (k_seg_tk)
    o.d_lo = g.d_lo;
    o.d_hi = g.d_hi;
    if constexpr (kMode == 1) sx->log_len = log_len;
    if constexpr (kMode == 1) {
      __syncwarp();
      if (lane == 0) *sx->sum = o;
    } else {
      sx->out = o;
    }
    return;
  }
  r.final_now_ns = now;
  r.steps = step;
  r.events = n_events;
  r.digest = dig;
  if (tk_on) {
    r.tk_seq = g.seq;
    r.tk_offset_ns = g.offset;
    r.tk_wall_ns = g.wall;
  }
  if (overflow) r.status |= 1 << 8;
  // the record is the config's completion signal: a host watching records in pinned memory
  // (HostSweep's streamed copy-back) may copy the config's stamps as soon as it sees it, so
  // every lane's stamp stores must be visible system-wide first
  __syncwarp();
  if (lane == 0) {
    __threadfence_system();
    p.res[c] = r;
    if (p.prof) {
#ifdef TWB_PROFILE_PHASES
      int64_t* q = p.prof + 32 * c;
      q[16] = x_walk_cyc;
      q[17] = x_fast_cyc;
      q[18] = pc.miss_cyc;
      q[19] = x_it_adm;
      q[20] = x_it_wait;
      q[21] = x_it_wide;
      q[22] = x_body_cyc;
      q[23] = x_it_chunk;
      q[24] = x_it_k1;
      q[25] = x_it_idle;
      q[26] = x_idle_cyc;
#else
      int64_t* q = p.prof + 16 * c;
#endif
      q[0] = clock64() - t_start;
      q[1] = n_normal;
      q[2] = n_runs;
      q[3] = n_run_steps;
      q[4] = tk_cyc;
      q[5] = ev_cyc;
      q[6] = g.seq;
      q[7] = arr_cyc;
      q[8] = plan_cyc;
      q[9] = adm_cyc;
      q[10] = pred_cyc;
      q[11] = apply_cyc;
      q[12] = pc.misses;
#ifdef TWB_PROFILE_PHASES
      q[13] = g.prof_calls;
      q[14] = g.prof_fast;
      q[15] = g.prof_loops;
#endif
    }
  }
}

#ifndef TWB_SIM_MIN_BLOCKS
#define TWB_SIM_MIN_BLOCKS 1
#endif
#ifndef TWB_SIM_TPUT_MIN_BLOCKS
#define TWB_SIM_TPUT_MIN_BLOCKS 4
#endif
// Two variants of the same loop (profiles/README.md, session-4 occupancy A/B):
//  * latency (kTput = false): every config has its own warp; the blob is staged in shared
//    memory (4 shared loads per prediction-cache miss), registers unconstrained (164);
//  * throughput (kTput = true, more configs than resident warps): 4 CTAs per SM at <= 128
//    registers, the blob read through L1 so shared memory holds only slot state
//    (16 warps per SM instead of 12: 65,536 configs 335 -> 289 ms).
// kGSlots (sim_big.cu only): slot capacities above kMaxSlotCap keep each warp's slot
// state in a global scratch slice instead of shared memory (max_running has no limit in
// the reference); the blob is read from global memory as in the throughput variant.
template <bool kTput, bool kGSlots = false, bool kCheck = false>
__global__ void __launch_bounds__(kSimThreads, kTput ? TWB_SIM_TPUT_MIN_BLOCKS : TWB_SIM_MIN_BLOCKS)
    k_sim(SimParams p) {
  extern __shared__ __align__(128) char smem[];
  // (one expression, so ptxas still sees the staged blob as shared memory: LDS, not LD)
  const char* ps = kTput ? static_cast<const char*>(p.pset) : smem + 128;
  if constexpr (!kTput) tma_stage_to_smem(smem + 128, p.pset, p.pset_bytes, reinterpret_cast<uint64_t*>(smem));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t* base;
  if constexpr (kGSlots) base = p.gslots + ((size_t)blockIdx.x * (blockDim.x >> 5) + warp) * 7 * (size_t)p.cap;
  else base = reinterpret_cast<int32_t*>(smem + 128 + p.pset_smem) + (size_t)warp * 7 * p.cap;
  Slots sl;
  sl.req = base;
  sl.prompt = base + p.cap;
  sl.output = base + 2 * p.cap;
  sl.done = base + 3 * p.cap;
  sl.emit = base + 4 * p.cap;
  sl.plan = base + 5 * p.cap;
  sl.dlist = base + 6 * p.cap;
  for (;;) {
    int idx = 0;
    if (lane == 0) idx = atomicAdd(p.counter, 1);
    idx = __shfl_sync(kFull, idx, 0);
    if (idx >= p.n_cfg) break;
    const int c = p.order ? p.order[idx] : idx;
    run_config<kTput>(p, ps, sl, c);
    __syncwarp();

  }
}

#ifdef TWB_SIM_SEG_TU
// ---- busy-period segments: planner, speculative segments, join (sim_seg.cu) -------------

// Segment boundaries: W = min(wmax, n / min_req) equal shares of the arrivals, each
// boundary moved (within +-15 arrivals) to the largest inter-arrival gap, where the
// engine is most likely to be empty. One warp per config.
__global__ void __launch_bounds__(128) k_seg_plan(SimParams p, SegParams q) {
  // block (x = config, y = share of its boundaries); the warps of the grid's y dimension
  // split the boundaries (a single config has up to 255 of them)
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x;
  const int wy = blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5), ny = gridDim.y * (blockDim.x >> 5);
  if (c >= p.n_cfg) return;
  const tw_sim_cfg cfg = p.cfgs[c];
  const int64_t wl0 = p.wl_off[cfg.workload_id];
  const int32_t n = (int32_t)(p.wl_off[cfg.workload_id + 1] - wl0);
  const int64_t* __restrict__ ts = p.ts + wl0;
  int32_t W = n / q.min_req;
  W = W < 1 ? 1 : (W > q.wmax ? q.wmax : W);
  if (p.req_base[p.n_cfg] > q.r_max) W = 0;  // scratch too small for the per-request records
  if (lane == 0 && wy == 0) {
    q.nseg[c] = W;
    q.seg_a0[(int64_t)c * q.wmax] = 0;
  }
  if (W <= 1) return;
  const int32_t len = n / W;
  const int32_t h = min(15, len / 2 - 1);
  for (int k = 1 + wy; k < W; k += ny) {
    const int32_t center = (int32_t)((int64_t)k * n / W);
    const int32_t j = center - h + lane;
    int64_t gap = -1;
    if (lane <= 2 * h && j >= 1 && j < n) gap = __ldg(ts + j) - __ldg(ts + j - 1);
    const int64_t best = -warp_min_i64(-gap);
    const unsigned m = __ballot_sync(kFull, gap == best);
    if (lane == 0) q.seg_a0[(int64_t)c * q.wmax + k] = center - h + (__ffs(m) - 1);
  }
}

// A segment's Timekeeper, replayed from its log after the run (a tight loop of its own,
// so the event loop's code stays small): the config's start state for segment 0, else a
// guess at arrival a0 (just broadcast, so last broadcast = wall; every earlier arrival
// dispatched; wall 0). Records the state at each regeneration point and at the stop, and
// the wall shifts [d_lo, d_hi) that keep every decision (tk_compose checks the truth).
#ifdef TWB_SEG_REPLAY_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
void seg_tk_replay(const SimParams& p, int c, int32_t a0, int32_t a1, int32_t n,
                                           const TkLog* __restrict__ log, int32_t len_log,
                                           const int32_t* __restrict__ regpos, SegRegen* reg, SegSummary* sum) {
  const int lane = threadIdx.x & 31;
  const tw_sim_cfg cfg = p.cfgs[c];
  const int64_t wl0 = p.wl_off[cfg.workload_id];
  const int64_t* __restrict__ ts = p.ts + wl0;
  const int64_t epoch = cfg.epoch_ns;
  const int S = cfg.pp_stages;
  TkGrid g;
  g.cooldown = cfg.tk_cooldown_ns;
  g.conv_cooldown = g.cooldown > 0 ? cold_fake_sleep(g.cooldown) : 0;
  g.rcp_cooldown = g.conv_cooldown > 0 ? __drcp_rn(__ll2double_rn(g.conv_cooldown)) : 0.0;
  g.seq = 0;
  g.d_lo = INT64_MIN;
  g.d_hi = INT64_MAX;
#ifdef TWB_PROFILE_PHASES
  g.prof_calls = g.prof_fast = g.prof_loops = 0;
#endif
  if (a0 == 0) {
    g.wall = epoch;
    g.offset = 0;
    g.last_bcast = INT64_MIN;
    g.V = epoch;
  } else {
    g.wall = 0;
    g.offset = 0;
    g.last_bcast = 0;
    g.V = 0;
  }
  g.disp = a0;
  g.win.load(ts, n, epoch, a0);
  g.disp_ts = a0 < n ? __shfl_sync(kFull, g.win.v, 0) : INT64_MAX;
  // the regeneration points in order: jn (next), pn its log position
  int32_t jn = a0, pn = 0;
  auto next_regen = [&](int32_t from) {  // first j >= from in [from, a1) with regpos[j] >= 0
    for (int32_t b = from; b < a1; b += 32) {
      const int32_t j = b + lane;
      const unsigned m = __ballot_sync(kFull, j < a1 && regpos[j] >= 0);
      if (m) {
        jn = b + __ffs(m) - 1;
        pn = regpos[jn];
        return;
      }
    }
    jn = a1;
    pn = INT32_MAX;
  };
  auto mark = [&](int32_t idx) {  // states at the regeneration points logged at idx
    while (pn == idx) {
      if (lane == 0) reg[jn].tk = tk_state(g);
      next_regen(jn + 1);
    }
  };
#pragma unroll 1
  for (int32_t b = 0; b < len_log; b += 32) {
    int64_t x0 = 0, x1 = 0, x2 = 0;
    if (b + lane < len_log) {
      const TkLog* e = log + b + lane;
      x0 = e->now0;
      x1 = e->d;
      x2 = e->K;
    }
    const int m = min(32, len_log - b);
#pragma unroll 1
    for (int k = 0; k < m; k++) {
      mark(b + k);
      const int64_t now0 = __shfl_sync(kFull, x0, k), d = __shfl_sync(kFull, x1, k), K = __shfl_sync(kFull, x2, k);
      if (K == 0) tk_idle<true>(g, ts, n, epoch, now0);
      else tk_run<true>(g, ts, n, epoch, S, now0, d, K);
    }
  }
  mark(len_log);
  if (lane == 0) {
    sum->tk = tk_state(g);
    sum->d_lo = g.d_lo;
    sum->d_hi = g.d_hi;
  }
}

// Speculative segments: warps pull (config, segment) pairs, heaviest configs first.
// kLat: the latency variant's geometry instead (blob staged in shared memory, registers
// up to 3 CTAs per SM), an A/B alternative (TWB_SIM_SEG_LAT)
template <bool kLat>
__global__ void __launch_bounds__(kSimThreads, kLat ? 3 : TWB_SIM_TPUT_MIN_BLOCKS) k_sim_seg(SimParams p, SegParams q) {
  extern __shared__ __align__(128) char smem[];
  const char* ps = kLat ? smem + 128 : static_cast<const char*>(p.pset);
  if constexpr (kLat) tma_stage_to_smem(smem + 128, p.pset, p.pset_bytes, reinterpret_cast<uint64_t*>(smem));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t* base = reinterpret_cast<int32_t*>(smem + 128 + p.pset_smem) + (size_t)warp * 7 * p.cap;
  Slots sl;
  sl.req = base;
  sl.prompt = base + p.cap;
  sl.output = base + 2 * p.cap;
  sl.done = base + 3 * p.cap;
  sl.emit = base + 4 * p.cap;
  sl.plan = base + 5 * p.cap;
  sl.dlist = base + 6 * p.cap;
  const int64_t n_items = (int64_t)p.n_cfg * q.wmax;
  for (;;) {
    int64_t idx = 0;
    if (lane == 0) idx = (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(q.counter), 1ULL);
    idx = __shfl_sync(kFull, idx, 0);
    if (idx >= n_items) break;
    const int32_t rank = (int32_t)(idx / q.wmax), w = (int32_t)(idx - (int64_t)rank * q.wmax);
    const int c = p.order ? p.order[rank] : rank;
    const int32_t W = q.nseg[c];
    if (w >= W) continue;
    const tw_sim_cfg& cfg = p.cfgs[c];
    const int32_t n = (int32_t)(p.wl_off[cfg.workload_id + 1] - p.wl_off[cfg.workload_id]);
    const int64_t rb = p.req_base[c];
    SegCtx sx;
    sx.a0 = q.seg_a0[(int64_t)c * q.wmax + w];
    sx.a1 = (w + 1 < W) ? q.seg_a0[(int64_t)c * q.wmax + w + 1] : n;
    const int32_t len = sx.a1 - sx.a0;
    const int64_t unit = rb + sx.a0 + q.xtra * ((int64_t)c * q.wmax + w);  // this segment's room
    sx.log = q.log + (int64_t)kSegLogPerReq * unit;
    sx.log_cap = (int32_t)(kSegLogPerReq * (len + q.xtra) / q.cap_div);
    sx.side = q.side + 8 * unit;
    sx.side_cap = (int32_t)(4 * (len + q.xtra) / q.cap_div);
    sx.regpos = q.regpos + rb;
    sx.reg = q.reg + rb;
    sx.g = nullptr;
    sx.sum = q.summ + (int64_t)c * q.wmax + w;
    run_config<!kLat, 1>(p, ps, sl, c, &sx);
    __syncwarp();
    if (lane == 0) {
      sx.sum->log_len = sx.log_len;
      __threadfence();
      *reinterpret_cast<volatile int32_t*>(&sx.sum->pad) = q.epoch;  // the segment is done
    }
    __syncwarp();
  }
#ifdef TWB_SEG_TAIL_REPLAY
  // A/B: with the segments handed out, the warps replay the Timekeeper logs themselves
  // (waiting for segments still running), filling the kernel's tail
  for (;;) {
    int64_t idx = 0;
    if (lane == 0) idx = (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(q.counter + 4), 1ULL);
    idx = __shfl_sync(kFull, idx, 0);
    if (idx >= n_items) break;
    const int32_t rank = (int32_t)(idx / q.wmax), w = (int32_t)(idx - (int64_t)rank * q.wmax);
    const int c = p.order ? p.order[rank] : rank;
    const int32_t W = q.nseg[c];
    if (w >= W) continue;
    const tw_sim_cfg& cfg = p.cfgs[c];
    if (!(cfg.flags & TW_SIM_TIMEKEEPER)) continue;
    SegSummary* sum = q.summ + (int64_t)c * q.wmax + w;
    while (*reinterpret_cast<volatile int32_t*>(&sum->pad) != q.epoch) __nanosleep(256);
    __threadfence();
    const int32_t n = (int32_t)(p.wl_off[cfg.workload_id + 1] - p.wl_off[cfg.workload_id]);
    if (sum->status == TW_SIM_BAD_CONFIG || sum->status == TW_SIM_CAPACITY || n == 0) continue;
    const int64_t rb = p.req_base[c];
    const int32_t a0 = q.seg_a0[(int64_t)c * q.wmax + w];
    const int32_t a1 = (w + 1 < W) ? q.seg_a0[(int64_t)c * q.wmax + w + 1] : n;
    seg_tk_replay(p, c, a0, a1, n, q.log + (int64_t)kSegLogPerReq * (rb + a0 + q.xtra * ((int64_t)c * q.wmax + w)),
                  sum->log_len, q.regpos + rb, q.reg + rb, sum);
  }
#endif
}

// The segments' Timekeeper replays, one warp per (config, segment), in a kernel of their
// own: inside k_sim_seg the replay loop next to the event loop pushed the kernel's code
// past the instruction caches (ncu: stall_no_inst 46%, 7.3 ms vs 3.8 + this kernel).
#ifndef TWB_SEG_TK_BLOCKS
#define TWB_SEG_TK_BLOCKS 6
#endif
__global__ void __launch_bounds__(128, TWB_SEG_TK_BLOCKS) k_seg_tk(SimParams p, SegParams q) {
  const int lane = threadIdx.x & 31;
  const int64_t n_items = (int64_t)p.n_cfg * q.wmax;
  for (;;) {  // persistent warps pull segments (their logs differ in length)
    int64_t idx = 0;
    if (lane == 0) idx = (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(q.counter + 4), 1ULL);
    idx = __shfl_sync(kFull, idx, 0);
    if (idx >= n_items) break;
    const int32_t rank = (int32_t)(idx / q.wmax), w = (int32_t)(idx - (int64_t)rank * q.wmax);
    const int c = p.order ? p.order[rank] : rank;
    const int32_t W = q.nseg[c];
    if (w >= W) continue;
    const tw_sim_cfg& cfg = p.cfgs[c];
    if (!(cfg.flags & TW_SIM_TIMEKEEPER)) continue;
    const int32_t n = (int32_t)(p.wl_off[cfg.workload_id + 1] - p.wl_off[cfg.workload_id]);
    const int64_t rb = p.req_base[c];
    const int32_t a0 = q.seg_a0[(int64_t)c * q.wmax + w];
    const int32_t a1 = (w + 1 < W) ? q.seg_a0[(int64_t)c * q.wmax + w + 1] : n;
    SegSummary* sum = q.summ + (int64_t)c * q.wmax + w;
    if (sum->status == TW_SIM_BAD_CONFIG || sum->status == TW_SIM_CAPACITY || a0 >= n) continue;
    seg_tk_replay(p, c, a0, a1, n, q.log + (int64_t)kSegLogPerReq * (rb + a0 + q.xtra * ((int64_t)c * q.wmax + w)),
                  sum->log_len, q.regpos + rb,
                  q.reg + rb, sum);
    (void)lane;
  }
}

// Carries the true Timekeeper g across a speculative piece: E is the piece's speculative
// state before the idle round at its entry arrival j, T its state at the piece's end,
// [d_lo, d_hi) the wall shifts its decisions allow. Both runs are empty at j; the idle
// round at j lands both on V = ts_j after the same sleep when (a) both dispatchers wait
// for arrival j, (b) last broadcast - wall agree, (c) both V lie below ts_j - sleep. From
// there the true run is the speculative one with its wall shifted by delta (offset by
// -delta), provided delta keeps every wall decision. Returns false when that cannot be
// shown (the caller re-runs the piece serially); `exact` (the config's own start) copies.
__device__ __forceinline__ bool tk_compose(TkGrid& g, const TkState& E, const TkState& T, int64_t d_lo,
                                           int64_t d_hi, bool exact, int32_t j, int64_t tj) {
  int64_t delta = 0;
  if (!exact && T.seq == E.seq) {
    // no broadcast in the piece: it is empty (entry = exit, e.g. a segment out of room at
    // its entry) and the true state stands; anything else cannot be shown to carry over
    return T.wall == E.wall && T.offset == E.offset && T.last_bcast == E.last_bcast && T.disp == E.disp;
  }
  if (!exact) {
    if (g.disp != j || E.disp != j) return false;
    const bool set_t = g.last_bcast != INT64_MIN, set_e = E.last_bcast != INT64_MIN;
    if (set_t != set_e || (set_t && g.last_bcast - g.wall != E.last_bcast - E.wall)) return false;
    int64_t slp = 0;
    if (set_t && g.cooldown > 0) {
      const int64_t wait = g.last_bcast + g.cooldown - g.wall;
      if (wait > 0) slp = (wait == g.cooldown) ? g.conv_cooldown : cold_fake_sleep(wait);
    }
    if (!(g.wall + g.offset < tj - slp) || !(E.wall + E.offset < tj - slp)) return false;
    delta = g.wall - E.wall;
    if (delta < d_lo || delta >= d_hi) return false;
  }
  g.wall = T.wall + delta;
  g.seq += T.seq - E.seq;
  g.last_bcast = T.last_bcast == INT64_MIN ? INT64_MIN : T.last_bcast + delta;
  g.offset = T.offset - delta;
  g.V = g.wall + g.offset;
  g.disp = T.disp;  // the dispatcher's window is reloaded only before a serial piece
  return true;
}

// The join pass: one warp per config walks the chain of valid pieces (a segment from its
// entry point to its stop; where a segment's stop is not a regeneration point of the next
// run, or its Timekeeper cannot be carried over, a serial piece in mode 2 until the chain
// meets a regeneration point again), adds each piece's counters in the true frame
// (positions and steps shifted: digest += msum * (dk*A + ds*G)), carries the Timekeeper,
// copies overrun stamps and writes the config's record.
__global__ void __launch_bounds__(kSimThreads, 1) k_sim_join(SimParams p, SegParams q) {
  extern __shared__ __align__(128) char smem[];
  const char* ps = static_cast<const char*>(p.pset);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t* base = reinterpret_cast<int32_t*>(smem + 128) + (size_t)warp * 7 * p.cap;
  Slots sl;
  sl.req = base;
  sl.prompt = base + p.cap;
  sl.output = base + 2 * p.cap;
  sl.done = base + 3 * p.cap;
  sl.emit = base + 4 * p.cap;
  sl.plan = base + 5 * p.cap;
  sl.dlist = base + 6 * p.cap;
  for (;;) {
    int idx = 0;
    if (lane == 0) idx = atomicAdd(q.counter + 2, 1);
    idx = __shfl_sync(kFull, idx, 0);
    if (idx >= p.n_cfg) break;
    const int c = p.order ? p.order[idx] : idx;
    const tw_sim_cfg cfg = p.cfgs[c];
    const int64_t wl0 = p.wl_off[cfg.workload_id];
    const int32_t n = (int32_t)(p.wl_off[cfg.workload_id + 1] - wl0);
    const int64_t* __restrict__ ts = p.ts + wl0;
    const int64_t epoch = cfg.epoch_ns;
    const bool tk_on = (cfg.flags & TW_SIM_TIMEKEEPER) != 0;
    const int64_t rb = p.req_base[c];
    const int32_t W = q.nseg[c];
    // the segment starts and their arrival times in shared memory (the chain reads them at
    // every piece), and the next segment's summary loaded ahead of its turn
    int64_t* ta0 = reinterpret_cast<int64_t*>(smem + 128 + (size_t)(blockDim.x >> 5) * 7 * 4 * p.cap) +
                   (size_t)warp * 2 * q.wmax;
    int32_t* a0s = reinterpret_cast<int32_t*>(ta0 + q.wmax);
    for (int32_t k = lane; k < W; k += 32) {
      const int32_t a = q.seg_a0[(int64_t)c * q.wmax + k];
      a0s[k] = a;
      ta0[k] = a < n ? epoch + __ldg(ts + a) : INT64_MAX;
    }
    __syncwarp();
    const SegSummary* sm = q.summ + (int64_t)c * q.wmax;
    int32_t* regpos = q.regpos + rb;
    SegRegen* reg = q.reg + rb;
    int64_t* first = p.first ? p.first + rb : nullptr;
    int64_t* finish = p.finish ? p.finish + rb : nullptr;

    TkGrid g;
    g.wall = epoch;
    g.offset = 0;
    g.seq = 0;
    g.last_bcast = INT64_MIN;
    g.V = epoch;
    g.cooldown = cfg.tk_cooldown_ns;
    g.conv_cooldown = g.cooldown > 0 ? cold_fake_sleep(g.cooldown) : 0;
    g.rcp_cooldown = g.conv_cooldown > 0 ? __drcp_rn(__ll2double_rn(g.conv_cooldown)) : 0.0;
    g.disp = 0;
    g.d_lo = INT64_MIN;
    g.d_hi = INT64_MAX;
#ifdef TWB_PROFILE_PHASES
    g.prof_calls = g.prof_fast = g.prof_loops = 0;
#endif
    g.win.load(ts, n, epoch, 0);
    g.disp_ts = n > 0 ? __shfl_sync(kFull, g.win.v, 0) : INT64_MAX;

    int64_t ev_t = 0, now_t = epoch;
    uint64_t dig_t = 0;
    int32_t st_t = 0, status = TW_SIM_OK, pred_code = 0, adm_end = 0;
    bool invalid_cfg = false;
    // a piece's counters relative to its entry record e, moved into the true frame
    auto add = [&](int64_t ev, uint64_t dg, uint64_t ms, int32_t st, const SegRegen& e) {
      const uint64_t dm = ms - e.msum;
      dig_t += (dg - e.dig) +
               ((uint64_t)(ev_t - e.events) * TW_DIG_A + (uint64_t)(int64_t)(st_t - e.steps) * TW_DIG_G) * dm;
      ev_t += ev - e.events;
      st_t += st - e.steps;
    };
    auto copy_side = [&](int32_t w, int32_t lo, int32_t hi) {  // overrun stamps of segment w
      const int64_t* side = q.side + 8 * (rb + a0s[w] + q.xtra * ((int64_t)c * q.wmax + w));
      const int32_t a1 = (w + 1 < W) ? a0s[w + 1] : n;
      for (int32_t i = lo + lane; i < hi; i += 32) {
        if (first) first[i] = side[2 * (int64_t)(i - a1)];
        if (finish) finish[i] = side[2 * (int64_t)(i - a1) + 1];
      }
    };
    auto owner = [&](int32_t j) {
      int32_t lo = 0, hi = W - 1;  // the last segment whose first arrival is <= j
      while (lo < hi) {
        const int32_t mid = (lo + hi + 1) >> 1;
        if (a0s[mid] <= j) lo = mid;
        else hi = mid - 1;
      }
      return lo;
    };

    int32_t w = 0, j_in = 0, js = 0, n_joined = 0, n_serial = 0, n_tkfail = 0, n_ovf = 0, n_noconv = 0;
    SegRegen e{};
    bool exact = true;     // the chain's first piece starts with the config (no guess)
    bool serial = W == 0;  // not segmented: the whole config serially from arrival 0
    SegSummary s_next;
    int32_t w_next = -1;
    for (;;) {
      if (!serial) {
        const SegSummary s = (w == w_next) ? s_next : sm[w];
        if (w + 1 < W) {  // the usual successor, fetched while this piece is joined
          s_next = sm[w + 1];
          w_next = w + 1;
        }
        const int32_t a1w = (w + 1 < W) ? a0s[w + 1] : n;
        const int64_t tj = (j_in == a0s[w]) ? ta0[w] : epoch + __ldg(ts + j_in);
        if (s.status == TW_SIM_BAD_CONFIG || s.status == TW_SIM_CAPACITY) {
          status = s.status;
          invalid_cfg = true;
          break;
        }
        if (exact) e = SegRegen{};  // the config's start: zero counters, Timekeeper seq 0
        if (s.status == kSegOverflow) {
          // valid from the entry up to its last regeneration point, serial from there
          n_ovf++;
          const int32_t jr = s.last_regen;
          const SegRegen E = reg[jr];
          if (!tk_on || tk_compose(g, e.tk, E.tk, s.d_lo, s.d_hi, exact, j_in, tj)) {
            add(E.events, E.dig, E.msum, E.steps, e);
            js = jr;
          } else {
            js = j_in;
            n_tkfail++;
          }
          serial = true;
        } else if (tk_on && !tk_compose(g, e.tk, s.tk, s.d_lo, s.d_hi, exact, j_in, tj)) {
          js = j_in;  // the Timekeeper guess does not carry over: this piece serially
          serial = true;
          n_tkfail++;
        } else {
          n_joined++;
          add(s.events, s.dig, s.msum, s.steps, e);
          now_t = s.final_now;
          if (s.status != TW_SIM_OK) {
            status = s.status;
            pred_code = s.pred_code;
            adm_end = s.adm_end;
            if (adm_end > a1w) copy_side(w, a1w, adm_end);
            break;
          }
          if (s.j_stop > a1w) copy_side(w, a1w, s.j_stop);
          if (s.j_stop >= n) break;
          js = s.j_stop;
          if (w + 1 < W && a0s[w + 1] == js) {  // the usual case: the next segment's start
            w++;
            e = SegRegen{0, 0, 0, 0, 0, TkState{0, 0, 0, 0, js, 0}};  // k_seg_tk's guess at a0
            j_in = js;
            exact = false;
            continue;
          }
          if (regpos[js] >= 0) {  // the owner's run was empty at js too: continue with it
            w = owner(js);
            e = reg[js];
            j_in = js;
            exact = false;
            continue;
          }
          n_noconv++;
          serial = true;
        }
      }
      // a serial piece from arrival js (the engine empty there), the true Timekeeper inline
      g.win.load(ts, n, epoch, g.disp);
      g.disp_ts = g.disp < n ? __shfl_sync(kFull, g.win.v, 0) : INT64_MAX;
      SegCtx sx;
      sx.a0 = js;
      sx.a1 = n;
      sx.side = nullptr;
      sx.side_cap = 0;
      sx.regpos = W > 0 ? regpos : nullptr;
      sx.reg = reg;
      sx.g = &g;
      sx.sum = nullptr;
      run_config<true, 2>(p, ps, sl, c, &sx);
      n_serial++;
      const SegSummary s2 = sx.out;
      const SegRegen z{};
      if (s2.status == TW_SIM_BAD_CONFIG || s2.status == TW_SIM_CAPACITY) {
        status = s2.status;
        invalid_cfg = true;
        break;
      }
      add(s2.events, s2.dig, s2.msum, s2.steps, z);
      now_t = s2.final_now;
      if (s2.status != TW_SIM_OK) {
        status = s2.status;
        pred_code = s2.pred_code;
        adm_end = s2.adm_end;
        break;
      }
      if (s2.j_stop >= n) break;
      js = s2.j_stop;  // converged: a regeneration point of its owner's run
      w = owner(js);
      e = reg[js];
      j_in = js;
      exact = false;
      serial = false;
    }
    if (status != TW_SIM_OK && !invalid_cfg && W > 0) {
      // the run stopped early: requests a speculative segment stamped past the stop are
      // reset to unset (-1)
      for (int32_t v = 0; v < W; v++) {
        const int32_t a0v = a0s[v], a1v = (v + 1 < W) ? a0s[v + 1] : n;
        const int32_t lo = max(a0v, adm_end), hi = min(a1v, sm[v].adm_end);
        for (int32_t i = lo + lane; i < hi; i += 32) {
          if (first) first[i] = -1;
          if (finish) finish[i] = -1;
        }
      }
    }
    tw_sim_result r;
    r.final_now_ns = invalid_cfg ? epoch : now_t;
    r.steps = invalid_cfg ? 0 : st_t;
    r.events = invalid_cfg ? 0 : ev_t;
    r.digest = invalid_cfg ? 0 : dig_t;
    r.tk_seq = 0;
    r.tk_offset_ns = 0;
    r.tk_wall_ns = 0;
    if (tk_on && !invalid_cfg) {
      r.tk_seq = g.seq;
      r.tk_offset_ns = g.offset;
      r.tk_wall_ns = g.wall;
    }
    r.status = status;
    r.pred_code = pred_code;
    __syncwarp();
    if (lane == 0) {
      __threadfence_system();
      p.res[c] = r;
      if (q.stats) {
        int32_t* st = q.stats + 8 * (int64_t)c;
        st[0] = W;
        st[1] = n_joined;
        st[2] = n_serial;
        st[3] = n_tkfail;
        st[4] = n_ovf;
        st[5] = n_noconv;
        st[6] = 0;
        st[7] = 0;
      }
    }
    __syncwarp();
  }
}

int sim_seg_prepare(int threads, size_t smem, int* per_sm, bool lat) {
  if (lat) {
    cudaFuncSetAttribute(k_sim_seg<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, k_sim_seg<true>, threads, smem);
  }
  cudaFuncSetAttribute(k_sim_seg<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, k_sim_seg<false>, threads, smem);
}
void sim_seg_launch(int grid, int threads, size_t smem, cudaStream_t s, const SimParams& p, const SegParams& q,
                    int join_grid, bool lat, size_t join_smem, uint32_t join_pset_bytes) {
  k_seg_plan<<<dim3((unsigned)p.n_cfg, (unsigned)std::min(64, (q.wmax + 3) / 4)), 128, 0, s>>>(p, q);
  if (lat) k_sim_seg<true><<<grid, threads, smem, s>>>(p, q);
  else k_sim_seg<false><<<grid, threads, smem, s>>>(p, q);
  const int64_t items = (int64_t)p.n_cfg * q.wmax;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_seg_tk, 128, 0);
  k_seg_tk<<<(int)std::min<int64_t>((items + 3) / 4, (int64_t)sms * std::max(per_sm, 1)), 128, 0, s>>>(p, q);
  cudaFuncSetAttribute(k_sim_join, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)join_smem);
  SimParams pj = p;  // the join reads the whole blob from global memory
  pj.pset_smem = 0;
  pj.pset_bytes = join_pset_bytes;
  k_sim_join<<<join_grid, threads, join_smem, s>>>(pj, q);
}
}  // namespace twb
#elif defined(TWB_SIM_TPUT_TU)
// sim_tput.cu compiles this file a second time for the throughput variant alone: with
// both variants in one translation unit the shared helpers stop being inlined into the
// latency variant, whose blob reads then turn from LDS into generic loads (164 -> 173
// registers, 1-2% slower at 1,024 configs).
#if defined(TWB_SIM_CHECK)
int sim_check_prepare(int threads, size_t smem, int* per_sm) {
  cudaFuncSetAttribute(k_sim<true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, k_sim<true, false, true>, threads, smem);
}
void sim_check_launch(int grid, int threads, size_t smem, cudaStream_t s, const SimParams& p) {
  k_sim<true, false, true><<<grid, threads, smem, s>>>(p);
}
#elif defined(TWB_SIM_BIG_TU)
int sim_big_prepare(int threads, int* per_sm) {
  return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, k_sim<true, true>, threads, 128);
}
void sim_big_launch(int grid, int threads, cudaStream_t s, const SimParams& p) {
  k_sim<true, true><<<grid, threads, 128, s>>>(p);
}
#else
int sim_tput_prepare(int threads, size_t smem, int* per_sm) {
  cudaFuncSetAttribute(k_sim<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, k_sim<true>, threads, smem);
}
void sim_tput_launch(int grid, int threads, size_t smem, cudaStream_t s, const SimParams& p) {
  k_sim<true><<<grid, threads, smem, s>>>(p);
}
#endif
}  // namespace twb
#else
int sim_tput_prepare(int threads, size_t smem, int* per_sm);  // sim_tput.cu
void sim_tput_launch(int grid, int threads, size_t smem, cudaStream_t s, const SimParams& p);
int sim_big_prepare(int threads, int* per_sm);  // sim_big.cu
void sim_big_launch(int grid, int threads, cudaStream_t s, const SimParams& p);
int sim_check_prepare(int threads, size_t smem, int* per_sm);  // sim_check.cu
void sim_check_launch(int grid, int threads, size_t smem, cudaStream_t s, const SimParams& p);
int sim_seg_prepare(int threads, size_t smem, int* per_sm, bool lat);  // sim_seg.cu
void sim_seg_launch(int grid, int threads, size_t smem, cudaStream_t s, const SimParams& p, const SegParams& q,
                    int join_grid, bool lat, size_t join_smem, uint32_t join_pset_bytes);
static thread_local int32_t* g_checks = nullptr;

// ---- busy-period segments (latency regime): scratch layout ----------------------------
// [64 B counters | nseg[n_cfg] | seg_a0[n_cfg*W] | summ[n_cfg*W] |
//  regpos[R] | reg[R] | log[kSegLogPerReq*(R+X)] | side[8*(R+X)]], X = xtra * segments,
//  R (request capacity) = what the rest of scratch holds
static int seg_min_req() {  // requests per segment at least (TWB_SIM_SEG_MINREQ: A/B only)
  const char* e = getenv("TWB_SIM_SEG_MINREQ");
  const int v = e ? atoi(e) : 16;
  return v < 2 ? 2 : v;
}
static int seg_wcap() {  // segments per config at most (TWB_SIM_SEG_WCAP: A/B only)
  const char* e = getenv("TWB_SIM_SEG_WCAP");
  const int v = e ? atoi(e) : 256;
  return v < 1 ? 1 : (v > 4096 ? 4096 : v);
}
constexpr int64_t kSegPerReqBytes =
    (int64_t)sizeof(int32_t) + (int64_t)sizeof(SegRegen) + 8 * (int64_t)sizeof(int64_t) +
    kSegLogPerReq * (int64_t)sizeof(TkLog);
static int64_t align256(int64_t x) { return (x + 255) & ~255LL; }
static int seg_sms() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}
static bool seg_enabled_for(int32_t n_cfg, int sms) {
  const char* e = getenv("TWB_SIM_SEG");
  if (e && e[0] == '0') return false;
  return n_cfg >= 1 && (int64_t)n_cfg <= (int64_t)kLatencyConfigsPerSm * sms;
}
static int seg_wmax(int32_t n_cfg, int sms) {
  const char* e = getenv("TWB_SIM_SEG_W");
  int64_t w = e ? atoll(e) : 0;
  if (w <= 0) w = ((int64_t)sms * 16 * 7 + n_cfg - 1) / n_cfg;  // ~7 segments per resident warp
  if (w > seg_wcap()) w = seg_wcap();
  if (w < 1) w = 1;
  return (int)w;
}
// Extra requests of room per segment: ~256 MB of overrun room in all, at most 4,096 and at
// most an eighth of the launch's requests (an overrun past the room re-runs serially from the
// segment's last regeneration point, so the bound trades memory for rare serial pieces)
static int64_t seg_xtra(int32_t n_cfg, int wmax, int64_t total_requests) {
  const int64_t per = kSegLogPerReq * (int64_t)sizeof(TkLog) + 64;
  int64_t x = (256LL << 20) / (per * (int64_t)n_cfg * wmax);
  x = x > 4096 ? 4096 : x;
  x = std::min(x, total_requests / 8);
  return x < 64 ? 64 : x;
}
static int64_t seg_header_bytes(int32_t n_cfg, int wmax) {  // counters, plan, summaries
  return align256(64 + align256(4LL * n_cfg) + align256(4LL * n_cfg * wmax) +
                  align256((int64_t)sizeof(SegSummary) * n_cfg * wmax));
}
// the scratch the segments need for R requests (tw_sim_seg_scratch_bytes)
static int64_t seg_bytes(int32_t n_cfg, int wmax, int64_t R) {
  return seg_header_bytes(n_cfg, wmax) + 4 * 256 + kSegPerReqBytes * R +
         seg_xtra(n_cfg, wmax, R) * n_cfg * wmax * (kSegLogPerReq * (int64_t)sizeof(TkLog) + 64);
}
// the largest request count whose segment records fit in `bytes` (seg_bytes is increasing)
static int64_t seg_r_max(int32_t n_cfg, int wmax, int64_t bytes) {
  int64_t lo = 0, hi = bytes / kSegPerReqBytes + 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) / 2;
    if (seg_bytes(n_cfg, wmax, mid) <= bytes) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// bytes of scratch tw_sim_many needs: the 64-byte work counter, plus the global slot state
// of every resident warp when the capacity exceeds what shared memory holds
static int64_t sim_scratch_bytes(int32_t n_cfg, int cap, int sms, int per_sm, int64_t* grid_out) {
  int64_t grid = (int64_t)sms * (per_sm < 1 ? 1 : per_sm);
  const int64_t want = ((int64_t)n_cfg + kSimWarps - 1) / kSimWarps;
  if (grid > want) grid = want;
  if (grid < 1) grid = 1;
  if (grid_out) *grid_out = grid;
  return 64 + grid * kSimWarps * 7 * (int64_t)sizeof(int32_t) * (int64_t)cap;
}

static thread_local int32_t g_last[4] = {0, 0, 0, 0};
static thread_local int32_t g_last_path = 0;  // tw_sim_last_path
static thread_local int64_t* g_prof = nullptr;
static thread_local int32_t* g_seg_stats = nullptr;

}  // namespace twb

using namespace twb;

extern "C" int tw_sim_many(const void* pset, int64_t pset_bytes, const tw_sim_cfg* cfgs, int32_t n_cfg,
                           const int32_t* order, const int64_t* wl_off, const int64_t* req_offset_ns,
                           const int32_t* req_prompt, const int32_t* req_output, tw_sim_result* results,
                           const int64_t* req_base, int64_t* req_first_ns, int64_t* req_finish_ns,
                           const int64_t* ev_off, tw_event* ev, int32_t slot_capacity, void* scratch,
                           int64_t scratch_bytes, void* stream) {
  if (!pset || pset_bytes < (int64_t)sizeof(tw_pset_header) || (pset_bytes & 15) ||
      ((uintptr_t)pset & 15)) {
    set_error("tw_sim_many: pset null, misaligned or not a multiple of 16 bytes");
    return TW_EINVAL;
  }
  if (n_cfg < 0 || (n_cfg > 0 && (!cfgs || !wl_off || !req_offset_ns || !req_prompt || !req_output ||
                                  !results || !scratch)) ||
      ((req_first_ns || req_finish_ns) && !req_base) || (ev && !ev_off)) {
    set_error("tw_sim_many: bad arguments");
    return TW_EINVAL;
  }
  if (n_cfg == 0) return TW_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (slot_capacity > (1 << 26)) {
    set_error("tw_sim_many: slot capacity %d beyond 2^26", slot_capacity);
    return TW_EINVAL;
  }
  int cap = slot_capacity < 32 ? 32 : slot_capacity;
  cap = (cap + 31) & ~31;
  int dev = 0, sms = 148, per_sm = 0, max_optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  SimParams p;
  p.gslots = nullptr;
  p.checks = g_checks;
  if (cap > kMaxSlotCap) {  // slot state in global memory (sim_big.cu), one slice per resident warp
    sim_big_prepare(kSimThreads, &per_sm);
    int64_t grid = 0;
    const int64_t need = sim_scratch_bytes(n_cfg, cap, sms, per_sm, &grid);
    if (scratch_bytes < need) {
      const int64_t fit = (scratch_bytes - 64) / ((int64_t)kSimWarps * 7 * (int64_t)sizeof(int32_t) * cap);
      if (fit < 1) {
        set_error("tw_sim_many: slot capacity %d needs %lld bytes of scratch (tw_sim_scratch_bytes), got %lld",
                  cap, (long long)need, (long long)scratch_bytes);
        return TW_ENOSMEM;
      }
      grid = fit;  // fewer resident warps: the work counter still hands out every config
    }
    cudaMemsetAsync(scratch, 0, sizeof(int32_t), s);
    p.pset = pset;
    p.pset_bytes = (uint32_t)pset_bytes;
    p.pset_smem = 0;
    p.cfgs = cfgs;
    p.n_cfg = n_cfg;
    p.order = order;
    p.wl_off = wl_off;
    p.ts = req_offset_ns;
    p.prompt = req_prompt;
    p.output = req_output;
    p.res = results;
    p.req_base = req_base;
    p.first = req_first_ns;
    p.finish = req_finish_ns;
    p.ev_off = ev_off;
    p.ev = ev;
    p.counter = reinterpret_cast<int32_t*>(scratch);
    p.cap = cap;
    p.prof = g_prof;
    p.gslots = reinterpret_cast<int32_t*>(static_cast<char*>(scratch) + 64);
    sim_big_launch((int)grid, kSimThreads, s, p);
    count_launch();
    g_last[0] = (int32_t)grid;
    g_last[1] = kSimThreads;
    g_last[2] = 128;
    g_last[3] = cap;
    g_last_path = 3;
    return check_launch("tw_sim_many");
  }
  // slot state is 7 int32 arrays of cap per warp: large capacities get fewer warps per CTA
  const size_t per_warp = 7 * sizeof(int32_t) * (size_t)cap;
  // latency regime: busy-period segments when the caller gave per-request bases and the
  // scratch for the segment records (tw_sim_seg_scratch_bytes); not with event dumps,
  // profiling or the invariant build, which run the serial loop
  if (req_base && !ev && !g_checks && !g_prof && seg_enabled_for(n_cfg, sms) &&
      128 + 4 * per_warp <= (size_t)max_optin) {
    const int wmax = seg_wmax(n_cfg, sms);
    const int64_t r_max = seg_r_max(n_cfg, wmax, scratch_bytes);
    // the join adds each warp's segment starts and their arrival times (12 B per segment)
    const size_t join_smem = 128 + 4 * per_warp + (size_t)kSimWarps * 16 * wmax;
    if (r_max >= 1 && join_smem <= (size_t)max_optin) {
      char* b = static_cast<char*>(scratch);
      SegParams q;
      q.wmax = wmax;
      q.min_req = seg_min_req();
      q.counter = reinterpret_cast<int32_t*>(b);
      int64_t o = 64;
      q.nseg = reinterpret_cast<int32_t*>(b + o);
      o += align256(4LL * n_cfg);
      q.seg_a0 = reinterpret_cast<int32_t*>(b + o);
      o += align256(4LL * n_cfg * wmax);
      q.summ = reinterpret_cast<SegSummary*>(b + o);
      o = seg_header_bytes(n_cfg, wmax);
      q.regpos = reinterpret_cast<int32_t*>(b + o);
      o += align256(4 * r_max);
      q.reg = reinterpret_cast<SegRegen*>(b + o);
      o += align256((int64_t)sizeof(SegRegen) * r_max);
      q.xtra = seg_xtra(n_cfg, wmax, r_max);
      const int64_t units = r_max + q.xtra * n_cfg * wmax;
      q.log = reinterpret_cast<TkLog*>(b + o);
      o += align256((int64_t)sizeof(TkLog) * kSegLogPerReq * units);
      q.side = reinterpret_cast<int64_t*>(b + o);
      q.r_max = r_max;
      const char* cd = getenv("TWB_SIM_SEG_CAPDIV");  // tests only: force the overflow path
      q.cap_div = cd && atoi(cd) > 1 ? atoi(cd) : 1;
      q.stats = g_seg_stats;
      static thread_local int32_t seg_epoch = 0;
      q.epoch = ++seg_epoch;
      const int threads = kSimThreads;
      // A/B only: TWB_SIM_SEG_LAT=1 stages the blob in shared memory (the latency variant's
      // geometry), TWB_SIM_SEG_STAGE=<bytes> stages only that prefix (e.g. the core)
      const char* lat_env = getenv("TWB_SIM_SEG_LAT");
      const int lat = lat_env ? atoi(lat_env) : 0;
      const size_t seg_smem = 128 + 4 * per_warp;
      size_t smem = seg_smem;
      sim_seg_prepare(threads, seg_smem, &per_sm, false);
      uint32_t seg_pset_bytes = (uint32_t)pset_bytes, seg_pset_smem = 0;
      if (lat >= 1) {
        const char* st_env = getenv("TWB_SIM_SEG_STAGE");
        seg_pset_bytes = st_env ? (uint32_t)atoll(st_env) : (uint32_t)pset_bytes;
        if (seg_pset_bytes < 64 || seg_pset_bytes > (uint32_t)pset_bytes) seg_pset_bytes = (uint32_t)pset_bytes;
        seg_pset_smem = (seg_pset_bytes + 127) & ~127u;
        smem = 128 + seg_pset_smem + 4 * per_warp;
        if (smem <= (size_t)max_optin) sim_seg_prepare(threads, smem, &per_sm, true);
        else {
          smem = seg_smem;
          seg_pset_smem = 0;
          seg_pset_bytes = (uint32_t)pset_bytes;
        }
      }
      if (per_sm < 1) per_sm = 1;
      cudaMemsetAsync(scratch, 0, 64, s);
      cudaMemsetAsync(q.regpos, 0xff, 4 * r_max, s);
      p.pset = pset;
      p.pset_bytes = seg_pset_bytes;
      p.pset_smem = seg_pset_smem;
      p.cfgs = cfgs;
      p.n_cfg = n_cfg;
      p.order = order;
      p.wl_off = wl_off;
      p.ts = req_offset_ns;
      p.prompt = req_prompt;
      p.output = req_output;
      p.res = results;
      p.req_base = req_base;
      p.first = req_first_ns;
      p.finish = req_finish_ns;
      p.ev_off = nullptr;
      p.ev = nullptr;
      p.counter = q.counter;
      p.cap = cap;
      p.prof = nullptr;
      const int grid = sms * per_sm;
      const int join_grid = (int)std::min<int64_t>(((int64_t)n_cfg + kSimWarps - 1) / kSimWarps, (int64_t)sms * 4);
      sim_seg_launch(grid, threads, smem, s, p, q, join_grid, lat >= 1 && seg_pset_smem > 0, join_smem,
                     (uint32_t)pset_bytes);
      for (int k = 0; k < 4; k++) count_launch();  // plan, segments, Timekeeper replays, join
      g_last[0] = grid;
      g_last[1] = threads;
      g_last[2] = (int32_t)smem;
      g_last[3] = cap;
      g_last_path = 2;
      return check_launch("tw_sim_many");
    }
  }
  // more configs than 8 per SM, or a blob too large to stage next to one warp's slot
  // state: the throughput variant (blob read from global memory)
  const uint32_t blob_smem = (uint32_t)((pset_bytes + 127) & ~127LL);
  const bool tput = (int64_t)n_cfg > (int64_t)kLatencyConfigsPerSm * sms ||
                    128 + (size_t)blob_smem + per_warp > (size_t)max_optin || g_checks != nullptr;
  const uint32_t pset_smem = tput ? 0u : blob_smem;
  int warps = kSimWarps;
  while (warps > 1 && 128 + pset_smem + warps * per_warp > (size_t)max_optin) warps--;
  const int threads = 32 * warps;
  const size_t smem = 128 + pset_smem + warps * per_warp;
  if ((int)smem > max_optin) {
    set_error("tw_sim_many: %zu B of shared memory needed (slot capacity %d), device allows %d", smem, cap,
              max_optin);
    return TW_ENOSMEM;
  }
  if (g_checks) {
    sim_check_prepare(threads, smem, &per_sm);
  } else if (tput) {
    sim_tput_prepare(threads, smem, &per_sm);
  } else {
    cudaFuncSetAttribute(k_sim<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sim<false>, threads, smem);
  }
  if (per_sm < 1) per_sm = 1;
  int64_t want = ((int64_t)n_cfg + warps - 1) / warps;
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > want) grid = want;
  cudaMemsetAsync(scratch, 0, sizeof(int32_t), s);
  p.pset = pset;
  p.pset_bytes = (uint32_t)pset_bytes;
  p.pset_smem = pset_smem;
  p.cfgs = cfgs;
  p.n_cfg = n_cfg;
  p.order = order;
  p.wl_off = wl_off;
  p.ts = req_offset_ns;
  p.prompt = req_prompt;
  p.output = req_output;
  p.res = results;
  p.req_base = req_base;
  p.first = req_first_ns;
  p.finish = req_finish_ns;
  p.ev_off = ev_off;
  p.ev = ev;
  p.counter = reinterpret_cast<int32_t*>(scratch);
  p.cap = cap;
  p.prof = g_prof;
  if (g_checks) sim_check_launch((int)grid, threads, smem, s, p);
  else if (tput) sim_tput_launch((int)grid, threads, smem, s, p);
  else k_sim<false><<<(int)grid, threads, smem, s>>>(p);
  count_launch();
  g_last[0] = (int32_t)grid;
  g_last[1] = threads;
  g_last[2] = (int32_t)smem;
  g_last[3] = cap;
  g_last_path = tput ? 1 : 0;
  return check_launch("tw_sim_many");
}

extern "C" int64_t tw_sim_scratch_bytes(int32_t n_cfg, int32_t slot_capacity) {
  int cap = slot_capacity < 32 ? 32 : slot_capacity;
  cap = (cap + 31) & ~31;
  if (cap <= kMaxSlotCap || n_cfg <= 0) return 64;
  int dev = 0, sms = 148, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  sim_big_prepare(kSimThreads, &per_sm);
  return sim_scratch_bytes(n_cfg, cap, sms, per_sm, nullptr);
}

extern "C" int64_t tw_sim_seg_scratch_bytes(int32_t n_cfg, int64_t total_requests) {
  const int sms = seg_sms();
  if (!seg_enabled_for(n_cfg, sms) || total_requests < 0) return 0;
  const int wmax = seg_wmax(n_cfg, sms);
  return seg_bytes(n_cfg, wmax, total_requests > 0 ? total_requests : 1);
}

extern "C" int tw_sim_set_checks(int32_t* per_config_8xi32) {
  g_checks = per_config_8xi32;
  return TW_OK;
}

extern "C" int tw_sim_set_seg_stats(int32_t* per_config_8xi32) {
  g_seg_stats = per_config_8xi32;
  return TW_OK;
}

extern "C" int tw_sim_set_profile(int64_t* per_config_16xi64) {
  g_prof = per_config_16xi64;
  return TW_OK;
}

extern "C" int tw_sim_last_path(void) { return g_last_path; }

extern "C" int tw_sim_last_launch(int32_t* grid, int32_t* block, int32_t* smem_bytes, int32_t* slot_capacity) {
  if (grid) *grid = g_last[0];
  if (block) *block = g_last[1];
  if (smem_bytes) *smem_bytes = g_last[2];
  if (slot_capacity) *slot_capacity = g_last[3];
  return TW_OK;
}
#endif  // TWB_SIM_TPUT_TU
