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
//  * virtual time advances through the Timekeeper min-advance: lane a holds actor a
//    (dispatcher + TP x PP workers) and each round is one int64 REDUX min;
//  * every token event is hashed into a position-bound digest (tw_event_hash) and
//    FIRST_TOKEN / FINISHED stamps are stored per request; full event dumps only
//    for audited configs.
#include "common.cuh"

namespace twb {

constexpr int kSimThreads = 128;  // 4 warps per CTA
constexpr int kSimWarps = kSimThreads / 32;
constexpr int kMaxSlotCap = 4096;

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
};

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// int64 warp min with two REDUX ops (hi signed, then lo unsigned among hi-minimal lanes)
__device__ __forceinline__ int64_t warp_min_i64_redux(int64_t v) {
  const int hi = (int)(v >> 32);
  const int mh = __reduce_min_sync(kFull, hi);
  const unsigned lo = (hi == mh) ? (unsigned)(uint64_t)v : 0xffffffffu;
  const unsigned ml = __reduce_min_sync(kFull, lo);
  return (int64_t)(((uint64_t)(uint32_t)mh << 32) | ml);
}
// int64 warp sum of non-negative values < 2^50 per lane, with two REDUX ops
__device__ __forceinline__ int64_t warp_sum_i64_redux(int64_t v) {
  const unsigned lo = (unsigned)(v & 0xffffff);
  const unsigned hi = (unsigned)(v >> 24);
  const unsigned sl = __reduce_add_sync(kFull, lo);
  const unsigned sh = __reduce_add_sync(kFull, hi);
  return ((int64_t)sh << 24) + (int64_t)sl;
}
// inclusive int64 scan across the warp
__device__ __forceinline__ int64_t warp_incl_scan_i64(int64_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t w = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += w;
  }
  return v;
}

__device__ __forceinline__ int64_t blocks_of(int64_t tokens, int64_t bk) {
  return tokens > 0 ? (tokens + bk - 1) / bk : 0;  // oracle.py:39-40
}

struct Slots {
  int32_t* req;
  int32_t* prompt;
  int32_t* output;
  int32_t* done;
  int32_t* emit;
  int32_t* plan;  // >= 0 chunk tokens, -1 decode, -2 idle (this step)
};

// Per-config Timekeeper actor grid: actor 0 is the
// dispatcher, actors 1..TP*S the workers; BarrierCore semantics on a FakeClock.
struct TkGrid {
  int64_t wall, offset, seq, last_bcast, V, cooldown, conv_cooldown;
  int64_t disp, disp_ts;
};

__device__ __forceinline__ void tk_resolve(TkGrid& g, int64_t t_min) {
  // timekeeper.py:326-366 with FakeClock sleep
  if (g.wall < t_min && g.last_bcast != INT64_MIN && g.cooldown > 0) {
    const int64_t wait = g.last_bcast + g.cooldown - g.wall;
    if (wait > 0) g.wall += (wait == g.cooldown) ? g.conv_cooldown : fake_sleep_ns(wait);
  }
  if (g.wall < t_min) {
    const int64_t cand = t_min - g.wall;
    if (cand > g.offset) g.offset = cand;
    g.seq++;
    g.last_bcast = g.wall;
  }
  g.V = g.wall + g.offset;
}

// Advance until V >= end. stages == 0: idle jump, only the dispatcher drives time.
__device__ __forceinline__ void tk_advance(TkGrid& g, const int64_t* __restrict__ ts, int64_t n,
                                           int64_t epoch, int S, int TP, int stages_on, int64_t base,
                                           int64_t d, int64_t end) {
  const int lane = threadIdx.x & 31;
  const int64_t per = d / S;
  for (;;) {
    while (g.disp < n && g.disp_ts <= g.V) {  // dispatcher passes every arrival <= V
      g.disp++;
      g.disp_ts = g.disp < n ? epoch + __ldg(ts + g.disp) : INT64_MAX;
    }
    if (g.V >= end) return;
    int cs = S;
    if (stages_on) {
      for (int s = 0; s < S; s++) {
        const int64_t e = (s == S - 1) ? base + d : base + per * (s + 1);
        if (e > g.V) { cs = s; break; }
      }
    }
    int64_t tgt = INT64_MAX;
    if (lane == 0) {
      tgt = g.disp_ts;
    } else if (stages_on && lane <= TP * S) {
      const int s = (lane - 1) / TP;
      if (s == cs) tgt = (s == S - 1) ? base + d : base + per * (s + 1);
    }
    tk_resolve(g, warp_min_i64_redux(tgt));
  }
}

__device__ void run_config(const SimParams& p, const char* ps, Slots sl, int c) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
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
  } else if (cfg.max_running > p.cap || (tk_on && 1 + TP * S > 32)) {
    r.status = TW_SIM_CAPACITY;
  }
  if (r.status != TW_SIM_OK) {
    if (lane == 0) p.res[c] = r;
    return;
  }

  const int64_t wl0 = p.wl_off[cfg.workload_id];
  const int64_t n = p.wl_off[cfg.workload_id + 1] - wl0;
  const int64_t* __restrict__ ts = p.ts + wl0;
  const int32_t* __restrict__ prm = p.prompt + wl0;
  const int32_t* __restrict__ outp = p.output + wl0;
  const int64_t epoch = cfg.epoch_ns;
  const int64_t bk = cfg.kv_block_tokens;
  const int64_t chunk = cfg.chunk_size;
  const int64_t mbt = cfg.max_batch_tokens;
  const int64_t max_running = cfg.max_running;
  int64_t* first = p.first ? p.first + p.req_base[c] : nullptr;
  int64_t* finish = p.finish ? p.finish + p.req_base[c] : nullptr;
  tw_event* evp = nullptr;
  int64_t ev_cap = 0;
  if (p.ev && p.ev_off[c + 1] > p.ev_off[c]) {  // audited config: full event dump
    evp = p.ev + p.ev_off[c];
    ev_cap = p.ev_off[c + 1] - p.ev_off[c];
  }

  TkGrid g;
  g.wall = epoch;
  g.offset = 0;
  g.seq = 0;
  g.last_bcast = INT64_MIN;
  g.V = epoch;
  g.cooldown = cfg.tk_cooldown_ns;
  g.conv_cooldown = g.cooldown > 0 ? fake_sleep_ns(g.cooldown) : 0;
  g.disp = 0;
  g.disp_ts = n > 0 ? epoch + __ldg(ts) : INT64_MAX;

  int64_t now = epoch, step = 0, n_events = 0, held_sum = 0;
  int64_t fut = 0, w_head = 0;  // waiting = [w_head, fut), future = [fut, n)
  int n_act = 0;
  uint64_t dig = 0;  // lane-partial digest
  // arrival-offset cache: lane l holds ts[cbase + l]
  int64_t cbase = 0;
  int64_t cts = (lane < n) ? __ldg(ts + lane) : INT64_MAX;
  int overflow = 0;

  while (fut < n || w_head < fut || n_act > 0) {
    // ---- arrivals with epoch + offset <= now join the waiting queue (oracle.py:73-75)
    for (;;) {
      if (fut >= n) break;
      if (fut - cbase >= 32) {
        cbase = fut;
        cts = (cbase + lane < n) ? __ldg(ts + cbase + lane) : INT64_MAX;
      }
      const int sh = (int)(fut - cbase);
      const bool le = (lane >= sh) && (cbase + lane < n) && (epoch + cts <= now);
      const unsigned m = __ballot_sync(kFull, le) >> sh;    // bit 0 = arrival `fut`
      const int width = 32 - sh;
      const int k = (~m == 0u) ? width : min(__ffs(~m) - 1, width);
      fut += k;
      if (k < width) break;
    }

    // ---- _plan (oracle.py:117-180), pass 1a: counts
    const int64_t free0 = (int64_t)cfg.kv_capacity_blocks - held_sum;
    int total_dec = 0;
    bool any_mid = false;
    for (int b = 0; b < n_act; b += 32) {
      const int i = b + lane;
      const bool v = i < n_act;
      const int32_t pr = v ? sl.prompt[i] : 0, dn = v ? sl.done[i] : 0;
      const int32_t em = v ? sl.emit[i] : 0, op = v ? sl.output[i] : 0;
      const bool mid = v && dn < pr;
      total_dec += __popc(__ballot_sync(kFull, v && !mid && em < op));
      any_mid |= __any_sync(kFull, mid);
    }
    bool do_dec = true, do_chunks = true;
    if (cfg.policy == TW_POLICY_PREFILL_PRIORITIZED) {
      bool have_prefill = any_mid;
      if (!have_prefill && w_head < fut) {
        const int64_t hp = __ldg(prm + w_head);
        have_prefill = (int64_t)n_act < max_running && blocks_of(hp, bk) <= free0;
      }
      do_chunks = have_prefill;
      do_dec = !have_prefill;
    }
    const int64_t n_dec = do_dec ? min((int64_t)total_dec, mbt) : 0;
    int64_t budget = mbt - n_dec;

    // ---- pass 1b: decode cutoff, chunk takes, features
    int64_t p_l = 0, c_l = 0;  // lane partial P and C
    int n_chunk = 0, chunk_ev = 0;
    int dec_before = 0;
    int64_t want_before = 0;
    for (int b = 0; b < n_act; b += 32) {
      const int i = b + lane;
      const bool v = i < n_act;
      const int32_t pr = v ? sl.prompt[i] : 0, dn = v ? sl.done[i] : 0;
      const int32_t em = v ? sl.emit[i] : 0, op = v ? sl.output[i] : 0;
      const bool mid = v && dn < pr;
      const bool dcand = v && !mid && em < op;
      const unsigned dm = __ballot_sync(kFull, dcand);
      const int rank = dec_before + __popc(dm & lt);
      const bool is_dec = do_dec && dcand && rank < mbt;
      dec_before += __popc(dm);
      int32_t plan = is_dec ? -1 : -2;
      if (is_dec) c_l += (int64_t)pr + em;  // DecodeSlot.context_len = prompt + emitted
      if (do_chunks && __any_sync(kFull, mid)) {
        const int64_t want = mid ? min(chunk, (int64_t)(pr - dn)) : 0;
        const int64_t incl = warp_incl_scan_i64(want);
        const int64_t E = want_before + incl - want;  // tokens taken by earlier chunks
        const bool chosen = mid && budget - E > 0;
        if (chosen) {
          const int64_t take = min(want, budget - E);
          plan = (int32_t)take;
          p_l += take;
          c_l += dn;  // PrefillChunk.context_len_before = done_prefill
          if (dn + take >= pr) chunk_ev += (op <= 1) ? 2 : 1;
        }
        n_chunk += __popc(__ballot_sync(kFull, chosen));
        want_before += __shfl_sync(kFull, incl, 31);
      }
      if (v) sl.plan[i] = plan;
    }
    // tokens the chunks consumed: every chosen chunk took `want` except possibly the last
    {
      const int64_t took = min(want_before, budget > 0 ? budget : 0);
      budget -= took;
    }

    // ---- admission from the waiting head: strict FCFS, KV + slot + budget gates
    int n_adm = 0;
    if (do_chunks && budget > 0 && w_head < fut) {
      int64_t free_l = free0, slots = max_running - n_act;
      while (budget > 0 && slots > 0 && w_head + n_adm < fut) {
        const int64_t idx = w_head + n_adm + lane;
        const bool cand = idx < fut && lane < slots;
        const int64_t pr = cand ? __ldg(prm + idx) : 0;
        const int64_t need = blocks_of(pr, bk);
        const int64_t want = min(chunk, pr);
        const int64_t NEi = warp_incl_scan_i64(cand ? need : 0);
        const int64_t WEi = warp_incl_scan_i64(cand ? want : 0);
        const int64_t NE = NEi - need, WE = WEi - want;
        const bool ok = cand && (budget - WE > 0) && (need <= free_l - NE);
        const unsigned bad = __ballot_sync(kFull, !ok);
        const int k = bad ? __ffs(bad) - 1 : 32;
        if (lane < k) {
          const int slot = n_act + n_adm + lane;
          const int64_t take = min(want, budget - WE);
          sl.req[slot] = (int32_t)idx;
          sl.prompt[slot] = (int32_t)pr;
          const int32_t op = __ldg(outp + idx);
          sl.output[slot] = op;
          sl.done[slot] = 0;
          sl.emit[slot] = 0;
          sl.plan[slot] = (int32_t)take;
          p_l += take;
          if (take >= pr) chunk_ev += (op <= 1) ? 2 : 1;
        }
        if (k == 0) break;
        const int64_t tot_need = __shfl_sync(kFull, NEi, k - 1);
        const int64_t tot_want = __shfl_sync(kFull, WEi, k - 1);
        const int64_t last_want = __shfl_sync(kFull, want, k - 1);
        const int64_t last_we = tot_want - last_want;
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
      if (n_act > 0 || w_head < fut) {  // oracle.py:78-80 -> _diagnose_stall
        r.status = n_act > 0 ? TW_SIM_STALLED_ACTIVE : TW_SIM_STALLED_KV;
        break;
      }
      // idle until the next arrival (oracle.py:81-83)
      const int sh = (int)(fut - cbase);
      const int64_t t_next = (sh < 32) ? __shfl_sync(kFull, cts, sh) : __ldg(ts + fut);
      now = epoch + t_next;
      if (tk_on) tk_advance(g, ts, n, epoch, S, TP, 0, now, 0, now);
      continue;
    }

    // ---- predict (oracle.py:85-86)
    const int64_t P = (int64_t)__reduce_add_sync(kFull, (unsigned)p_l);  // P <= max_batch_tokens
    const int64_t C = warp_sum_i64_redux(c_l);
    const int64_t d = predict_warp(ps, cfg.pred_id, P, n_dec, C);
    if (d < 0) {
      r.status = TW_SIM_PRED_ERROR;
      r.pred_code = (int32_t)d;
      break;
    }
    step += 1;
    const int64_t base = now;
    now += d;
    if (tk_on) tk_advance(g, ts, n, epoch, S, TP, 1, base, d, now);  // WorkerGrid stage deadlines

    // ---- apply (oracle.py:88-112): chunks' events first, then decodes', in slot order
    const int n_tot = n_act + n_adm;
    const int chunk_ev_total = __reduce_add_sync(kFull, (unsigned)chunk_ev);
    int64_t pos_c = n_events, pos_d = n_events + chunk_ev_total;
    int kept = 0;
    int64_t held_l = 0;
    for (int b = 0; b < n_tot; b += 32) {
      const int i = b + lane;
      const bool v = i < n_tot;
      int32_t rq = 0, pr = 0, op = 0, dn = 0, em = 0, plan = -2;
      if (v) {
        rq = sl.req[i];
        pr = sl.prompt[i];
        op = sl.output[i];
        dn = sl.done[i];
        em = sl.emit[i];
        plan = sl.plan[i];
      }
      int nev = 0, k0 = 0, k1 = 0;
      bool fin = false;
      const bool is_chunk = plan >= 0, is_dec = plan == -1;
      if (is_chunk) {
        dn += plan;
        if (dn >= pr) {
          em = 1;
          nev = 1;
          k0 = TW_EV_FIRST_TOKEN;
          if (em >= op) { nev = 2; k1 = TW_EV_FINISHED; fin = true; }
        }
      } else if (is_dec) {
        em += 1;
        nev = 1;
        k0 = TW_EV_OUTPUT_TOKEN;
        if (em >= op) { nev = 2; k1 = TW_EV_FINISHED; fin = true; }
      }
      const unsigned c1 = __ballot_sync(kFull, is_chunk && nev >= 1);
      const unsigned c2 = __ballot_sync(kFull, is_chunk && nev == 2);
      const unsigned d1 = __ballot_sync(kFull, is_dec && nev >= 1);
      const unsigned d2 = __ballot_sync(kFull, is_dec && nev == 2);
      if (nev) {
        const int64_t pos = is_chunk ? pos_c + __popc(c1 & lt) + __popc(c2 & lt)
                                     : pos_d + __popc(d1 & lt) + __popc(d2 & lt);
        dig += tw_event_hash((uint64_t)pos, (uint64_t)rq, (uint64_t)k0, now, step);
        if (k0 == TW_EV_FIRST_TOKEN && first) first[rq] = now;
        if (evp && pos < ev_cap) {
          tw_event e;
          e.ts_ns = now;
          e.step = (int32_t)step;
          e.req_kind = (rq << 2) | k0;
          evp[pos] = e;
        }
        if (nev == 2) {
          dig += tw_event_hash((uint64_t)(pos + 1), (uint64_t)rq, (uint64_t)k1, now, step);
          if (finish) finish[rq] = now;
          if (evp && pos + 1 < ev_cap) {
            tw_event e;
            e.ts_ns = now;
            e.step = (int32_t)step;
            e.req_kind = (rq << 2) | k1;
            evp[pos + 1] = e;
          }
        }
      }
      pos_c += __popc(c1) + __popc(c2);
      pos_d += __popc(d1) + __popc(d2);
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
        sl.emit[np] = em;
        const int64_t h0 = blocks_of(pr, bk), h1 = blocks_of((int64_t)dn + em, bk);
        held_l += h0 > h1 ? h0 : h1;  // _held (oracle.py:43-46)
      }
      kept += __popc(km);
      __syncwarp();
    }
    n_events = pos_d;
    if (evp && n_events > ev_cap) overflow = 1;
    held_sum = warp_sum_i64_redux(held_l);
    w_head += n_adm;
    n_act = kept;
  }

  // digest: sum of lane partials mod 2^64
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dig += __shfl_xor_sync(kFull, dig, o);
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
  if (lane == 0) p.res[c] = r;
}

__global__ void __launch_bounds__(kSimThreads) k_sim(SimParams p) {
  extern __shared__ __align__(128) char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  char* ps = smem + 128;
  tma_stage_to_smem(ps, p.pset, p.pset_bytes, bar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t* base = reinterpret_cast<int32_t*>(smem + 128 + p.pset_smem) + (size_t)warp * 6 * p.cap;
  Slots sl;
  sl.req = base;
  sl.prompt = base + p.cap;
  sl.output = base + 2 * p.cap;
  sl.done = base + 3 * p.cap;
  sl.emit = base + 4 * p.cap;
  sl.plan = base + 5 * p.cap;
  for (;;) {
    int idx = 0;
    if (lane == 0) idx = atomicAdd(p.counter, 1);
    idx = __shfl_sync(kFull, idx, 0);
    if (idx >= p.n_cfg) break;
    const int c = p.order ? p.order[idx] : idx;
    run_config(p, ps, sl, c);
    __syncwarp();
  }
}

static thread_local int32_t g_last[4] = {0, 0, 0, 0};

}  // namespace twb

using namespace twb;

extern "C" int tw_sim_many(const void* pset, int64_t pset_bytes, const tw_sim_cfg* cfgs, int32_t n_cfg,
                           const int32_t* order, const int64_t* wl_off, const int64_t* req_offset_ns,
                           const int32_t* req_prompt, const int32_t* req_output, tw_sim_result* results,
                           const int64_t* req_base, int64_t* req_first_ns, int64_t* req_finish_ns,
                           const int64_t* ev_off, tw_event* ev, int32_t slot_capacity, void* scratch,
                           void* stream) {
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
  int cap = slot_capacity < 32 ? 32 : slot_capacity;
  cap = (cap + 31) & ~31;
  if (cap > kMaxSlotCap) {
    set_error("tw_sim_many: slot capacity %d exceeds the engine limit %d", slot_capacity, kMaxSlotCap);
    return TW_ENOSMEM;
  }
  const uint32_t pset_smem = (uint32_t)((pset_bytes + 127) & ~127LL);
  const size_t smem = 128 + pset_smem + (size_t)kSimWarps * 6 * sizeof(int32_t) * cap;
  int dev = 0, sms = 148, per_sm = 0, max_optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if ((int)smem > max_optin) {
    set_error("tw_sim_many: %zu B of shared memory needed (slot capacity %d), device allows %d", smem, cap,
              max_optin);
    return TW_ENOSMEM;
  }
  cudaFuncSetAttribute(k_sim, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sim, kSimThreads, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t want = ((int64_t)n_cfg + kSimWarps - 1) / kSimWarps;
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > want) grid = want;
  cudaMemsetAsync(scratch, 0, sizeof(int32_t), s);
  SimParams p;
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
  k_sim<<<(int)grid, kSimThreads, smem, s>>>(p);
  count_launch();
  g_last[0] = (int32_t)grid;
  g_last[1] = kSimThreads;
  g_last[2] = (int32_t)smem;
  g_last[3] = cap;
  return check_launch("tw_sim_many");
}

extern "C" int tw_sim_last_launch(int32_t* grid, int32_t* block, int32_t* smem_bytes, int32_t* slot_capacity) {
  if (grid) *grid = g_last[0];
  if (block) *block = g_last[1];
  if (smem_bytes) *smem_bytes = g_last[2];
  if (slot_capacity) *slot_capacity = g_last[3];
  return TW_OK;
}
