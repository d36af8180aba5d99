// timekeeper.cu — the Timekeeper's causal min-advance (north-star kernel 3).
//
// Reference: BarrierCore (pkg/src/timewarp/timekeeper.py:68-366) driven by a
// FakeClock (pkg/tests/_support.py:25-38).
//
//   tw_tk_replay  : one warp per Timekeeper; lane a holds client a (pending target,
//                   role, active, exempt) and lane g holds collective group g, so
//                   eligible_count / |pending| are one ballot+popc each and t_min is
//                   one int64 warp min — the per-config segmented reduction.
//   tw_tk_resolve : one round of _try_resolve/_resolve for C Timekeepers x A actor
//                   slots; A is padded to a power of two and 32/A Timekeepers share
//                   a warp, reduced with shuffles inside their lane segment.
#include <cmath>

#include "common.cuh"

namespace twb {

constexpr int kTkThreads = 128;

struct TkWarp {
  // uniform
  int64_t wall, offset, seq, last_bcast, cooldown, rounds, broadcasts, n_ev, ev_cap;
  int sealed, nclients, limit;
  bool suppress;
  tw_tk_event* ev;
  // per lane: client `lane`
  int64_t target;
  bool pending, active, observer, exempt;
  // per lane: group `lane`
  int64_t g_gen, g_expected;
  uint32_t g_arrived;
};

__device__ __forceinline__ void tk_emit(TkWarp& k, int kind, int64_t a, int64_t b, int op_index) {
  if ((threadIdx.x & 31) == 0 && k.n_ev < k.ev_cap) {
    tw_tk_event e;
    e.offset_ns = a;
    e.seq = b;
    e.wall_ns = k.wall;
    e.kind = kind;
    e.op_index = op_index;
    k.ev[k.n_ev] = e;
  }
  k.n_ev++;
}

__device__ __forceinline__ void tk_try_resolve(TkWarp& k, int op_index) {
  if (!k.sealed) return;  // timekeeper.py:318-324
  const int lane = threadIdx.x & 31;
  const bool is_client = lane < k.nclients;
  const int elig = __popc(__ballot_sync(kFull, is_client && k.active && !k.observer && !k.exempt));
  const int npend = __popc(__ballot_sync(kFull, is_client && k.pending));
  if (elig <= 0 || npend != elig) return;
  // _resolve: timekeeper.py:326-366
  const int64_t t_min = warp_min_i64(k.pending ? k.target : INT64_MAX);
  if (k.wall < t_min && k.last_bcast != INT64_MIN && k.cooldown > 0) {
    const int64_t wait = k.last_bcast + k.cooldown - k.wall;
    if (wait > 0) k.wall += fake_sleep_ns(wait);
  }
  k.rounds++;
  if (k.wall < t_min) {
    const int64_t cand = t_min - k.wall;
    if (cand > k.offset) k.offset = cand;
    k.seq++;
    k.broadcasts++;
    tk_emit(k, 0, k.offset, k.seq, op_index);
    k.last_bcast = k.wall;
  }
  k.pending = false;
}

__global__ void __launch_bounds__(kTkThreads) k_tk_replay(
    const tw_tk_op* __restrict__ ops, const int64_t* __restrict__ op_off, int32_t n_streams,
    const int64_t* __restrict__ wall0, const int64_t* __restrict__ cooldown,
    const uint8_t* __restrict__ suppress, int32_t* __restrict__ ack, tw_tk_event* __restrict__ ev,
    const int64_t* __restrict__ ev_off, tw_tk_final* __restrict__ fin) {
  const int lane = threadIdx.x & 31;
  const int s = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (s >= n_streams) return;  // warp-uniform
  TkWarp k;
  k.wall = wall0[s];
  k.offset = 0;
  k.seq = 0;
  k.last_bcast = INT64_MIN;
  k.cooldown = cooldown[s];
  k.rounds = k.broadcasts = k.n_ev = 0;
  k.ev = ev ? ev + ev_off[s] : nullptr;
  k.ev_cap = ev ? ev_off[s + 1] - ev_off[s] : 0;
  k.sealed = 0;
  k.nclients = 0;
  k.limit = 0;
  k.suppress = suppress ? suppress[s] != 0 : false;
  k.target = 0;
  k.pending = k.active = k.observer = k.exempt = false;
  k.g_gen = 0;
  k.g_expected = 0;
  k.g_arrived = 0;

  const int64_t o0 = op_off[s], o1 = op_off[s + 1];
  for (int64_t i = o0; i < o1; i++) {
    const tw_tk_op op = ops[i];  // same address in every lane: one broadcast load
    const int op_index = (int)(i - o0);
    const int c = op.client;
    int a = TW_ACK_OK;
    // _require_client (timekeeper.py:121-127), for ops that name a client
    const bool cvalid = c >= 0 && c < k.nclients;
    const bool c_active = __shfl_sync(kFull, k.active, cvalid ? c : 0) && cvalid;
    const bool c_observer = __shfl_sync(kFull, k.observer, cvalid ? c : 0);
    switch (op.type) {
      case TW_OP_REGISTER_ACTOR:
      case TW_OP_REGISTER_OBSERVER:  // timekeeper.py:155-182
        if (k.sealed) { a = TW_ACK_REGISTRATION_SEALED; break; }
        if (k.nclients >= TW_TK_MAX_CLIENTS) { a = TW_ACK_TOO_MANY; k.limit = 1; break; }
        if (lane == k.nclients) {
          k.active = true;
          k.observer = op.type == TW_OP_REGISTER_OBSERVER;
          k.pending = false;
          k.exempt = false;
        }
        k.nclients++;
        break;
      case TW_OP_SEAL: {  // timekeeper.py:184-200
        if (!k.sealed) {
          const bool any = __any_sync(kFull, lane < k.nclients && k.active && !k.observer);
          if (!any) { a = TW_ACK_NO_ACTORS; break; }
          k.sealed = 1;
        }
        tk_try_resolve(k, op_index);
        break;
      }
      case TW_OP_JUMP:  // timekeeper.py:202-225
        if (!cvalid) { a = TW_ACK_UNKNOWN_CLIENT; break; }
        if (!c_active) { a = TW_ACK_INVALID_STATE; break; }
        if (c_observer) { a = TW_ACK_ROLE_VIOLATION; break; }
        if (op.arg <= 0) { a = TW_ACK_INVALID_DELTA; break; }
        if (lane == c) {
          k.target = op.arg;  // a re-request overwrites
          k.pending = true;
          k.exempt = false;
        }
        tk_try_resolve(k, op_index);
        break;
      case TW_OP_ENTER: {  // timekeeper.py:227-292
        if (!cvalid) { a = TW_ACK_UNKNOWN_CLIENT; break; }
        if (!c_active) { a = TW_ACK_INVALID_STATE; break; }
        if (c_observer) { a = TW_ACK_ROLE_VIOLATION; break; }
        if (op.arg < 1) { a = TW_ACK_EXPECTED_MISMATCH; break; }
        const int g = op.group;
        if (g < 0 || g >= TW_TK_MAX_GROUPS) { a = TW_ACK_TOO_MANY; k.limit = 1; break; }
        const uint32_t arrived = __shfl_sync(kFull, k.g_arrived, g);
        const int64_t expected = __shfl_sync(kFull, k.g_expected, g);
        if (arrived != 0 && expected != op.arg) { a = TW_ACK_EXPECTED_MISMATCH; break; }
        const uint32_t now_arrived = arrived | (1u << c);
        const int64_t now_expected = arrived ? expected : op.arg;
        if (lane == c) {
          k.exempt = true;
          k.pending = false;
        }
        if (__popc(now_arrived) == now_expected) {
          const int64_t gen = __shfl_sync(kFull, k.g_gen, g);
          tk_emit(k, 1, g, gen, op_index);
          if (lane == g) {
            k.g_gen++;
            k.g_arrived = 0;
            k.g_expected = 0;
          }
          if ((now_arrived >> lane) & 1u) k.exempt = false;
        } else if (lane == g) {
          k.g_arrived = now_arrived;
          k.g_expected = now_expected;
        }
        tk_try_resolve(k, op_index);
        break;
      }
      case TW_OP_DEREGISTER:  // timekeeper.py:294-314
        if (!cvalid) { a = TW_ACK_UNKNOWN_CLIENT; break; }
        if (c_active) {
          if (lane == c) {
            k.active = false;
            k.pending = false;
            k.exempt = false;
          }
          k.g_arrived &= ~(1u << c);
        }
        tk_try_resolve(k, op_index);
        break;
      case TW_OP_ADVANCE_CLOCK:
        k.wall += op.arg;
        break;
      default:
        a = TW_ACK_UNKNOWN_CLIENT;
        break;
    }
    if (lane == 0) ack[i] = a;
  }
  if (lane == 0) {
    tw_tk_final f;
    f.offset_ns = k.offset;
    f.seq = k.seq;
    f.wall_ns = k.wall;
    f.rounds = k.rounds;
    f.broadcasts = k.broadcasts;
    f.n_events = k.n_ev;
    f.status = k.limit ? 2 : (k.n_ev > k.ev_cap ? 1 : 0);
    f.pad = 0;
    f.pad2 = 0;
    fin[s] = f;
  }
}

// Wide op streams (more than 32 clients or groups; BarrierCore itself has no limit):
// still one warp per stream, but client and group state live in the warp's shared-memory
// slice and lanes stride over clients, so eligible / |pending| are lane-strided counts and
// t_min a lane-strided min finished by one warp reduction; a group's arrived set is a
// bitset of TW_TK_MAX_CLIENTS_WIDE bits. Same state machine and acks as k_tk_replay.
constexpr int kTkWideWarps = 2;
constexpr int kWideWords = TW_TK_MAX_CLIENTS_WIDE / 32;
struct TkWideSlice {
  int64_t target[TW_TK_MAX_CLIENTS_WIDE];
  int64_t g_gen[TW_TK_MAX_GROUPS_WIDE], g_expected[TW_TK_MAX_GROUPS_WIDE];
  uint32_t g_arrived[TW_TK_MAX_GROUPS_WIDE][kWideWords];
  uint8_t flags[TW_TK_MAX_CLIENTS_WIDE];  // bit 0 active, 1 observer, 2 pending, 3 exempt
};
constexpr uint8_t kFActive = 1, kFObserver = 2, kFPending = 4, kFExempt = 8;

struct TkWide {
  int64_t wall, offset, seq, last_bcast, cooldown, rounds, broadcasts, n_ev, ev_cap;
  int sealed, nclients, limit;
  tw_tk_event* ev;
};

__device__ __forceinline__ void tkw_emit(TkWide& k, int kind, int64_t a, int64_t b, int op_index) {
  if ((threadIdx.x & 31) == 0 && k.n_ev < k.ev_cap) {
    tw_tk_event e;
    e.offset_ns = a;
    e.seq = b;
    e.wall_ns = k.wall;
    e.kind = kind;
    e.op_index = op_index;
    k.ev[k.n_ev] = e;
  }
  k.n_ev++;
}

__device__ __forceinline__ void tkw_try_resolve(TkWide& k, TkWideSlice& w, int op_index) {
  if (!k.sealed) return;  // timekeeper.py:318-324
  const int lane = threadIdx.x & 31;
  int elig = 0, npend = 0;
  int64_t t = INT64_MAX;
  for (int c = lane; c < k.nclients; c += 32) {
    const uint8_t f = w.flags[c];
    elig += (f & (kFActive | kFObserver | kFExempt)) == kFActive;
    if (f & kFPending) {
      npend++;
      t = w.target[c] < t ? w.target[c] : t;
    }
  }
  elig = __reduce_add_sync(kFull, elig);
  npend = __reduce_add_sync(kFull, npend);
  if (elig <= 0 || npend != elig) return;
  // _resolve: timekeeper.py:326-366
  const int64_t t_min = warp_min_i64(t);
  if (k.wall < t_min && k.last_bcast != INT64_MIN && k.cooldown > 0) {
    const int64_t wait = k.last_bcast + k.cooldown - k.wall;
    if (wait > 0) k.wall += fake_sleep_ns(wait);
  }
  k.rounds++;
  if (k.wall < t_min) {
    const int64_t cand = t_min - k.wall;
    if (cand > k.offset) k.offset = cand;
    k.seq++;
    k.broadcasts++;
    tkw_emit(k, 0, k.offset, k.seq, op_index);
    k.last_bcast = k.wall;
  }
  for (int c = lane; c < k.nclients; c += 32) w.flags[c] &= (uint8_t)~kFPending;
  __syncwarp();
}

__global__ void __launch_bounds__(32 * kTkWideWarps) k_tk_replay_wide(
    const tw_tk_op* __restrict__ ops, const int64_t* __restrict__ op_off, int32_t n_streams,
    const int64_t* __restrict__ wall0, const int64_t* __restrict__ cooldown,
    const uint8_t* __restrict__ suppress, int32_t* __restrict__ ack, tw_tk_event* __restrict__ ev,
    const int64_t* __restrict__ ev_off, tw_tk_final* __restrict__ fin) {
  extern __shared__ __align__(16) char tkw_smem[];
  const int lane = threadIdx.x & 31;
  const int s = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (s >= n_streams) return;  // warp-uniform
  TkWideSlice& w = reinterpret_cast<TkWideSlice*>(tkw_smem)[threadIdx.x >> 5];
  for (int g = 0; g < TW_TK_MAX_GROUPS_WIDE; g++) {
    if (lane == 0) {
      w.g_gen[g] = 0;
      w.g_expected[g] = 0;
    }
    w.g_arrived[g][lane] = 0;  // kWideWords == 32
  }
  __syncwarp();
  TkWide k;
  k.wall = wall0[s];
  k.offset = 0;
  k.seq = 0;
  k.last_bcast = INT64_MIN;
  k.cooldown = cooldown[s];
  k.rounds = k.broadcasts = k.n_ev = 0;
  k.ev = ev ? ev + ev_off[s] : nullptr;
  k.ev_cap = ev ? ev_off[s + 1] - ev_off[s] : 0;
  k.sealed = 0;
  k.nclients = 0;
  k.limit = 0;
  (void)suppress;  // suppressed broadcasts are still CLOCK_UPDATE events here (as k_tk_replay)

  const int64_t o0 = op_off[s], o1 = op_off[s + 1];
  for (int64_t i = o0; i < o1; i++) {
    const tw_tk_op op = ops[i];  // same address in every lane: one broadcast load
    const int op_index = (int)(i - o0);
    const int c = op.client;
    int a = TW_ACK_OK;
    // _require_client (timekeeper.py:121-127), for ops that name a client
    const bool cvalid = c >= 0 && c < k.nclients;
    const uint8_t cf = cvalid ? w.flags[c] : 0;
    const bool c_active = (cf & kFActive) != 0, c_observer = (cf & kFObserver) != 0;
    switch (op.type) {
      case TW_OP_REGISTER_ACTOR:
      case TW_OP_REGISTER_OBSERVER:  // timekeeper.py:155-182
        if (k.sealed) { a = TW_ACK_REGISTRATION_SEALED; break; }
        if (k.nclients >= TW_TK_MAX_CLIENTS_WIDE) { a = TW_ACK_TOO_MANY; k.limit = 1; break; }
        if (lane == 0) {
          w.flags[k.nclients] = kFActive | (op.type == TW_OP_REGISTER_OBSERVER ? kFObserver : 0);
          w.target[k.nclients] = 0;
        }
        k.nclients++;
        break;
      case TW_OP_SEAL: {  // timekeeper.py:184-200
        if (!k.sealed) {
          bool any = false;
          for (int q = lane; q < k.nclients; q += 32) any |= (w.flags[q] & (kFActive | kFObserver)) == kFActive;
          if (!__any_sync(kFull, any)) { a = TW_ACK_NO_ACTORS; break; }
          k.sealed = 1;
        }
        tkw_try_resolve(k, w, op_index);
        break;
      }
      case TW_OP_JUMP:  // timekeeper.py:202-225
        if (!cvalid) { a = TW_ACK_UNKNOWN_CLIENT; break; }
        if (!c_active) { a = TW_ACK_INVALID_STATE; break; }
        if (c_observer) { a = TW_ACK_ROLE_VIOLATION; break; }
        if (op.arg <= 0) { a = TW_ACK_INVALID_DELTA; break; }
        if (lane == 0) {
          w.target[c] = op.arg;  // a re-request overwrites
          w.flags[c] = (uint8_t)((cf | kFPending) & ~kFExempt);
        }
        __syncwarp();
        tkw_try_resolve(k, w, op_index);
        break;
      case TW_OP_ENTER: {  // timekeeper.py:227-292
        if (!cvalid) { a = TW_ACK_UNKNOWN_CLIENT; break; }
        if (!c_active) { a = TW_ACK_INVALID_STATE; break; }
        if (c_observer) { a = TW_ACK_ROLE_VIOLATION; break; }
        if (op.arg < 1) { a = TW_ACK_EXPECTED_MISMATCH; break; }
        const int g = op.group;
        if (g < 0 || g >= TW_TK_MAX_GROUPS_WIDE) { a = TW_ACK_TOO_MANY; k.limit = 1; break; }
        const uint32_t word = w.g_arrived[g][lane];
        const int n_arr = __reduce_add_sync(kFull, (unsigned)__popc(word));
        const int64_t expected = w.g_expected[g];
        if (n_arr != 0 && expected != op.arg) { a = TW_ACK_EXPECTED_MISMATCH; break; }
        const uint32_t now_word = word | (lane == (c >> 5) ? 1u << (c & 31) : 0u);
        const int n_now = __reduce_add_sync(kFull, (unsigned)__popc(now_word));
        const int64_t now_expected = n_arr ? expected : op.arg;
        __syncwarp();
        if (lane == 0) w.flags[c] = (uint8_t)((cf | kFExempt) & ~kFPending);
        __syncwarp();
        if (n_now == now_expected) {
          tkw_emit(k, 1, g, w.g_gen[g], op_index);
          // the released members stop being exempt (timekeeper.py:280-289)
          for (int b = 0; b < 32; b++) {
            const uint32_t m = __shfl_sync(kFull, now_word, b);
            if ((m >> lane) & 1u) {
              const int q = 32 * b + lane;
              w.flags[q] = (uint8_t)(w.flags[q] & ~kFExempt);
            }
          }
          __syncwarp();
          if (lane == 0) {
            w.g_gen[g]++;
            w.g_expected[g] = 0;
          }
          w.g_arrived[g][lane] = 0;
        } else {
          w.g_arrived[g][lane] = now_word;
          if (lane == 0) w.g_expected[g] = now_expected;
        }
        __syncwarp();
        tkw_try_resolve(k, w, op_index);
        break;
      }
      case TW_OP_DEREGISTER:  // timekeeper.py:294-314
        if (!cvalid) { a = TW_ACK_UNKNOWN_CLIENT; break; }
        if (c_active) {
          if (lane == 0) w.flags[c] = (uint8_t)(cf & ~(kFActive | kFPending | kFExempt));
          if (lane == (c >> 5))
            for (int g = 0; g < TW_TK_MAX_GROUPS_WIDE; g++) w.g_arrived[g][lane] &= ~(1u << (c & 31));
        }
        __syncwarp();
        tkw_try_resolve(k, w, op_index);
        break;
      case TW_OP_ADVANCE_CLOCK:
        k.wall += op.arg;
        break;
      default:
        a = TW_ACK_UNKNOWN_CLIENT;
        break;
    }
    if (lane == 0) ack[i] = a;
    __syncwarp();
  }
  if (lane == 0) {
    tw_tk_final f;
    f.offset_ns = k.offset;
    f.seq = k.seq;
    f.wall_ns = k.wall;
    f.rounds = k.rounds;
    f.broadcasts = k.broadcasts;
    f.n_events = k.n_ev;
    f.status = k.limit ? 2 : (k.n_ev > k.ev_cap ? 1 : 0);
    f.pad = 0;
    f.pad2 = 0;
    fin[s] = f;
  }
}

// One round of min-advance for n_cfg Timekeepers with A <= 32 actor slots each: one
// warp resolves 32 consecutive Timekeepers. Their 32*A pending
// targets are one contiguous run, read with coalesced loads into the warp's slice of
// shared memory; lane l then owns Timekeeper c0 + l (eligibility bits, pending count,
// t_min over its A entries) and its state (wall, last broadcast, offset, seq) is read
// and written as coalesced rows; resolved Timekeepers' targets are cleared with
// coalesced stores (timekeeper.py:318-366). (A warp-per-Timekeeper segmented-min form
// reached 18% of HBM bandwidth against 83% for this one; profiles/README.md.)
constexpr int kTkWarps2 = 8;
__global__ void __launch_bounds__(32 * kTkWarps2) k_tk_resolve_rows(
    int64_t* __restrict__ pending, const uint32_t* __restrict__ elig, int32_t n_cfg, int32_t A,
    int64_t cooldown, int64_t conv_cooldown, int64_t* __restrict__ offset, int64_t* __restrict__ seq,
    int64_t* __restrict__ wall, int64_t* __restrict__ last_bcast, int8_t* __restrict__ bcast) {
  extern __shared__ int64_t tk_rows[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t c0 = ((int64_t)blockIdx.x * kTkWarps2 + wib) * 32;
  if (c0 >= n_cfg) return;
  const int n_here = (int)min((int64_t)32, (int64_t)n_cfg - c0);
  const int total = n_here * A;
  int64_t* buf = tk_rows + (size_t)wib * 32 * A;
  int64_t* row = pending + c0 * A;
  for (int q = lane; q < total; q += 32) buf[q] = row[q];
  __syncwarp();
  const int64_t c = c0 + lane;
  const bool live = lane < n_here;
  const uint32_t m = live ? __ldg(elig + c) : 0u;
  int64_t t = INT64_MAX;
  int nel = 0, nhas = 0;
  for (int a = 0; a < A; a++) {
    if ((m >> a) & 1u) {
      const int64_t v = buf[lane * A + a];
      nel++;
      if (v != INT64_MAX) {
        nhas++;
        t = v < t ? v : t;
      }
    }
  }
  const bool resolves = live && nel > 0 && nhas == nel;  // sealed assumed; |pending| == eligible
  if (live) {
    if (!resolves) {
      bcast[c] = -1;
    } else {
      int64_t w = wall[c];
      const int64_t lb = last_bcast[c];
      if (w < t && lb != INT64_MIN && cooldown > 0) {
        const int64_t wait = lb + cooldown - w;
        if (wait > 0) w += (wait == cooldown) ? conv_cooldown : fake_sleep_ns(wait);
      }
      wall[c] = w;
      if (w < t) {
        const int64_t cand = t - w;
        const int64_t o = offset[c];
        if (cand > o) offset[c] = cand;
        seq[c] += 1;
        last_bcast[c] = w;
        bcast[c] = 1;
      } else {
        bcast[c] = 0;
      }
    }
  }
  const unsigned rmask = __ballot_sync(kFull, resolves);
  if (rmask) {  // pending.clear() of the resolved Timekeepers
    const uint32_t inv = (65536u + (uint32_t)A - 1u) / (uint32_t)A;  // q / A for q < 32 A, A <= 32
    for (int q = lane; q < total; q += 32)
      if ((rmask >> ((uint32_t)q * inv >> 16)) & 1u) row[q] = INT64_MAX;
  }
}

// One round for Timekeepers of A > 32 actor slots (eligibility: ceil(A/32) words each):
// one warp per Timekeeper, lanes striding over its A pending targets (coalesced), the
// eligible and pending counts one REDUX each and t_min one warp min: the per-config
// segmented reduction; lane 0 applies _resolve and the warp clears the row
// (timekeeper.py:318-366).
constexpr int kTkWideRes = 8;  // warps (Timekeepers) per CTA
__global__ void __launch_bounds__(32 * kTkWideRes) k_tk_resolve_wide(
    int64_t* __restrict__ pending, const uint32_t* __restrict__ elig, int32_t n_cfg, int32_t A,
    int64_t cooldown, int64_t conv_cooldown, int64_t* __restrict__ offset, int64_t* __restrict__ seq,
    int64_t* __restrict__ wall, int64_t* __restrict__ last_bcast, int8_t* __restrict__ bcast) {
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * kTkWideRes + (threadIdx.x >> 5);
  if (c >= n_cfg) return;  // warp-uniform
  const int W = (A + 31) >> 5;
  int64_t* row = pending + c * A;
  const uint32_t* m = elig + c * W;
  int nel = 0, nhas = 0;
  int64_t t = INT64_MAX;
  for (int a = lane; a < A; a += 32) {
    if ((__ldg(m + (a >> 5)) >> (a & 31)) & 1u) {
      const int64_t v = row[a];
      nel++;
      if (v != INT64_MAX) {
        nhas++;
        t = v < t ? v : t;
      }
    }
  }
  nel = (int)__reduce_add_sync(kFull, (unsigned)nel);
  nhas = (int)__reduce_add_sync(kFull, (unsigned)nhas);
  const bool resolves = nel > 0 && nhas == nel;  // sealed assumed; |pending| == eligible
  t = warp_min_i64(t);
  if (lane == 0) {
    if (!resolves) {
      bcast[c] = -1;
    } else {
      int64_t w = wall[c];
      const int64_t lb = last_bcast[c];
      if (w < t && lb != INT64_MIN && cooldown > 0) {
        const int64_t wait = lb + cooldown - w;
        if (wait > 0) w += (wait == cooldown) ? conv_cooldown : fake_sleep_ns(wait);
      }
      wall[c] = w;
      if (w < t) {
        const int64_t cand = t - w;
        if (cand > offset[c]) offset[c] = cand;
        seq[c] += 1;
        last_bcast[c] = w;
        bcast[c] = 1;
      } else {
        bcast[c] = 0;
      }
    }
  }
  if (resolves)  // pending.clear()
    for (int a = lane; a < A; a += 32) row[a] = INT64_MAX;
}

}  // namespace twb

using namespace twb;

extern "C" int tw_tk_replay(const tw_tk_op* ops, const int64_t* op_off, int32_t n_streams,
                            const int64_t* wall0_ns, const int64_t* cooldown_ns,
                            const uint8_t* suppress, int32_t* ack, tw_tk_event* ev,
                            const int64_t* ev_off, tw_tk_final* fin, void* stream) {
  if (n_streams < 0 || (n_streams > 0 && (!op_off || !wall0_ns || !cooldown_ns || !fin)) ||
      (ev && !ev_off)) {
    set_error("tw_tk_replay: bad arguments");
    return TW_EINVAL;
  }
  if (n_streams == 0) return TW_OK;
  const int64_t threads = (int64_t)n_streams * 32;
  const int grid = (int)((threads + kTkThreads - 1) / kTkThreads);
  k_tk_replay<<<grid, kTkThreads, 0, (cudaStream_t)stream>>>(ops, op_off, n_streams, wall0_ns,
                                                              cooldown_ns, suppress, ack, ev, ev_off, fin);
  count_launch();
  return check_launch("tw_tk_replay");
}

extern "C" int tw_tk_replay_wide(const tw_tk_op* ops, const int64_t* op_off, int32_t n_streams,
                                 const int64_t* wall0_ns, const int64_t* cooldown_ns,
                                 const uint8_t* suppress, int32_t* ack, tw_tk_event* ev,
                                 const int64_t* ev_off, tw_tk_final* fin, void* stream) {
  if (n_streams < 0 || (n_streams > 0 && (!op_off || !wall0_ns || !cooldown_ns || !fin)) ||
      (ev && !ev_off)) {
    set_error("tw_tk_replay_wide: bad arguments");
    return TW_EINVAL;
  }
  if (n_streams == 0) return TW_OK;
  const int64_t threads = (int64_t)n_streams * 32;
  const int block = 32 * kTkWideWarps;
  const int grid = (int)((threads + block - 1) / block);
  const size_t smem = sizeof(TkWideSlice) * kTkWideWarps;
  cudaFuncSetAttribute(k_tk_replay_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_tk_replay_wide<<<grid, block, smem, (cudaStream_t)stream>>>(ops, op_off, n_streams, wall0_ns, cooldown_ns,
                                                                 suppress, ack, ev, ev_off, fin);
  count_launch();
  return check_launch("tw_tk_replay_wide");
}

extern "C" int tw_tk_resolve_wide(int64_t* pending, const uint32_t* eligible_words, int32_t n_cfg, int32_t A,
                                  int64_t cooldown_ns, int64_t* offset_ns, int64_t* seq, int64_t* wall_ns,
                                  int64_t* last_bcast_ns, int8_t* broadcast, void* stream) {
  if (A < 1 || n_cfg < 0 || cooldown_ns < 0) {
    set_error("tw_tk_resolve_wide: need A >= 1, n_cfg >= 0, cooldown >= 0");
    return TW_EINVAL;
  }
  if (n_cfg == 0) return TW_OK;
  const double secs = (double)cooldown_ns / 1e9;  // as tw_tk_resolve
  const int64_t conv = cooldown_ns > 0 ? (int64_t)nearbyint(secs * 1e9) : 0;
  const int blocks = (int)(((int64_t)n_cfg + kTkWideRes - 1) / kTkWideRes);
  k_tk_resolve_wide<<<blocks, 32 * kTkWideRes, 0, (cudaStream_t)stream>>>(
      pending, eligible_words, n_cfg, A, cooldown_ns, conv, offset_ns, seq, wall_ns, last_bcast_ns, broadcast);
  count_launch();
  return check_launch("tw_tk_resolve_wide");
}

extern "C" int tw_tk_resolve(int64_t* pending, const uint32_t* eligible_mask, int32_t n_cfg, int32_t A,
                             int64_t cooldown_ns, int64_t* offset_ns, int64_t* seq, int64_t* wall_ns,
                             int64_t* last_bcast_ns, int8_t* broadcast, void* stream) {
  if (A < 1 || A > 32 || n_cfg < 0 || cooldown_ns < 0) {
    set_error("tw_tk_resolve: need 1 <= A <= 32, n_cfg >= 0, cooldown >= 0");
    return TW_EINVAL;
  }
  if (n_cfg == 0) return TW_OK;
  cudaStream_t s = (cudaStream_t)stream;
  // FakeClock.sleep(cooldown / 1e9) -> int(round(seconds * 1e9)) in host IEEE fp64
  // (SSE2: each op rounds once, nearest-even), the same ops as fake_sleep_ns
  const double secs = (double)cooldown_ns / 1e9;
  const int64_t conv = cooldown_ns > 0 ? (int64_t)nearbyint(secs * 1e9) : 0;
  {
    const int64_t warps = ((int64_t)n_cfg + 31) / 32;
    const int blocks = (int)((warps + kTkWarps2 - 1) / kTkWarps2);
    const size_t smem = (size_t)kTkWarps2 * 32 * A * sizeof(int64_t);
    if (smem > 48 * 1024)  // A > 24: opt in to more than the default dynamic shared memory
      cudaFuncSetAttribute(k_tk_resolve_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_tk_resolve_rows<<<blocks, 32 * kTkWarps2, smem, s>>>(pending, eligible_mask, n_cfg, A, cooldown_ns, conv,
                                                           offset_ns, seq, wall_ns, last_bcast_ns, broadcast);
  }
  count_launch();
  return check_launch("tw_tk_resolve");
}
