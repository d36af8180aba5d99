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

// One round of min-advance for n_cfg Timekeepers with A actor slots each.
template <int AP>
__global__ void __launch_bounds__(kTkThreads) k_tk_resolve(
    int64_t* __restrict__ pending, const uint32_t* __restrict__ elig, int32_t n_cfg, int32_t A,
    int64_t cooldown, int64_t* __restrict__ offset, int64_t* __restrict__ seq,
    int64_t* __restrict__ wall, int64_t* __restrict__ last_bcast, int8_t* __restrict__ bcast) {
  constexpr int kPerWarp = 32 / AP;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int seg = lane / AP, a = lane % AP;
  const int64_t c = warp * kPerWarp + seg;
  const bool live = c < n_cfg;
  const uint32_t m = live ? __ldg(elig + c) : 0u;
  const bool el = live && a < A && ((m >> a) & 1u);
  int64_t p = el ? pending[c * A + a] : INT64_MAX;
  const unsigned seg_mask = (AP == 32) ? kFull : (((1u << AP) - 1u) << (seg * AP));
  const unsigned has = __ballot_sync(kFull, el && p != INT64_MAX) & seg_mask;
  const unsigned els = __ballot_sync(kFull, el) & seg_mask;
  // segmented int64 min inside the AP-lane segment
  int64_t t = p;
#pragma unroll
  for (int o = AP / 2; o > 0; o >>= 1) {
    const int64_t w = __shfl_xor_sync(kFull, t, o);
    t = w < t ? w : t;
  }
  const bool resolves = live && els != 0 && has == els;  // sealed assumed; |pending| == eligible
  if (live && a == 0) {
    if (!resolves) {
      bcast[c] = -1;
    } else {
      int64_t w = wall[c];
      const int64_t lb = last_bcast[c];
      if (w < t && lb != INT64_MIN && cooldown > 0) {
        const int64_t wait = lb + cooldown - w;
        if (wait > 0) w += fake_sleep_ns(wait);
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
  if (resolves && a < A) pending[c * A + a] = INT64_MAX;  // pending.clear()
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

extern "C" int tw_tk_resolve(int64_t* pending, const uint32_t* eligible_mask, int32_t n_cfg, int32_t A,
                             int64_t cooldown_ns, int64_t* offset_ns, int64_t* seq, int64_t* wall_ns,
                             int64_t* last_bcast_ns, int8_t* broadcast, void* stream) {
  if (A < 1 || A > 32 || n_cfg < 0 || cooldown_ns < 0) {
    set_error("tw_tk_resolve: need 1 <= A <= 32, n_cfg >= 0, cooldown >= 0");
    return TW_EINVAL;
  }
  if (n_cfg == 0) return TW_OK;
  int ap = 1;
  while (ap < A) ap <<= 1;
  const int64_t warps = ((int64_t)n_cfg * ap + 31) / 32;
  const int grid = (int)((warps * 32 + kTkThreads - 1) / kTkThreads);
  cudaStream_t s = (cudaStream_t)stream;
#define TW_RESOLVE(APV)                                                                      \
  k_tk_resolve<APV><<<grid, kTkThreads, 0, s>>>(pending, eligible_mask, n_cfg, A, cooldown_ns, \
                                                offset_ns, seq, wall_ns, last_bcast_ns, broadcast)
  switch (ap) {
    case 1: TW_RESOLVE(1); break;
    case 2: TW_RESOLVE(2); break;
    case 4: TW_RESOLVE(4); break;
    case 8: TW_RESOLVE(8); break;
    case 16: TW_RESOLVE(16); break;
    default: TW_RESOLVE(32); break;
  }
#undef TW_RESOLVE
  count_launch();
  return check_launch("tw_tk_resolve");
}
