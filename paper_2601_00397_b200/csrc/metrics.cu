// metrics.cu — per-config latency summary on device.
//
// Reference: metrics.py:38-124 (RequestOutcome, percentile, _stats, RunReport.summary)
// and collect_metrics (metrics.py:173-253) over an oracle-mode event log
// (runner.py:339-365). The event log itself never exists here: tw_sim_many already
// wrote each request's FIRST_TOKEN and FINISHED stamps, which is all the summary
// needs. One CTA per config:
//   * one pass over the requests: missing stamps, output tokens, max FINISHED, exact
//     int64 sums of TTFT and e2e (all partial sums of non-negative integers below
//     2^53 are exact in fp64, so Python's compensated float sum equals them);
//   * TPOT values (correctly rounded int/int divisions) are scattered into shared
//     memory in the caller's arrival order and summed by one thread with CPython's
//     Neumaier recurrence (bltinmodule.c builtin_sum, CPython >= 3.12);
//   * each metric's values become order-preserving uint64 keys in shared memory, and
//     the keys at the nearest ranks ceil(p/100.0*n) - 1 are selected without sorting:
//     MSD radix selection over 8-bit digits, all three ranks per pass, starting
//     below the bits every key shares. A bitonic sort of the keys was
//     shared-memory-bandwidth-bound: 0.185 -> 0.123 ms for 1,024 x 1,000.
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace twb {

#ifndef TWB_MET_THREADS
#define TWB_MET_THREADS 128
#endif
constexpr int kMetThreads = TWB_MET_THREADS;
constexpr int kMetWarps = kMetThreads / 32;
// keys (8 B per request) fill the dynamic shared memory: the largest workload a summary
// takes is (max opt-in shared memory - the kernel's static shared memory) / 8
constexpr int kMetStaticSmem = 8192;

// total-order key of a non-NaN double (negatives flipped, positives offset)
__device__ __forceinline__ uint64_t dkey(double v) {
  const uint64_t b = (uint64_t)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double dval(uint64_t k) {
  return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffULL) : ~k));
}

// 0-based index of the nearest-rank percentile p of n sorted values (metrics.py:65-71)
__device__ __forceinline__ int nearest_rank_index(int p, int n) {
  const double q = __dmul_rn(__ddiv_rn((double)p, 100.0), (double)n);
  const int r = (int)ceil(q);
  return (r < 1 ? 1 : r) - 1;
}

// CPython sum() of floats: Neumaier's compensated recurrence, then f += c when c is a
// non-zero finite number. NaN entries (no value) are skipped.
__device__ double neumaier_sum(const double* v, int n) {
  double f = 0.0, c = 0.0;
  // branch-free body (a NaN entry adds +0.0, which changes neither f nor c), unrolled
  // so the shared-memory loads run ahead of the two fp64 dependency chains
#pragma unroll 8
  for (int i = 0; i < n; i++) {
    double x = v[i];
    x = isnan(x) ? 0.0 : x;
    const double t = __dadd_rn(f, x);
    const double e = fabs(f) >= fabs(x) ? __dadd_rn(__dsub_rn(f, t), x) : __dadd_rn(__dsub_rn(x, t), f);
    c = __dadd_rn(c, e);
    f = t;
  }
  if (c != 0.0 && isfinite(c)) f = __dadd_rn(f, c);
  return f;
}

struct MetParams {
  const tw_sim_cfg* cfgs;
  int32_t n_cfg;
  const int64_t* wl_off;
  const int64_t* ts;
  const int32_t* output;
  const int64_t* req_base;
  const int64_t* first;
  const int64_t* finish;
  const tw_sim_result* sim;
  const int32_t* sum_order;
  int32_t cap;  // keys capacity
  uint64_t* gkeys;  // global-memory keys (cap per CTA) for workloads shared memory cannot hold
  tw_run_metrics* out;
  // TPOT values in caller order, cap per config (k_metrics_tpot sums them one lane per
  // config); nullptr: one thread of the config's CTA sums them (scratch too small)
  double* tpot_vals;
};

// CPython's sum of one config's TPOT values per lane: 32 configs per warp, each lane running
// the same Neumaier recurrence as neumaier_sum over its config's row (caller order), then
// mean = sum / count. Inside k_metrics the sum was one thread's serial loop while the CTA
// waited: ~22% of the kernel's instructions (ncu, config 5).
__global__ void __launch_bounds__(128) k_metrics_tpot(MetParams p) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= p.n_cfg) return;
  tw_run_metrics* o = p.out + c;
  if (o->status != TW_METRICS_OK || o->tpot.count <= 0) return;
  const tw_sim_cfg& cfg = p.cfgs[c];
  const int n = (int)(p.wl_off[cfg.workload_id + 1] - p.wl_off[cfg.workload_id]);
  const double* v = p.tpot_vals + (int64_t)c * p.cap;
  double f = 0.0, cc = 0.0;
#pragma unroll 4
  for (int i = 0; i < n; i++) {
    double x = __ldg(v + i);
    x = isnan(x) ? 0.0 : x;
    const double t = __dadd_rn(f, x);
    const double e = fabs(f) >= fabs(x) ? __dadd_rn(__dsub_rn(f, t), x) : __dadd_rn(__dsub_rn(x, t), f);
    cc = __dadd_rn(cc, e);
    f = t;
  }
  if (cc != 0.0 && isfinite(cc)) f = __dadd_rn(f, cc);
  o->tpot.mean = __ddiv_rn(f, (double)o->tpot.count);
}

struct BlockRed {
  int64_t miss, tokens, maxfin, s_ttft, s_e2e, n_tpot;
};

__device__ __forceinline__ int64_t warp_max_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t w = __shfl_xor_sync(kFull, v, o);
    v = w > v ? w : v;
  }
  return v;
}

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t w = __shfl_xor_sync(kFull, v, o);
    v = w < v ? w : v;
  }
  return v;
}
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t w = __shfl_xor_sync(kFull, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// The keys at 0-based ranks r[0..2] (< the number of valid keys) of keys[0, n) in
// ascending order, without sorting: MSD radix selection, 8-bit digits below the bits
// every valid key shares, all three ranks per pass. Keys equal to ~0 (no value) are
// never selected and sit above every valid key, so they are skipped.
// After the first digit, the keys still matching one of the three prefixes (usually a few
// dozen of ~1,000) are compacted into a small buffer and the later passes scan only those.
constexpr int kMetCand = 448;
__device__ void select3(const uint64_t* keys, int n, const int r[3], uint64_t out[3]) {
  __shared__ __align__(16) uint32_t hist[3][256];
  __shared__ uint64_t pre[3], red_mn[kMetWarps], red_mx[kMetWarps];
  __shared__ uint64_t cand[kMetCand];
  __shared__ int rem[3], sh_shift, ncand;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint64_t mn = ~0ULL, mx = 0;
  for (int i = tid; i < n; i += kMetThreads) {
    const uint64_t k = keys[i];
    if (k != ~0ULL) {
      mn = k < mn ? k : mn;
      mx = k > mx ? k : mx;
    }
  }
  mn = warp_min_u64(mn);
  mx = warp_max_u64(mx);
  if (lane == 0) {
    red_mn[warp] = mn;
    red_mx[warp] = mx;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < kMetWarps; w++) {
      mn = red_mn[w] < mn ? red_mn[w] : mn;
      mx = red_mx[w] > mx ? red_mx[w] : mx;
    }
    mn = red_mn[0] < mn ? red_mn[0] : mn;
    mx = red_mx[0] > mx ? red_mx[0] : mx;
    const uint64_t diff = mn ^ mx;
    // the first digit is the 8 bits from the highest differing bit h down (all of it split
    // 256 ways, not the few bits of an aligned digit); -8: every valid key is the same (mn)
    const int h = diff ? 63 - __clzll((long long)diff) : -1;
    sh_shift = h < 0 ? -8 : (h >= 7 ? h - 7 : 0);
    const uint64_t keep = h < 0 ? ~0ULL : (h >= 63 ? 0ULL : ~((2ULL << h) - 1));
    for (int t = 0; t < 3; t++) {
      pre[t] = mn & keep;
      rem[t] = r[t];
    }
  }
  __syncthreads();
  const uint64_t* src = keys;
  int nsrc = n;
  bool compacted = false;
  // digits of 8 bits from sh_shift down, the last one (at bit 0) narrower
  for (int shift = sh_shift, width = sh_shift >= 0 ? min(8, 64 - sh_shift) : 0, top = shift + width; shift >= 0;
       top = shift, width = min(8, shift), shift -= width) {
    if (width == 0) break;
    // the first digit: every target still shares the prefix, one histogram serves all three
    const bool one = shift == sh_shift;
    const uint32_t dmask = (1u << width) - 1u;
    for (int i = tid; i < (one ? 256 : 3 * 256) / 4; i += kMetThreads)
      reinterpret_cast<uint4*>(&hist[0][0])[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    const uint64_t p0 = pre[0], p1 = pre[1], p2 = pre[2];
    for (int i = tid; i < nsrc; i += kMetThreads) {
      const uint64_t k = src[i];
      if (k == ~0ULL) continue;
      const uint32_t dg = (uint32_t)(k >> shift) & dmask;
      if (one) {
        atomicAdd(&hist[0][dg], 1u);
      } else {
        const int hs = top;  // < 64: not the first digit
        if (((k ^ p0) >> hs) == 0) atomicAdd(&hist[0][dg], 1u);
        if (((k ^ p1) >> hs) == 0) atomicAdd(&hist[1][dg], 1u);
        if (((k ^ p2) >> hs) == 0) atomicAdd(&hist[2][dg], 1u);
      }
    }
    __syncthreads();
    if (warp < 3) {  // warp t picks target t's digit
      const int t = warp;
      uint32_t c[8], sl = 0;
#pragma unroll
      for (int b = 0; b < 8; b++) {
        c[b] = hist[one ? 0 : t][8 * lane + b];
        sl += c[b];
      }
      uint32_t incl = sl;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t w = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += w;
      }
      const int target = rem[t];
      __syncwarp();  // every lane has read rem[t] before one of them rewrites it
      const unsigned hit = __ballot_sync(kFull, (int)incl > target);
      if (lane == __ffs(hit) - 1) {
        int cum = (int)(incl - sl);
        int d = 8 * lane;
#pragma unroll
        for (int b = 0; b < 8; b++) {
          if (cum + (int)c[b] > target) break;
          cum += (int)c[b];
          d++;
        }
        rem[t] = target - cum;
        pre[t] |= (uint64_t)d << shift;
      }
    }
    if (tid == 0) ncand = 0;
    __syncthreads();
    if (!compacted && shift > 0) {  // keep the keys that can still be selected
      const uint64_t q0 = pre[0], q1 = pre[1], q2 = pre[2];
      for (int i = tid; i < nsrc; i += kMetThreads) {
        const uint64_t k = src[i];
        if (k != ~0ULL && (((k ^ q0) >> shift) == 0 || ((k ^ q1) >> shift) == 0 || ((k ^ q2) >> shift) == 0)) {
          const int j = atomicAdd(&ncand, 1);
          if (j < kMetCand) cand[j] = k;
        }
      }
      __syncthreads();
      if (ncand <= kMetCand) {
        src = cand;
        nsrc = ncand;
        compacted = true;
      }
      __syncthreads();
    }
  }
  out[0] = pre[0];
  out[1] = pre[1];
  out[2] = pre[2];
  __syncthreads();
}

constexpr uint64_t kSignBit = 0x8000000000000000ULL;

// nearest-rank p50 / p90 / p99 of the count valid keys among keys[0, n) (metrics.py:62-79)
// kInt: keys are int64 values with the sign bit flipped (TTFT, e2e: the reference's float(t)
// is monotone in t, so the order statistics of the floats are the floats of the int64 order
// statistics, and integer keys share more high bits: fewer radix passes than float keys)
template <bool kInt>
__device__ void stats_from_keys(const uint64_t* keys, int n, int count, double mean, tw_latency_stats& st) {
  if (count > 0) {
    const int r[3] = {nearest_rank_index(50, count), nearest_rank_index(90, count), nearest_rank_index(99, count)};
    uint64_t v[3];
    select3(keys, n, r, v);
    if (threadIdx.x == 0) {
      st.count = count;
      st.p50 = kInt ? (double)(int64_t)(v[0] ^ kSignBit) : dval(v[0]);
      st.p90 = kInt ? (double)(int64_t)(v[1] ^ kSignBit) : dval(v[1]);
      st.p99 = kInt ? (double)(int64_t)(v[2] ^ kSignBit) : dval(v[2]);
      st.mean = mean;
    }
  } else if (threadIdx.x == 0) {
    st.count = 0;
    st.p50 = st.p90 = st.p99 = st.mean = __longlong_as_double(0x7ff8000000000000LL);  // NaN: absent
  }
  __syncthreads();
}

// kGlobal: the keys live in a caller-provided global scratch (cap per CTA) instead of
// dynamic shared memory: workloads above ~28,000 requests (metrics.py has no limit)
template <bool kGlobal>
__global__ void __launch_bounds__(kMetThreads, 12) k_metrics(MetParams p) {
  extern __shared__ __align__(16) uint64_t skeys[];
  uint64_t* keys = kGlobal ? p.gkeys + (size_t)blockIdx.x * (size_t)p.cap : skeys;
  __shared__ int64_t red[7][kMetWarps];
  __shared__ tw_run_metrics res;
  __shared__ double sh_mean;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int c = blockIdx.x; c < p.n_cfg; c += gridDim.x) {
    const tw_sim_cfg cfg = p.cfgs[c];
    const int64_t wl0 = p.wl_off[cfg.workload_id];
    const int n = (int)(p.wl_off[cfg.workload_id + 1] - wl0);
    const int64_t rb = p.req_base[c];
    const int64_t epoch = cfg.epoch_ns;
    if (tid == 0) {
      memset(&res, 0, sizeof(res));
      res.num_requests = n;
    }
    int status = TW_METRICS_OK;
    if (p.sim && (p.sim[c].status & 0xff) != TW_SIM_OK) status = TW_METRICS_SIM_FAILED;
    else if (n > p.cap) status = TW_METRICS_TOO_LARGE;
    __syncthreads();
    if (status != TW_METRICS_OK) {
      if (tid == 0) {
        res.status = status;
        p.out[c] = res;
      }
      __syncthreads();
      continue;
    }
    // ---- pass 1: per-request reductions (collect_metrics, metrics.py:213-247)
    BlockRed r = {0, 0, INT64_MIN, 0, 0, 0};
    // the int64 sums stand for the reference's float sums only when every partial sum is an
    // exact float: all values in [0, (2^53 - 1) / n] (else, e.g. past 2^63 or with
    // negative values, the CPython-order float sum below)
    const uint64_t lim = (uint64_t)(((1LL << 53) - 1) / (n > 0 ? n : 1));
    int32_t big = 0;  // bit 0: a TTFT value past the bound, bit 1: an e2e value
    for (int i = tid; i < n; i += kMetThreads) {
      const int64_t fin = p.finish[rb + i], fst = p.first[rb + i];
      const int64_t off = p.ts[wl0 + i];
      const int32_t op = p.output[wl0 + i];
      if (fin < 0 || fst < 0) {
        r.miss++;
        continue;
      }
      r.tokens += op;
      const int64_t fr = fin - epoch;
      r.maxfin = fr > r.maxfin ? fr : r.maxfin;
      const int64_t a = fst - epoch - off, b = fin - epoch - off;
      r.s_ttft += a;
      r.s_e2e += b;
      big |= ((uint64_t)a > lim) | (((uint64_t)b > lim) << 1);
      r.n_tpot += op > 1;
    }
    // the flags as two counts, 20 bits apart (at most 128 per CTA)
    int64_t v[7] = {r.miss, r.tokens, r.maxfin, r.s_ttft, r.s_e2e, r.n_tpot, (big & 1) + ((int64_t)(big >> 1) << 20)};
#pragma unroll
    for (int k = 0; k < 7; k++) {
      const int64_t w = (k == 2) ? warp_max_i64(v[k]) : warp_sum_i64(v[k]);
      if (lane == 0) red[k][warp] = w;
    }
    __syncthreads();
    if (tid < 32) {
#pragma unroll
      for (int k = 0; k < 7; k++) {
        int64_t w = lane < kMetWarps ? red[k][lane] : (k == 2 ? INT64_MIN : 0);
        w = (k == 2) ? warp_max_i64(w) : warp_sum_i64(w);
        if (lane == 0) red[k][0] = w;
      }
    }
    __syncthreads();
    const int64_t miss = red[0][0], tokens = red[1][0], maxfin = red[2][0];
    const int64_t s_ttft = red[3][0], s_e2e = red[4][0];
    const int n_tpot = (int)red[5][0];
    const bool big_sum[2] = {(red[6][0] & 0xfffff) != 0, (red[6][0] >> 20) != 0};
    if (miss > 0) {  // IncompleteLog (metrics.py:236-240)
      if (tid == 0) {
        res.status = TW_METRICS_INCOMPLETE;
        res.n_missing = (int32_t)miss;
        p.out[c] = res;
      }
      __syncthreads();
      continue;
    }
    if (tid == 0) {
      res.output_tokens = tokens;
      res.virtual_elapsed_ns = n > 0 ? maxfin : 0;
      // tokens_per_virtual_s = total / (virtual_elapsed_ns / NS_PER_S) (metrics.py:113-115)
      const double vs = __ddiv_rn((double)res.virtual_elapsed_ns, 1e9);
      res.tokens_per_virtual_s = vs > 0.0 ? __ddiv_rn((double)tokens, vs) : 0.0;
    }
    double* vals = reinterpret_cast<double*>(keys);
    const int32_t* pos = p.sum_order ? p.sum_order + wl0 : nullptr;
    // ---- TTFT, e2e: exact integer sums unless they could round, then the CPython sum
    for (int m = 0; m < 2; m++) {
      const int64_t s = m == 0 ? s_ttft : s_e2e;
      const bool exact = !big_sum[m] && s >= 0 && s < (1LL << 53);
      if (!exact) {
        for (int i = tid; i < n; i += kMetThreads) {
          const int64_t t = (m == 0 ? p.first[rb + i] : p.finish[rb + i]) - epoch - p.ts[wl0 + i];
          vals[pos ? pos[i] : i] = (double)t;
        }
        __syncthreads();
        if (tid == 0) sh_mean = neumaier_sum(vals, n);
        __syncthreads();
      }
      for (int i = tid; i < n; i += kMetThreads) {
        const int64_t t = (m == 0 ? p.first[rb + i] : p.finish[rb + i]) - epoch - p.ts[wl0 + i];
        keys[i] = (uint64_t)t ^ kSignBit;  // t < INT64_MAX, so never the no-value key ~0
      }
      const double sum = exact ? (double)s : sh_mean;
      stats_from_keys<true>(keys, n, n, n > 0 ? __ddiv_rn(sum, (double)n) : 0.0, m == 0 ? res.ttft : res.e2e);
    }
    // ---- TPOT over requests with more than one output token (metrics.py:54-60, 100-101)
    double* tv = p.tpot_vals ? p.tpot_vals + (int64_t)c * p.cap : nullptr;
    for (int i = tid; i < n; i += kMetThreads) {
      const int32_t op = p.output[wl0 + i];
      double t = __longlong_as_double(0x7ff8000000000000LL);
      if (op > 1) t = __ddiv_rn((double)(p.finish[rb + i] - p.first[rb + i]), (double)(op - 1));
      vals[pos ? pos[i] : i] = t;
      if (tv) tv[pos ? pos[i] : i] = t;  // summed by k_metrics_tpot
    }
    __syncthreads();
    if (tid == 0) sh_mean = (n_tpot > 0 && !tv) ? __ddiv_rn(neumaier_sum(vals, n), (double)n_tpot) : 0.0;
    __syncthreads();
    for (int i = tid; i < n; i += kMetThreads) {
      const double t = vals[i];
      keys[i] = isnan(t) ? ~0ULL : dkey(t);
    }
    stats_from_keys<false>(keys, n, n_tpot, sh_mean, res.tpot);
    if (tid == 0) {
      res.status = TW_METRICS_OK;
      p.out[c] = res;
    }
    __syncthreads();
  }
}

}  // namespace twb

using namespace twb;

extern "C" int tw_metrics_many(const tw_sim_cfg* cfgs, int32_t n_cfg, const int64_t* wl_off,
                               const int64_t* req_offset_ns, const int32_t* req_output,
                               const int64_t* req_base, const int64_t* req_first_ns,
                               const int64_t* req_finish_ns, const tw_sim_result* sim,
                               const int32_t* sum_order, int32_t max_requests, void* scratch,
                               int64_t scratch_bytes, tw_run_metrics* out, void* stream) {
  if (n_cfg < 0 || (n_cfg > 0 && (!cfgs || !wl_off || !req_offset_ns || !req_output || !req_base ||
                                  !req_first_ns || !req_finish_ns || !out))) {
    set_error("tw_metrics_many: bad arguments");
    return TW_EINVAL;
  }
  if (max_requests < 0) {
    set_error("tw_metrics_many: max_requests %d < 0", max_requests);
    return TW_EINVAL;
  }
  if (n_cfg == 0) return TW_OK;
  int dev = 0, sms = 148, per_sm = 1, max_optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int limit = (max_optin - kMetStaticSmem) / (int)sizeof(uint64_t);
  const int cap = max_requests > 0 ? max_requests : 1;  // selection needs no power-of-two padding
  const bool global = max_requests > limit;
  int64_t grid;
  size_t smem = 0;
  // the TPOT rows (n_cfg x cap doubles) take the end of the scratch when it holds them
  const int64_t tpot_bytes = (int64_t)n_cfg * cap * (int64_t)sizeof(double);
  int64_t key_budget = scratch ? scratch_bytes : 0;
  bool tpot_ok = false;
  if (global) {
    const int64_t want = ((int64_t)std::min<int64_t>(4LL * sms, n_cfg) * cap * (int64_t)sizeof(uint64_t) + 255) & ~255LL;
    if (key_budget >= want + tpot_bytes) {
      key_budget -= tpot_bytes;
      tpot_ok = true;
    }
  } else {
    tpot_ok = key_budget >= tpot_bytes;
  }
  if (!global) {
    smem = (size_t)cap * sizeof(uint64_t);
    cudaFuncSetAttribute(k_metrics<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_metrics<false>, kMetThreads, smem);
    if (per_sm < 1) per_sm = 1;
    grid = (int64_t)sms * per_sm;
  } else {
    // keys in global scratch: one cap-sized slice per CTA, as many CTAs as the scratch holds
    const int64_t slices = key_budget / ((int64_t)cap * (int64_t)sizeof(uint64_t));
    if (slices < 1) {
      set_error("tw_metrics_many: max_requests %d above the %d requests shared memory holds and no scratch "
                "(%lld bytes; tw_metrics_scratch_bytes gives the size)", max_requests, limit,
                (long long)scratch_bytes);
      return TW_ENOSMEM;
    }
    grid = (int64_t)sms * 4;
    if (grid > slices) grid = slices;
  }
  if (grid > n_cfg) grid = n_cfg;
  MetParams p;
  p.cfgs = cfgs;
  p.n_cfg = n_cfg;
  p.wl_off = wl_off;
  p.ts = req_offset_ns;
  p.output = req_output;
  p.req_base = req_base;
  p.first = req_first_ns;
  p.finish = req_finish_ns;
  p.sim = sim;
  p.sum_order = sum_order;
  p.cap = cap;
  p.gkeys = static_cast<uint64_t*>(scratch);
  p.out = out;
  // scratch layout: [global keys (workloads above what shared memory holds)] [TPOT values]
  const int64_t keys_bytes = global ? (int64_t)grid * cap * (int64_t)sizeof(uint64_t) : 0;
  const int64_t keys_room = (keys_bytes + 255) & ~255LL;
  // lane-per-config sums pay off once each resident CTA has several configs to summarise
  // (65,536 configs: 6.84 -> 4.72 ms); with few configs the 1,000-step chains of a handful
  // of warps are slower than the in-CTA sums (1,024 configs: 0.113 -> 0.222 ms)
  p.tpot_vals = (tpot_ok && n_cfg >= 4096 && scratch_bytes >= keys_room + tpot_bytes)
                    ? reinterpret_cast<double*>(static_cast<char*>(scratch) + keys_room)
                    : nullptr;
  if (global) k_metrics<true><<<(int)grid, kMetThreads, 0, (cudaStream_t)stream>>>(p);
  else k_metrics<false><<<(int)grid, kMetThreads, smem, (cudaStream_t)stream>>>(p);
  count_launch();
  if (p.tpot_vals) {
    k_metrics_tpot<<<(n_cfg + 127) / 128, 128, 0, (cudaStream_t)stream>>>(p);
    count_launch();
  }
  return check_launch("tw_metrics_many");
}

extern "C" int64_t tw_metrics_scratch_bytes(int32_t n_cfg, int32_t max_requests) {
  int dev = 0, sms = 148, max_optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (n_cfg <= 0) return 0;
  const int cap = max_requests > 0 ? max_requests : 1;
  const int64_t tpot = (int64_t)n_cfg * cap * (int64_t)sizeof(double);  // k_metrics_tpot's rows
  if (max_requests <= (max_optin - kMetStaticSmem) / (int)sizeof(uint64_t)) return tpot;
  const int64_t ctas = n_cfg < 4 * sms ? n_cfg : 4 * sms;
  return ((ctas * (int64_t)cap * (int64_t)sizeof(uint64_t) + 255) & ~255LL) + tpot;
}
