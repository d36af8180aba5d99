// common.cuh — device helpers shared by the libtwb200 kernels (sm_100a).
//
//  * pset staging: the whole predictor blob is copied global -> shared with ONE
//    cp.async.bulk (TMA bulk-copy engine, SASS UBLKCP) completing on an mbarrier;
//  * the exact-fp64 duration predictor (reference: predictor.py:100-242) in a
//    scalar form (bulk kernel, one query per thread) and a warp-cooperative form
//    (event loop, one query per warp: ballot-based axis bracketing);
//  * int64 warp reductions.
//
// Bit-exactness contract: every fp64 op is an explicit _rn
// intrinsic (no FMA contraction possible), ints convert exactly, rounding to whole
// microseconds is half-to-even (__double2ll_rn), durations are int64 ns.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/twb200.h"

namespace twb {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;

// ------------------------------------------------------------------------------
// error / launch bookkeeping (abi.cu)
// ------------------------------------------------------------------------------
void set_error(const char* fmt, ...);
int check_launch(const char* what);
void count_launch();

// ------------------------------------------------------------------------------
// TMA bulk copy of the predictor blob into shared memory
// ------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Copies `bytes` (multiple of 16, both addresses 16-B aligned) from global `src` to
// shared `dst` using the bulk-copy (TMA) engine. Must be called by ALL threads of
// the CTA; thread 0 issues, everyone waits on the mbarrier's phase 0.
__device__ __forceinline__ void tma_stage_to_smem(void* dst, const void* src, uint32_t bytes,
                                                  uint64_t* mbar) {
  const uint32_t bar = smem_u32(mbar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
    // chunks of <= 64 KiB keep each transfer well inside the tx-count range
    uint32_t off = 0;
    while (off < bytes) {
      uint32_t n = bytes - off;
      if (n > 65536u) n = 65536u;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(static_cast<char*>(dst) + off)),
          "l"(static_cast<const char*>(src) + off), "r"(n), "r"(bar)
          : "memory");
      off += n;
    }
  }
  __syncthreads();
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(bar)
        : "memory");
  }
}

// ------------------------------------------------------------------------------
// predictor blob views
// ------------------------------------------------------------------------------
struct TableView {
  const int32_t* pax;
  const int32_t* dax;
  const int64_t* grid;
  const double* rp;  // RN(1 / (pax[k+1] - pax[k]))
  const double* rd;  // RN(1 / (dax[k+1] - dax[k]))
  const int16_t* lutp;  // bit-length LUTs (twb200.h table layout)
  const int16_t* lutd;
  const int32_t* grid32;  // int32 copy of the grid, or null
  int np, nd;
};

__device__ __forceinline__ const tw_pred_desc* pset_desc(const char* pset, int id) {
  return reinterpret_cast<const tw_pred_desc*>(pset + sizeof(tw_pset_header)) + id;
}
__device__ __forceinline__ int pset_ndesc(const char* pset) {
  return reinterpret_cast<const tw_pset_header*>(pset)->n_desc;
}
__device__ __forceinline__ TableView table_view(const char* pset, const tw_pred_desc* d) {
  TableView t;
  const char* base = pset + d->table_off;
  t.pax = reinterpret_cast<const int32_t*>(base);
  t.dax = t.pax + d->np;
  uint32_t goff = (uint32_t)(d->np + d->nd) * 4u;
  goff = (goff + 7u) & ~7u;
  t.grid = reinterpret_cast<const int64_t*>(base + goff);
  t.rp = reinterpret_cast<const double*>(t.grid + d->np * d->nd);
  t.rd = t.rp + d->np;
  t.lutp = reinterpret_cast<const int16_t*>(t.rd + d->nd);
  t.lutd = t.lutp + 68;
  t.grid32 = d->pad ? reinterpret_cast<const int32_t*>(t.lutp + 136) : nullptr;
  t.np = d->np;
  t.nd = d->nd;
  return t;
}

// Python round(float) -> int (half to even), then us -> ns.
__device__ __forceinline__ int64_t us_to_ns_rn(double us) { return __double2ll_rn(us) * 1000; }

// LinearPredictor.predict's quantisation (predictor.py:142-146): int(round(us)), a
// negative result raises NegativeDuration, then * 1000. round() itself raises for NaN
// (ValueError) and +-inf (OverflowError); a finite result beyond int64 ns is the engine's
// limit (TW_PRED_OVERFLOW) instead of the reference's unbounded Python int.
__device__ __forceinline__ int64_t linear_us_to_ns(double us) {
  if (us != us) return TW_PRED_NAN;
  if (__dadd_rn(us, -us) != 0.0) return TW_PRED_OVERFLOW;  // +-inf (inf - inf = nan)
  if (us < -0.5) return TW_PRED_NEGATIVE;                  // round(us) < 0 (half-even: -0.5 -> 0)
  if (us >= 9223372036854775807.0) return TW_PRED_OVERFLOW;
  const int64_t q = __double2ll_rn(us);
  return q > INT64_MAX / 1000 ? (int64_t)TW_PRED_OVERFLOW : q * 1000;
}

// Correctly rounded a / b for an integer-valued b > 0 given rb = RN(1/b): a first
// quotient RN(a*rb) within 2 ulps, then two FMA residual corrections (Markstein: with a
// correctly rounded reciprocal, q + (a - b q) rb rounded once is RN(a/b) once q is
// faithful). a / b is never a rounding midpoint here (a is a double, b an integer, so
// the exact quotient is either representable or not dyadic), so the result equals
// __ddiv_rn(a, b) bit for bit; tw_selftest_division checks it on device.
__device__ __forceinline__ double div_rn_rcp(double a, double b, double rb) {
  double q = __dmul_rn(a, rb);
#ifndef TWB_NO_POW2_RCP
  // RN(1/b) is a power of two only for b = 2^k (b an integer < 2^52): then a * rb is the
  // exact quotient and the corrections are no-ops (calibration axes are mostly 2^k gaps)
  if ((__double_as_longlong(rb) & 0xFFFFFFFFFFFFFLL) == 0) return q;
#endif
  double r = __fma_rn(-q, b, a);
  q = __fma_rn(r, rb, q);
  r = __fma_rn(-q, b, a);
  return __fma_rn(r, rb, q);
}

// lerp with exact-int operands: Python evaluates (b-a)*(x-lo) exactly and the
// int/int true division correctly rounded; equal to one correctly rounded fp64
// division while |num| < 2^53 (the host rejects tables that could exceed it).
__device__ __forceinline__ double lerp_int(int64_t a, int64_t b, int64_t lo, int64_t hi, int64_t x, double rgap) {
  const int64_t num = (b - a) * (x - lo);
  const double q = div_rn_rcp(__ll2double_rn(num), __ll2double_rn(hi - lo), rgap);
  return __dadd_rn(__ll2double_rn(a), q);
}
__device__ __forceinline__ double lerp_dbl(double a, double b, int64_t lo, int64_t hi, int64_t x, double rgap) {
  const double diff = __dsub_rn(b, a);
  const double prod = __dmul_rn(diff, __ll2double_rn(x - lo));
  return __dadd_rn(a, div_rn_rcp(prod, __ll2double_rn(hi - lo), rgap));
}

// Bilinear evaluation once both axes are bracketed (indices into the axes).
// Returns TW_PRED_TABLE_MISS (as a sentinel) when a corner is a hole.
__device__ __forceinline__ int64_t table_corners(const TableView& t, int p0, int p1, int d0, int d1,
                                                 int64_t P, int64_t D) {
  const int64_t c00 = t.grid[p0 * t.nd + d0];
  const int64_t c10 = t.grid[p1 * t.nd + d0];
  const int64_t c01 = t.grid[p0 * t.nd + d1];
  const int64_t c11 = t.grid[p1 * t.nd + d1];
  if (c00 == TW_TABLE_HOLE || c10 == TW_TABLE_HOLE || c01 == TW_TABLE_HOLE || c11 == TW_TABLE_HOLE)
    return TW_PRED_TABLE_MISS;
  const int64_t P0 = t.pax[p0], P1 = t.pax[p1], D0 = t.dax[d0], D1 = t.dax[d1];
  double us;
  if (P1 == P0) {
    // level-1 lerps return the int corners (predictor.py:229-230); an exact hit
    // (predictor.py:213-215) is the P1==P0, D1==D0 case
    us = (D1 == D0) ? __ll2double_rn(c00) : lerp_int(c00, c01, D0, D1, D, t.rd[d0]);
  } else {
    const double rp = t.rp[p0];
    const double at_d0 = lerp_int(c00, c10, P0, P1, P, rp);
    const double at_d1 = lerp_int(c01, c11, P0, P1, P, rp);
    us = (D1 == D0) ? at_d0 : lerp_dbl(at_d0, at_d1, D0, D1, D, t.rd[d0]);
  }
  return us_to_ns_rn(us);
}

// scalar bracket: lo = index of max axis <= v, hi = index of min axis >= v.
// Branchless binary search: power-of-two steps from the largest below n.
__device__ __forceinline__ bool bracket_scalar(const int32_t* axis, int n, int64_t v, int& lo, int& hi) {
  if (v < axis[0] || v > axis[n - 1]) return false;
  int pos = 0;
  int32_t at = axis[0];
  for (int step = (n > 1) ? (1 << (31 - __clz(n - 1))) : 0; step > 0; step >>= 1) {
    const int cand = pos + step;
    if (cand < n) {
      const int32_t a = axis[cand];
      if ((int64_t)a <= v) {
        pos = cand;
        at = a;
      }
    }
  }
  lo = pos;
  hi = ((int64_t)at == v) ? pos : pos + 1;
  return true;
}

// bracket through the bit-length LUT: the floor index lies in [lut[b][0], lut[b][1]]
// with b = bitlen(v - axis[0]); power-of-two-like axes need no search step at all.
__device__ __forceinline__ bool bracket_lut(const int32_t* axis, const int16_t* lut, int n, int64_t v, int& lo,
                                            int& hi, int64_t& vlo, int64_t& vhi) {
  const int64_t a0 = axis[0];
  if (v < a0 || v > (int64_t)axis[n - 1]) return false;
  const uint32_t x = (uint32_t)(v - a0);
  const int b = 32 - __clz(x);
  const uint32_t pr = *reinterpret_cast<const uint32_t*>(lut + 2 * b);  // (lo, hi) pair
  int i = (int16_t)(pr & 0xffff), j = (int16_t)(pr >> 16);
  while (i < j) {
    const int m = (i + j + 1) >> 1;
    if ((int64_t)axis[m] <= v) i = m; else j = m - 1;
  }
  lo = i;
  vlo = axis[i];
  if (vlo == v) {
    hi = i;
    vhi = vlo;
  } else {
    hi = i + 1;
    vhi = axis[i + 1];
  }
  return true;
}

// 32-bit variant for the bulk path (features are int32 there)
__device__ __forceinline__ bool bracket_lut32(const int32_t* axis, const int16_t* lut, int n, int32_t v, int& lo,
                                              int& hi, int32_t& vlo, int32_t& vhi) {
  const int32_t a0 = axis[0];
  if (v < a0 || v > axis[n - 1]) return false;
  const int b = 32 - __clz((uint32_t)(v - a0));
  const uint32_t pr = *reinterpret_cast<const uint32_t*>(lut + 2 * b);
  int i = (int16_t)(pr & 0xffff), j = (int16_t)(pr >> 16);
  while (i < j) {
    const int m = (i + j + 1) >> 1;
    if (axis[m] <= v) i = m; else j = m - 1;
  }
  lo = i;
  vlo = axis[i];
  if (vlo == v) {
    hi = i;
    vhi = vlo;
  } else {
    hi = i + 1;
    vhi = axis[i + 1];
  }
  return true;
}

// int32-grid bilinear evaluation for the bulk path: 4-byte corner gathers; the int
// lerp numerators are one 32x32->64 multiply each (values and axes are int32)
__device__ __forceinline__ int64_t table_corners32(const TableView& t, int p0, int p1, int d0, int d1, int32_t P0,
                                                   int32_t P1, int32_t D0, int32_t D1, int32_t P, int32_t D) {
  const int32_t c00 = t.grid32[p0 * t.nd + d0];
  const int32_t c10 = t.grid32[p1 * t.nd + d0];
  const int32_t c01 = t.grid32[p0 * t.nd + d1];
  const int32_t c11 = t.grid32[p1 * t.nd + d1];
  if ((c00 | c10 | c01 | c11) < 0) return TW_PRED_TABLE_MISS;  // holes are the only negatives
  double us;
  if (P1 == P0) {
    if (D1 == D0) {
      us = (double)c00;
    } else {
      const int64_t num = (int64_t)(c01 - c00) * (int64_t)(D - D0);
#ifndef TWB_RCP_FROM_BLOB
      const double gd = (double)(D1 - D0);
      us = __dadd_rn((double)c00, div_rn_rcp(__ll2double_rn(num), gd, __drcp_rn(gd)));
#else
      us = __dadd_rn((double)c00, div_rn_rcp(__ll2double_rn(num), (double)(D1 - D0), t.rd[d0]));
#endif
    }
  } else {
#ifndef TWB_RCP_FROM_BLOB
    const double gp = (double)(P1 - P0), rp = __drcp_rn(gp);
#else
    const double rp = t.rp[p0], gp = (double)(P1 - P0);
#endif
    const int64_t n0 = (int64_t)(c10 - c00) * (int64_t)(P - P0);
    const int64_t n1 = (int64_t)(c11 - c01) * (int64_t)(P - P0);
    const double at_d0 = __dadd_rn((double)c00, div_rn_rcp(__ll2double_rn(n0), gp, rp));
    const double at_d1 = __dadd_rn((double)c01, div_rn_rcp(__ll2double_rn(n1), gp, rp));
    if (D1 == D0) {
      us = at_d0;
    } else {
      const double prod = __dmul_rn(__dsub_rn(at_d1, at_d0), (double)(D - D0));
#ifndef TWB_RCP_FROM_BLOB
      const double gd = (double)(D1 - D0);
      us = __dadd_rn(at_d0, div_rn_rcp(prod, gd, __drcp_rn(gd)));
#else
      us = __dadd_rn(at_d0, div_rn_rcp(prod, (double)(D1 - D0), t.rd[d0]));
#endif
    }
  }
  return us_to_ns_rn(us);
}

// bilinear evaluation from bracket indices and their axis values (int64 grid: values may
// be negative, holes are TW_TABLE_HOLE)
__device__ __forceinline__ int64_t table_corners2(const TableView& t, int p0, int p1, int d0, int d1, int64_t P0,
                                                  int64_t P1, int64_t D0, int64_t D1, int64_t P, int64_t D) {
  const int64_t c00 = t.grid[p0 * t.nd + d0];
  const int64_t c10 = t.grid[p1 * t.nd + d0];
  const int64_t c01 = t.grid[p0 * t.nd + d1];
  const int64_t c11 = t.grid[p1 * t.nd + d1];
  if (c00 == TW_TABLE_HOLE || c10 == TW_TABLE_HOLE || c01 == TW_TABLE_HOLE || c11 == TW_TABLE_HOLE)
    return TW_PRED_TABLE_MISS;
  double us;
  if (P1 == P0) {
    us = (D1 == D0) ? __ll2double_rn(c00) : lerp_int(c00, c01, D0, D1, D, t.rd[d0]);
  } else {
    const double rp = t.rp[p0];
    const double at_d0 = lerp_int(c00, c10, P0, P1, P, rp);
    const double at_d1 = lerp_int(c01, c11, P0, P1, P, rp);
    us = (D1 == D0) ? at_d0 : lerp_dbl(at_d0, at_d1, D0, D1, D, t.rd[d0]);
  }
  return us_to_ns_rn(us);
}

__device__ __forceinline__ uint2 lds_u2(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ int4 lds_i4(uint32_t a) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}

// Exact RN(a / g) for an integer gap g > 0: a power-of-two gap scales exactly (a is an
// integer or a product of magnitude >= 1, so no underflow); any other gap takes the
// reciprocal division (div_rn_rcp, == __ddiv_rn).
__device__ __forceinline__ double div_gap(double a, int32_t g) {
  if ((g & (g - 1)) == 0) {
    const int k = __ffs(g) - 1;
    return __dmul_rn(a, __hiloint2double((1023 - k) << 20, 0));
  }
  const double gd = (double)g;
  return div_rn_rcp(a, gd, __drcp_rn(gd));
}

// One query through the bulk-lookup section (twb200.h): one 8-byte descriptor header,
// one 16-byte axis record per axis (shared by every table on the same axis, so lanes
// on different tables mostly hit the same records), one 16-byte corner quad; exact
// fp64 lerps in the reference's order (predictor.py:209-236). Returns false when the
// section cannot answer (non-table kinds, int64-grid tables, straddling buckets,
// out-of-range keys, holes): the caller then takes the generic path. With kShared, ps
// is the blob staged in shared memory (32-bit ld.shared addressing); otherwise ps is the
// blob in global memory, read through the read-only path. Either way the section must
// be present (the blob's full total_bytes).
template <bool kShared = true>
__device__ __forceinline__ int4 pset_unit16(const char* ps, uint32_t base, uint32_t unit) {
  if constexpr (kShared) return lds_i4(base + 16u * unit);
  else return __ldg(reinterpret_cast<const int4*>(ps) + unit);
}
template <bool kShared = true>
__device__ __forceinline__ bool predict_fast(const char* ps, const uint2* qh, int n_desc, int32_t p, int32_t d,
                                             int32_t id, int64_t& out) {
  if ((unsigned)id < (unsigned)n_desc && (p | d) >= 0) {
    uint2 h;
    if constexpr (kShared) h = lds_u2(smem_u32(qh) + 8u * (uint32_t)id);
    else h = __ldg(qh + id);
    if (h.y & TW_QHDR_FAST) {
      // records and quads are 16-byte units of the blob
      const uint32_t base = kShared ? smem_u32(ps) : 0u;
      const int4 rp = pset_unit16<kShared>(ps, base, (h.x >> 16) + (32u - __clz(p)));
      const int4 rd = pset_unit16<kShared>(ps, base, (h.y & 0xffffu) + (32u - __clz(d)));
      if ((rp.z | rd.z) >= 0 && p >= rp.x && p <= rp.y && d >= rd.x && d <= rd.y) {
        const int nd = (int)((h.y >> 16) & 0x7fffu);
        const int4 q = pset_unit16<kShared>(ps, base, (h.x & 0xffffu) + (uint32_t)(rp.z * nd + rd.z));
        const bool pex = p == rp.x, dex = d == rd.x;
        const int32_t c00 = q.x;
        const int32_t c10 = pex ? c00 : q.y;
        const int32_t c01 = dex ? c00 : q.z;
        const int32_t c11 = pex ? c01 : (dex ? c10 : q.w);
        if ((c00 | c10 | c01 | c11) >= 0) {  // holes are the only negative entries
          double us;
          if (pex) {
            us = dex ? (double)c00
                     : __dadd_rn((double)c00, div_gap(__ll2double_rn((int64_t)(c01 - c00) * (d - rd.x)), rd.y - rd.x));
          } else {
            const int32_t gp = rp.y - rp.x, xp = p - rp.x;
            const double a0 = __dadd_rn((double)c00, div_gap(__ll2double_rn((int64_t)(c10 - c00) * xp), gp));
            if (dex) {
              us = a0;
            } else {
              const double a1 = __dadd_rn((double)c01, div_gap(__ll2double_rn((int64_t)(c11 - c01) * xp), gp));
              us = __dadd_rn(a0, div_gap(__dmul_rn(__dsub_rn(a1, a0), (double)(d - rd.x)), rd.y - rd.x));
            }
          }
          out = __double2ll_rn(us) * 1000;
          return true;
        }
      }
    }
  }
  return false;
}

__device__ __forceinline__ const uint2* pset_qhdr(const char* ps) {
  return reinterpret_cast<const uint2*>(ps + reinterpret_cast<const tw_pset_header*>(ps)->fast_off);
}

// manhattan-nearest row, ties -> smallest (p, d) (predictor.py:205-207); scalar
__device__ __forceinline__ int64_t table_nearest_scalar(const TableView& t, int64_t P, int64_t D) {
  int64_t best = INT64_MAX, bv = 0;
  for (int i = 0; i < t.np; i++) {
    const int64_t dp = llabs((int64_t)t.pax[i] - P);
    if (dp > best) continue;  // rows further in p alone cannot win (p ascending)
    for (int j = 0; j < t.nd; j++) {
      const int64_t v = t.grid[i * t.nd + j];
      if (v == TW_TABLE_HOLE) continue;
      const int64_t dist = dp + llabs((int64_t)t.dax[j] - D);
      if (dist < best) {  // strict: first in (p, d) order wins ties
        best = dist;
        bv = v;
      }
    }
  }
  return bv * 1000;
}

// One prediction, scalar (bulk kernel). Not for empty batches.
__device__ __forceinline__ int64_t predict_scalar(const char* pset, int id, int64_t P, int64_t D,
                                                  int64_t C) {
  if (id < 0 || id >= pset_ndesc(pset)) return TW_PRED_BAD_DESC;
  const tw_pred_desc* d = pset_desc(pset, id);
  if (d->kind == TW_PRED_CONSTANT) return d->constant_us * 1000;
  if (d->kind == TW_PRED_LINEAR) {
    double us = __dadd_rn(d->base_us, __dmul_rn(d->per_prefill_token_us, __ll2double_rn(P)));
    us = __dadd_rn(us, __dmul_rn(d->per_decode_us, __ll2double_rn(D)));
    us = __dadd_rn(us, __dmul_rn(d->per_context_token_us, __ll2double_rn(C)));
    return linear_us_to_ns(us);
  }
  if (d->kind != TW_PRED_TABLE) return TW_PRED_BAD_DESC;
  const TableView t = table_view(pset, d);
  int p0, p1, d0, d1;
  int64_t P0, P1, D0, D1;
  if (bracket_lut(t.pax, t.lutp, t.np, P, p0, p1, P0, P1) && bracket_lut(t.dax, t.lutd, t.nd, D, d0, d1, D0, D1)) {
    const int64_t r = table_corners2(t, p0, p1, d0, d1, P0, P1, D0, D1, P, D);
    if (r != TW_PRED_TABLE_MISS) return r;
  }
  if (d->allow_extrapolation) return table_nearest_scalar(t, P, D);
  return TW_PRED_TABLE_MISS;
}

// One prediction for the bulk kernel: int32 P and D (the features API), table path
// first. Same results as predict_scalar.
__device__ __forceinline__ int64_t predict_bulk(const char* pset, int n_desc, int id, int32_t P, int32_t D,
                                                int64_t C) {
  if ((unsigned)id >= (unsigned)n_desc) return TW_PRED_BAD_DESC;
  const tw_pred_desc* d = pset_desc(pset, id);
  const int kind = d->kind;
  if (kind == TW_PRED_TABLE) {
    const TableView t = table_view(pset, d);
    int p0, p1, d0, d1;
    int32_t P0, P1, D0, D1;
    if (bracket_lut32(t.pax, t.lutp, t.np, P, p0, p1, P0, P1) &&
        bracket_lut32(t.dax, t.lutd, t.nd, D, d0, d1, D0, D1)) {
      const int64_t r = t.grid32 ? table_corners32(t, p0, p1, d0, d1, P0, P1, D0, D1, P, D)
                                 : table_corners2(t, p0, p1, d0, d1, P0, P1, D0, D1, P, D);
      if (r != TW_PRED_TABLE_MISS) return r;
    }
    if (d->allow_extrapolation) return table_nearest_scalar(t, P, D);
    return TW_PRED_TABLE_MISS;
  }
  return predict_scalar(pset, id, P, D, C);
}

// ------------------------------------------------------------------------------
// warp-cooperative prediction (event loop): all lanes get the same answer
// ------------------------------------------------------------------------------
__device__ __forceinline__ int64_t warp_min_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t w = __shfl_xor_sync(kFull, v, o);
    v = w < v ? w : v;
  }
  return v;
}
__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// lo/hi bracket with lanes comparing 32 axis entries at a time (one LDS + ballot).
__device__ __forceinline__ bool bracket_warp(const int32_t* axis, int n, int64_t v, int& lo, int& hi) {
  const int lane = threadIdx.x & 31;
  if (v < axis[0] || v > axis[n - 1]) return false;
  int cnt_le = 0;  // number of axis entries <= v  (axis sorted ascending)
  bool eq = false;
  for (int b = 0; b < n; b += 32) {
    const int i = b + lane;
    const int64_t a = (i < n) ? (int64_t)axis[i] : INT64_MAX;
    cnt_le += __popc(__ballot_sync(kFull, a <= v));
    eq |= __any_sync(kFull, a == v);
    if (b + 32 < n && (int64_t)axis[b + 31] > v) break;
  }
  lo = cnt_le - 1;
  hi = eq ? lo : lo + 1;
  return true;
}

__device__ __forceinline__ int64_t table_nearest_warp(const TableView& t, int64_t P, int64_t D) {
  const int lane = threadIdx.x & 31;
  // each lane scans cells lane, lane+32, ...; key = (dist, p-index, d-index) which is
  // the reference's (dist, (p, d)) order because the axes are sorted ascending
  int64_t best = INT64_MAX, bkey = INT64_MAX, bv = 0;
  const int cells = t.np * t.nd;
  for (int c = lane; c < cells; c += 32) {
    const int64_t v = t.grid[c];
    if (v == TW_TABLE_HOLE) continue;
    const int i = c / t.nd, j = c - i * t.nd;
    const int64_t dist = llabs((int64_t)t.pax[i] - P) + llabs((int64_t)t.dax[j] - D);
    if (dist < best || (dist == best && c < bkey)) {
      best = dist;
      bkey = c;
      bv = v;
    }
  }
  const int64_t mind = warp_min_i64(best);
  const int64_t k = warp_min_i64(best == mind ? bkey : INT64_MAX);
  const unsigned who = __ballot_sync(kFull, best == mind && bkey == k);
  return __shfl_sync(kFull, bv, __ffs(who) - 1) * 1000;
}

// Warp-uniform prediction for a non-empty batch; every lane must call.
__device__ __forceinline__ int64_t predict_warp(const char* pset, int id, int64_t P, int64_t D,
                                                int64_t C) {
  if (id < 0 || id >= pset_ndesc(pset)) return TW_PRED_BAD_DESC;
  const tw_pred_desc* d = pset_desc(pset, id);
  if (d->kind != TW_PRED_TABLE) return predict_scalar(pset, id, P, D, C);
  const TableView t = table_view(pset, d);
  int p0, p1, d0, d1;
  if (bracket_warp(t.pax, t.np, P, p0, p1) && bracket_warp(t.dax, t.nd, D, d0, d1)) {
    const int64_t r = table_corners(t, p0, p1, d0, d1, P, D);
    if (r != TW_PRED_TABLE_MISS) return r;
  }
  if (d->allow_extrapolation) return table_nearest_warp(t, P, D);
  return TW_PRED_TABLE_MISS;
}

// FakeClock.sleep(wait_ns / 1e9) -> int(round(seconds * 1e9)) (pkg/tests/_support.py:33-34)
__device__ __forceinline__ int64_t fake_sleep_ns(int64_t wait_ns) {
  const double seconds = __ddiv_rn(__ll2double_rn(wait_ns), 1e9);
  return __double2ll_rn(__dmul_rn(seconds, 1e9));
}

}  // namespace twb
