// predict.cu — bulk duration predictor (north-star kernels 1 and 2).
//
//   tw_predict_features : (P, D, C, desc_id) -> int64 ns        28 B / prediction
//   tw_predict_batches  : CSR slots -> features -> int64 ns     8 B/slot + 20 B/batch
//
// Reference: predictor.py:64-84 (features), 100-242 (predict). HBM-bound gather
// work: the predictor blob (descriptors + calibration tables, a few KB) is staged
// once per CTA into shared memory by one TMA bulk copy; the query streams are read
// with 16-byte vector loads marked evict-first, each thread handling 4 queries per
// iteration for memory-level parallelism; grid = one 1024-thread CTA per SM (A/B on
// B200: 1024x1 > 640x2 > 512x2 > 256x3; profiles/README.md).
#include <atomic>
#include <cstring>
#include <ctime>

#include "common.cuh"

namespace twb {

#ifndef TWB_PRED_THREADS
#define TWB_PRED_THREADS 1024
#endif
constexpr int kPredThreads = TWB_PRED_THREADS;

struct PsetSmem {
  static __device__ __forceinline__ char* stage(const void* pset, uint32_t bytes) {
    extern __shared__ __align__(128) char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    char* blob = smem + 128;
    tma_stage_to_smem(blob, pset, bytes, bar);
    return blob;
  }
};

// Everything the bulk-lookup section cannot answer (non-table kinds, int64 grids,
// ambiguous axis buckets, out-of-range keys, holes): the generic predictor, kept out
// of line so the common path stays short.
static __device__ __noinline__ int64_t predict_generic(const char* ps, int n_desc, int32_t id, int32_t p, int32_t d,
                                                int64_t c) {
  return predict_bulk(ps, n_desc, id, p, d, c);
}

// One query through the bulk-lookup section (twb200.h): one 8-byte descriptor header,
// one 16-byte axis record per axis (shared by every table on the same axis, so lanes
// on different tables mostly hit the same records), one 16-byte corner quad; exact
// fp64 lerps in the reference's order (predictor.py:209-236).
template <bool kShared = true>
__device__ __forceinline__ int64_t predict_one(const char* ps, const uint2* qh, int n_desc, int32_t p, int32_t d,
                                               int64_t c, int32_t id) {
  if ((p | d) == 0 && c < 0) return TW_PRED_EMPTY_BATCH;  // "no slots" marker
  int64_t r;
  if (predict_fast<kShared>(ps, qh, n_desc, p, d, id, r)) return r;
  return predict_generic(ps, n_desc, id, p, d, c);
}


#ifndef TWB_PRED_MIN_BLOCKS
#define TWB_PRED_MIN_BLOCKS 1
#endif
// kShared = false: a blob too large for shared memory, read through L1 instead
template <bool kShared>
__global__ void __launch_bounds__(kPredThreads, TWB_PRED_MIN_BLOCKS) k_predict_features(
    const void* __restrict__ pset, uint32_t pset_bytes, const int32_t* __restrict__ P,
    const int32_t* __restrict__ D, const int64_t* __restrict__ C, const int32_t* __restrict__ id,
    int64_t n, int64_t* __restrict__ out) {
  const char* ps = kShared ? PsetSmem::stage(pset, pset_bytes) : static_cast<const char*>(pset);
  const int n_desc = pset_ndesc(ps);
  const uint2* qh = pset_qhdr(ps);
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // vector body: groups of 4 consecutive queries (all arrays 16-B aligned by contract)
  const int64_t n4 = n >> 2;
  for (int64_t g = tid; g < n4; g += nthreads) {
    const int4 p4 = __ldcs(reinterpret_cast<const int4*>(P) + g);
    const int4 d4 = __ldcs(reinterpret_cast<const int4*>(D) + g);
    const int4 i4 = __ldcs(reinterpret_cast<const int4*>(id) + g);
    const longlong2 c01 = __ldcs(reinterpret_cast<const longlong2*>(C) + 2 * g);
    const longlong2 c23 = __ldcs(reinterpret_cast<const longlong2*>(C) + 2 * g + 1);
    longlong2 o01, o23;
    o01.x = predict_one<kShared>(ps, qh, n_desc, p4.x, d4.x, c01.x, i4.x);
    o01.y = predict_one<kShared>(ps, qh, n_desc, p4.y, d4.y, c01.y, i4.y);
    o23.x = predict_one<kShared>(ps, qh, n_desc, p4.z, d4.z, c23.x, i4.z);
    o23.y = predict_one<kShared>(ps, qh, n_desc, p4.w, d4.w, c23.y, i4.w);
    __stcs(reinterpret_cast<longlong2*>(out) + 2 * g, o01);
    __stcs(reinterpret_cast<longlong2*>(out) + 2 * g + 1, o23);
  }
  for (int64_t i = (n4 << 2) + tid; i < n; i += nthreads)
    out[i] = predict_one<kShared>(ps, qh, n_desc, P[i], D[i], C[i], id[i]);
}

// Fused batch-feature extraction + prediction (north-star kernels 1 + 2) over CSR batches.
//
// Warp-specialised TMA pipeline, one 1024-thread CTA per SM:
//  * warp 31 is the producer: for each tile of 992 batches it reads the tile's slot
//    range from batch_off and moves the contiguous slot_tok / slot_ctx runs into a
//    shared-memory stage with two cp.async.bulk copies (TMA bulk-copy engine) that
//    complete on the stage's "full" mbarrier (slot_ctx only when a model or the
//    features output needs total_context); it reuses a stage once all consumer warps
//    have arrived on its "empty" mbarrier (4 stages of tok + ctx or 8 of tok in flight);
//  * warps 0-30 consume: each thread owns one batch per tile, prefetches its
//    offsets and descriptor id for the next tile while the current one is reduced,
//    sums its slots from shared memory (predictor.py:69-84) and predicts through the
//    bulk-lookup section.
// So every HBM read of the CSR arrays is a bulk transfer or a coalesced row of
// offsets, and no CTA-wide barrier sits in the loop. A tile whose slots exceed a
// stage is flagged and its consumers load slots directly.
constexpr int kExtThreads = 1024;
#ifndef TWB_EXT_BPT
#define TWB_EXT_BPT 1
#endif
constexpr int kExtBpt = TWB_EXT_BPT;                        // batches per consumer thread per tile
constexpr int kExtConsumers = (kExtThreads - 32) * kExtBpt;  // batches per tile
// Stages in flight: 4 when the context slots travel too (tok + ctx, 8 B per slot), 8 when
// only the tokens do (4 B per slot): the same shared memory then holds twice as many tiles
// ahead of the consumers.
#ifndef TWB_EXT_STAGES_C
#define TWB_EXT_STAGES_C 4
#endif
#ifndef TWB_EXT_STAGES_T
#define TWB_EXT_STAGES_T 8
#endif
constexpr int kExtMaxStages = 8;
static_assert(TWB_EXT_STAGES_C <= kExtMaxStages && TWB_EXT_STAGES_T <= kExtMaxStages, "stages");

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

struct ExtTile {
  int64_t a0;      // first staged slot (tile's first slot rounded down to 4)
  int32_t staged;  // 1: slots in shared memory, 0: direct loads
  int32_t pad;
};

template <bool kShared>
__global__ void __launch_bounds__(kExtThreads, 1) k_predict_batches(
    const void* __restrict__ pset, uint32_t pset_bytes, uint32_t pset_smem, int32_t region,
    const int64_t* __restrict__ off, const int32_t* __restrict__ tok, const int32_t* __restrict__ ctx,
    const int32_t* __restrict__ id, int64_t nb, int64_t* __restrict__ feat, int64_t* __restrict__ out) {
  extern __shared__ __align__(128) char smem[];
  // the blob staged in shared memory (ends with a CTA barrier), or read through L1
  const char* ps = kShared ? PsetSmem::stage(pset, pset_bytes) : static_cast<const char*>(pset);
  const int n_desc = pset_ndesc(ps);
  const uint2* qh = pset_qhdr(ps);
  char* area = smem + 128 + pset_smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(area);  // full[kExtMaxStages], empty[kExtMaxStages]
  ExtTile* meta = reinterpret_cast<ExtTile*>(area + 16 * kExtMaxStages);
  int32_t* slots = reinterpret_cast<int32_t*>(area + 32 * kExtMaxStages);  // stage s: tok, then ctx if any_c
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (nb + kExtConsumers - 1) / kExtConsumers;
  // total_context feeds only Linear models with a context term (predictor.py:137-142) and
  // the features output: when neither occurs, slot_ctx is neither copied nor summed
  bool set_c = false;
  for (int i = lane; i < n_desc; i += 32) {
    const tw_pred_desc* dsc = pset_desc(ps, i);
    set_c |= dsc->kind == TW_PRED_LINEAR && dsc->per_context_token_us != 0.0;
  }
  const bool any_c = feat != nullptr || __any_sync(kFull, set_c);
  const int nst = any_c ? TWB_EXT_STAGES_C : TWB_EXT_STAGES_T;
  const int32_t cap = (region / (nst * (any_c ? 8 : 4))) & ~3;  // slots per stage
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; s++) {
      mbar_init(smem_u32(&bars[s]), 1);                                   // full: producer + tx bytes
      mbar_init(smem_u32(&bars[kExtMaxStages + s]), kExtThreads / 32 - 1);  // empty: one per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kExtThreads / 32 - 1) {  // ---------------- producer warp
    int k = 0;
    int64_t w0 = 0, w1 = 0;  // lane i: slot range of this CTA's tile k + i (window of 32 tiles)
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, k++) {
      const int s = k % nst;
      if ((k & 31) == 0) {  // prefetch the next 32 tiles' slot ranges, one per lane
        const int64_t tt = t + (int64_t)lane * gridDim.x;
        if (tt < ntiles) {
          const int64_t b0 = tt * kExtConsumers;
          w0 = __ldg(off + b0);
          w1 = __ldg(off + min(b0 + kExtConsumers, nb));
        }
      }
      const int64_t s0 = __shfl_sync(kFull, w0, k & 31), s1 = __shfl_sync(kFull, w1, k & 31);
      if (k >= nst) mbar_wait(smem_u32(&bars[kExtMaxStages + s]), ((k / nst) - 1) & 1);
      if (lane == 0) {
        const int64_t a0 = s0 & ~3LL, n = ((s1 + 3) & ~3LL) - a0;  // readable to a multiple of 4 (twb200.h)
        const uint32_t full = smem_u32(&bars[s]);
        meta[s].a0 = a0;
        meta[s].staged = n <= cap;
        if (n <= cap && n > 0) {
          const uint32_t bytes = (uint32_t)(n * 4);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(full),
                       "r"(any_c ? 2 * bytes : bytes)
                       : "memory");
          if (any_c) {
            bulk_g2s(slots + (size_t)(2 * s) * cap, tok + a0, bytes, full);
            bulk_g2s(slots + (size_t)(2 * s + 1) * cap, ctx + a0, bytes, full);
          } else {
            bulk_g2s(slots + (size_t)s * cap, tok + a0, bytes, full);
          }
        } else {
          mbar_arrive(full);
        }
      }
      __syncwarp();
    }
    return;
  }

  // ---------------------------------------------------------------- consumer warps
  constexpr int kC = kExtThreads - 32;
  int64_t t = blockIdx.x;
  int64_t s0[kExtBpt], s1[kExtBpt];
  int32_t ib[kExtBpt];
#pragma unroll
  for (int j = 0; j < kExtBpt; j++) {
    const int64_t b = t * kExtConsumers + j * kC + threadIdx.x;
    s0[j] = s1[j] = 0;
    ib[j] = 0;
    if (t < ntiles && b < nb) {
      s0[j] = __ldg(off + b);
      s1[j] = __ldg(off + b + 1);
      ib[j] = __ldg(id + b);
    }
  }
  for (int k = 0; t < ntiles; t += gridDim.x, k++) {
    const int s = k % nst;
    // prefetch the next tile's offsets and descriptor ids before waiting on this one
    const int64_t tn = t + gridDim.x;
    int64_t n0[kExtBpt], n1[kExtBpt];
    int32_t nid[kExtBpt];
#pragma unroll
    for (int j = 0; j < kExtBpt; j++) {
      const int64_t bn = tn * kExtConsumers + j * kC + threadIdx.x;
      n0[j] = n1[j] = 0;
      nid[j] = 0;
      if (tn < ntiles && bn < nb) {
        n0[j] = __ldg(off + bn);
        n1[j] = __ldg(off + bn + 1);
        nid[j] = __ldg(id + bn);
      }
    }
    mbar_wait(smem_u32(&bars[s]), (k / nst) & 1);
    const int64_t a0 = meta[s].a0;
    const bool staged = meta[s].staged;
    int64_t Pt[kExtBpt], Dn[kExtBpt], Ct[kExtBpt];
#pragma unroll
    for (int j = 0; j < kExtBpt; j++) {
      Pt[j] = Dn[j] = Ct[j] = 0;
      if (staged) {
        // 32-bit shared-memory addressing; the slot index is tile-relative (< cap)
        const uint32_t tbase = smem_u32(slots + (size_t)(any_c ? 2 * s : s) * cap), cbase = tbase + 4u * (uint32_t)cap;
        const uint32_t q1 = 4u * (uint32_t)(s1[j] - a0);
        int32_t dn = 0;
        uint32_t q = 4u * (uint32_t)(s0[j] - a0);
        // C (total_context) only feeds Linear models with a context term (predictor.py:
        // 137-142): when no batch of this warp needs it and no features are requested, the
        // context slots are not read (A/B: 58.9% -> 61.4% of HBM with the uniform loop)
        bool need_c = feat != nullptr;
        if (!need_c && any_c && (unsigned)ib[j] < (unsigned)n_desc) {
          const tw_pred_desc* dsc = pset_desc(ps, ib[j]);
          need_c = dsc->kind == TW_PRED_LINEAR && dsc->per_context_token_us != 0.0;
        }
        // warp-uniform trip count (the warp's longest batch) with predicated loads: a lane past
        // its batch's end loads nothing and adds zeros, so the loop carries no divergence
        // bookkeeping; a DecodeSlot is -1 (predictor.py:69-81)
        const uint32_t cnt = (q1 - q) >> 2;
        const uint32_t cmax = __reduce_max_sync(kFull, cnt);
        if (!__any_sync(kFull, need_c)) {
          for (uint32_t i = 0; i < cmax; i++, q += 4u) {
            int32_t x = 0;
            const int act = i < cnt;
            asm volatile("{\n .reg .pred p;\n setp.ne.s32 p, %2, 0;\n @p ld.shared.b32 %0, [%1];\n}"
                         : "+r"(x) : "r"(tbase + q), "r"(act));
            Pt[j] += x > 0 ? x : 0;
            dn += x < 0;
          }
        } else {
          for (uint32_t i = 0; i < cmax; i++, q += 4u) {
            int32_t x = 0, c = 0;
            const int act = i < cnt;
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.s32 p, %3, 0;\n @p ld.shared.b32 %0, [%2];\n @p ld.shared.b32 %1, [%4];\n}"
                : "+r"(x), "+r"(c) : "r"(tbase + q), "r"(act), "r"(cbase + q));
            Pt[j] += x > 0 ? x : 0;
            dn += x < 0;
            Ct[j] += c;
          }
        }
        Dn[j] = dn;
      } else {
        for (int64_t q = s0[j]; q < s1[j]; q++) {
          const int32_t x = __ldg(tok + q);
          if (x >= 0) Pt[j] += x; else Dn[j] += 1;
          Ct[j] += __ldg(ctx + q);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&bars[kExtMaxStages + s]));  // this warp is done with stage s
#pragma unroll
    for (int j = 0; j < kExtBpt; j++) {
      const int64_t b = t * kExtConsumers + j * kC + threadIdx.x;
      if (b < nb) {
        if (feat) {
          feat[3 * b] = Pt[j];
          feat[3 * b + 1] = Dn[j];
          feat[3 * b + 2] = Ct[j];
        }
        int64_t r;
#ifdef TWB_EXT_NOPRED  // A/B only: extraction without the predictor (not the product)
        r = Pt[j] * 3 + Dn[j] * 5 + Ct[j] + ib[j];
        __stcs(out + b, r);
        s0[j] = n0[j];
        s1[j] = n1[j];
        ib[j] = nid[j];
        continue;
#endif
        if (s1[j] == s0[j]) r = TW_PRED_EMPTY_BATCH;
        else if (((Pt[j] | Dn[j]) >> 31) == 0 && Ct[j] >= 0)
          r = predict_one<kShared>(ps, qh, n_desc, (int32_t)Pt[j], (int32_t)Dn[j], Ct[j], ib[j]);
        else r = predict_scalar(ps, ib[j], Pt[j], Dn[j], Ct[j]);
        __stcs(out + b, r);
      }
      s0[j] = n0[j];
      s1[j] = n1[j];
      ib[j] = nid[j];
    }
  }
}

static int pred_grid(int64_t work, size_t smem, const void* fn) {
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kPredThreads, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t want = (work + kPredThreads - 1) / kPredThreads;
  int64_t cap = (int64_t)sms * per_sm;  // one full wave, persistent grid-stride
  if (want > cap) want = cap;
  if (want < 1) want = 1;
  return (int)want;
}

#ifdef TWB_PRED_GLOBAL_TU
// predict_global.cu compiles this file a second time for the instantiations that read a
// blob too large for shared memory through L1. With both instantiations in one
// translation unit, shared helpers stopped being inlined into the staged bulk predictor
// (77% -> 72% of HBM).
void pred_global_features(cudaStream_t s, const void* pset, uint32_t pset_bytes, const int32_t* P, const int32_t* D,
                          const int64_t* C, const int32_t* id, int64_t n, int64_t* out) {
  const int grid = pred_grid((n + 3) / 4, 0, (const void*)k_predict_features<false>);
  k_predict_features<false><<<grid, kPredThreads, 0, s>>>(pset, pset_bytes, P, D, C, id, n, out);
}
void pred_global_batches(int grid, size_t smem, cudaStream_t s, const void* pset, uint32_t pset_bytes, int32_t cap,
                         const int64_t* off, const int32_t* tok, const int32_t* ctx, const int32_t* id, int64_t nb,
                         int64_t* feat, int64_t* out) {
  cudaFuncSetAttribute(k_predict_batches<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_predict_batches<false><<<grid, kExtThreads, smem, s>>>(pset, pset_bytes, 0u, cap, off, tok, ctx, id, nb, feat,
                                                           out);
}
}  // namespace twb
#else
void pred_global_features(cudaStream_t s, const void* pset, uint32_t pset_bytes, const int32_t* P, const int32_t* D,
                          const int64_t* C, const int32_t* id, int64_t n, int64_t* out);  // predict_global.cu
void pred_global_batches(int grid, size_t smem, cudaStream_t s, const void* pset, uint32_t pset_bytes, int32_t cap,
                         const int64_t* off, const int32_t* tok, const int32_t* ctx, const int32_t* id, int64_t nb,
                         int64_t* feat, int64_t* out);

// One batch's features to ns for the single-batch paths: the bulk-lookup section read
// through L1 (three dependent loads) when the blob carries it, else the scalar lookup.
__device__ __forceinline__ int64_t predict_one_global(const char* pset, uint32_t pset_bytes, int32_t desc_id,
                                                      int64_t Pt, int64_t Dn, int64_t Ct) {
  const tw_pset_header* h = reinterpret_cast<const tw_pset_header*>(pset);
  int64_t r;
  if (h->fast_off > 0 && pset_bytes >= (uint32_t)h->total_bytes && ((Pt | Dn) >> 31) == 0 &&
      predict_fast<false>(pset, pset_qhdr(pset), pset_ndesc(pset), (int32_t)Pt, (int32_t)Dn, desc_id, r))
    return r;
  return predict_scalar(pset, desc_id, Pt, Dn, Ct);
}

// Single-batch prediction for the live engine's per-step call (engine.py:684): one
// warp sums the batch's slots (lane-strided, shuffle reduction) and lane 0 predicts
// straight from the global predictor blob (L2-resident; no shared-memory staging for
// one query).
__global__ void __launch_bounds__(32) k_predict_single(const char* __restrict__ pset, const int32_t* __restrict__ io,
                                                      int32_t n, int32_t desc_id, int64_t* __restrict__ out,
                                                      uint32_t pset_bytes) {
  const int lane = threadIdx.x;
  int64_t Pt = 0, Dn = 0, Ct = 0;
  for (int i = lane; i < n; i += 32) {
    const int32_t x = io[i];
    if (x >= 0) Pt += x; else Dn += 1;  // PrefillChunk / DecodeSlot (predictor.py:69-81)
    Ct += io[n + i];
  }
  Pt = warp_sum_i64(Pt);
  Dn = warp_sum_i64(Dn);
  Ct = warp_sum_i64(Ct);
  if (lane == 0) {
    const int64_t r = n == 0 ? (int64_t)TW_PRED_EMPTY_BATCH : predict_one_global(pset, pset_bytes, desc_id, Pt, Dn, Ct);
    // system-scope store: the host polls this word in pinned memory
    asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(out), "l"(r) : "memory");
  }
}

// Self-test of div_rn_rcp against the hardware-correct __ddiv_rn on pseudo-random
// operands shaped like the lerps' (integer numerators up to 2^53, products of a double
// difference and a small integer, integer gaps up to 2^24).
__global__ void k_selftest_division(int64_t n, uint64_t seed, unsigned long long* bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long local = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t h1 = tw_mix64(seed ^ (uint64_t)i * 0x9E3779B97F4A7C15ULL);
    const uint64_t h2 = tw_mix64(h1 + 0x632BE59BD9B4E019ULL);
    const uint64_t h3 = tw_mix64(h2 ^ 0x85EBCA77C2B2AE63ULL);
    const int bits_b = 1 + (int)(h3 % 24);
    const double b = (double)(int64_t)(1 + (h2 >> (64 - bits_b)));
    double a;
    if (h3 & 64) {
      const int bits_a = 1 + (int)((h3 >> 8) % 53);
      a = (double)(int64_t)(h1 >> (64 - bits_a));
      if (h3 & 128) a = -a;
    } else {  // (at_d1 - at_d0) * (x - lo): a double difference times a small integer
      const double u = __ll2double_rn((int64_t)(h1 >> 12)) * 0x1p-30;
      const double v = __ll2double_rn((int64_t)(h2 >> 20)) * 0x1p-25;
      a = __dmul_rn(__dsub_rn(u, v), (double)(1 + (h3 >> 40) % 4096));
    }
    if (div_rn_rcp(a, b, __drcp_rn(b)) != __ddiv_rn(a, b)) local++;
  }
  if (local) atomicAdd(bad, local);
}

static int check_pset(const void* pset, int64_t bytes, size_t* smem) {
  if (!pset || bytes < (int64_t)sizeof(tw_pset_header) || (bytes & 15) ||
      (reinterpret_cast<uintptr_t>(pset) & 15)) {
    set_error("pset: null, misaligned or size %lld not a multiple of 16", (long long)bytes);
    return TW_EINVAL;
  }
  *smem = 128 + (size_t)bytes;
  if (*smem > 200 * 1024) *smem = 0;  // too large to stage: the kernels read it through L1
  return TW_OK;
}

}  // namespace twb

using namespace twb;

extern "C" int tw_predict_features(const void* pset, int64_t pset_bytes, const int32_t* P,
                                   const int32_t* D, const int64_t* C, const int32_t* desc_id,
                                   int64_t n, int64_t* out_ns, void* stream) {
  size_t smem;
  int rc = check_pset(pset, pset_bytes, &smem);
  if (rc) return rc;
  if (n < 0 || (n > 0 && (!P || !D || !C || !desc_id || !out_ns))) {
    set_error("tw_predict_features: bad arrays");
    return TW_EINVAL;
  }
  if (((uintptr_t)P | (uintptr_t)D | (uintptr_t)C | (uintptr_t)desc_id | (uintptr_t)out_ns) & 15) {
    set_error("tw_predict_features: arrays must be 16-byte aligned");
    return TW_EINVAL;
  }
  if (n == 0) return TW_OK;
  if (smem > 0) {
    cudaFuncSetAttribute(k_predict_features<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = pred_grid((n + 3) / 4, smem, (const void*)k_predict_features<true>);
    k_predict_features<true><<<grid, kPredThreads, smem, (cudaStream_t)stream>>>(
        pset, (uint32_t)pset_bytes, P, D, C, desc_id, n, out_ns);
  } else {
    pred_global_features((cudaStream_t)stream, pset, (uint32_t)pset_bytes, P, D, C, desc_id, n, out_ns);
  }
  count_launch();
  return check_launch("tw_predict_features");
}

extern "C" int tw_selftest_division(int64_t n, uint64_t seed, unsigned long long* mismatches, void* stream) {
  if (n < 0 || !mismatches) {
    set_error("tw_selftest_division: bad arguments");
    return TW_EINVAL;
  }
  k_selftest_division<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(n, seed, mismatches);
  count_launch();
  return check_launch("tw_selftest_division");
}

extern "C" int tw_predict_batches(const void* pset, int64_t pset_bytes, const int64_t* batch_off,
                                  const int32_t* slot_tok, const int32_t* slot_ctx,
                                  const int32_t* desc_id, int64_t n_batches, int64_t* feat_out,
                                  int64_t* out_ns, void* stream) {
  size_t smem;
  int rc = check_pset(pset, pset_bytes, &smem);
  if (rc) return rc;
  if (n_batches < 0 || (n_batches > 0 && (!batch_off || !desc_id || !out_ns))) {
    set_error("tw_predict_batches: bad arrays");
    return TW_EINVAL;
  }
  if (n_batches == 0) return TW_OK;
  if (((uintptr_t)slot_tok | (uintptr_t)slot_ctx) & 15) {
    set_error("tw_predict_batches: slot arrays must be 16-byte aligned");
    return TW_EINVAL;
  }
  // shared memory: pset | 2 mbarriers (128 B) | 2 stages x (tok, ctx) x cap slots
  int dev = 0, max_optin = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool staged = smem > 0;  // else the blob is read through L1 (check_pset)
  const uint32_t pset_smem = staged ? (uint32_t)((pset_bytes + 127) & ~127LL) : 0u;
  // the stage region (bytes): the kernel splits it into TWB_EXT_STAGES_C stages of (tok, ctx)
  // or TWB_EXT_STAGES_T stages of tok; a stage holds at most 16 slots per batch of a tile
  int64_t room = (int64_t)max_optin - 1024 /* static */ - 128 - (int64_t)pset_smem - 32 * kExtMaxStages;
  room &= ~127LL;
  if (room > 16LL * 8 * kExtConsumers * TWB_EXT_STAGES_C) room = 16LL * 8 * kExtConsumers * TWB_EXT_STAGES_C;
  if (room < 8LL * kExtConsumers * kExtMaxStages) {
    set_error("tw_predict_batches: predictor blob leaves no room for slot tiles");
    return TW_ENOSMEM;
  }
  const int32_t cap = (int32_t)room;  // the kernel's `region`
  const size_t esmem = 128 + pset_smem + 32 * kExtMaxStages + (size_t)room;
  const int64_t ntiles = (n_batches + kExtConsumers - 1) / kExtConsumers;
  const int grid = (int)(ntiles < sms ? ntiles : sms);
  if (staged) {
    cudaFuncSetAttribute(k_predict_batches<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)esmem);
    k_predict_batches<true><<<grid, kExtThreads, esmem, (cudaStream_t)stream>>>(
        pset, (uint32_t)pset_bytes, pset_smem, cap, batch_off, slot_tok, slot_ctx, desc_id, n_batches, feat_out,
        out_ns);
  } else {
    pred_global_batches(grid, esmem, (cudaStream_t)stream, pset, (uint32_t)pset_bytes, cap, batch_off, slot_tok,
                        slot_ctx, desc_id, n_batches, feat_out, out_ns);
  }
  count_launch();
  return check_launch("tw_predict_batches");
}

extern "C" int tw_predict_one_sync(const void* pset, int64_t pset_bytes, const int32_t* host_slots, int32_t n_slots,
                                   int32_t desc_id, void* pinned_io, int64_t io_bytes, int64_t* out_ns,
                                   void* stream) {
  if (!pset || !pinned_io || !out_ns || n_slots < 0 || (n_slots > 0 && !host_slots) ||
      io_bytes < 8 * (int64_t)n_slots + 8 || pset_bytes < (int64_t)sizeof(tw_pset_header)) {
    set_error("tw_predict_one_sync: bad arguments");
    return TW_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  // pinned layout: int32 tok[n] | int32 ctx[n] | (8-byte aligned) int64 result. Pinned
  // host memory is device-addressable under UVA, so the kernel reads the slots and
  // writes the answer in place (zero-copy: no memcpy calls on the round trip).
  char* h = static_cast<char*>(pinned_io);
  const size_t slots = 8 * (size_t)n_slots, res = (slots + 7) & ~(size_t)7;
  if (n_slots) memcpy(h, host_slots, slots);
  // the answer word starts as a value no answer takes (ns >= 0, TW_PRED_* codes are small
  // negatives); the host polls it instead of synchronizing the stream (~10 us less)
  volatile int64_t* ans = reinterpret_cast<volatile int64_t*>(h + res);
  *ans = INT64_MIN;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  k_predict_single<<<1, 32, 0, s>>>(static_cast<const char*>(pset), reinterpret_cast<const int32_t*>(h), n_slots,
                                    desc_id, reinterpret_cast<int64_t*>(h + res), (uint32_t)pset_bytes);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) {
    timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    for (uint32_t spin = 0; *ans == INT64_MIN; spin++) {
      if ((spin & 1023u) == 1023u) {  // a kernel that cannot answer: surface its error
        clock_gettime(CLOCK_MONOTONIC, &t1);
        if ((t1.tv_sec - t0.tv_sec) * 1000000000LL + (t1.tv_nsec - t0.tv_nsec) > 200000000LL) {
          e = cudaStreamSynchronize(s);
          if (e == cudaSuccess && *ans == INT64_MIN) e = cudaErrorUnknown;
          break;
        }
      }
    }
  }
  if (e != cudaSuccess) {
    set_error("tw_predict_one_sync: %s", cudaGetErrorString(e));
    return TW_ECUDA;
  }
  *out_ns = *ans;
  return TW_OK;
}

// ---------------------------------------------------------------------------------
// Resident predictor service for the live engine (engine.py:684 calls predict() once
// per step from one thread). One persistent warp polls a mailbox in mapped pinned
// host memory; a request is the batch's slots, the answer is written back into the
// mailbox. No launch, copy or stream synchronisation sits on the round trip, which is
// then bounded by PCIe latency (a few microseconds) instead of kernel launch + sync.
// ---------------------------------------------------------------------------------
struct tw_service_mailbox {
  // host -> device, 32 bytes read by one PCIe round trip of four lanes: q[0] is the request
  // word, written last: request counter (bits 40-63), descriptor (bits 24-39; 0xffff = stop)
  // and slot count (bits 0-23; 0xffffff = a features request). A features request carries
  // P, D, C in q[1..3], each tagged with the counter's low 16 bits in bits 48-63, so a read
  // torn against the host's writes is recognised and repeated.
  volatile uint64_t q[4];
  volatile int64_t result;  // device -> host: ns or a TW_PRED_* code
  volatile uint64_t ack;    // device -> host: the request word answered (ordered after result)
  volatile int32_t cap, pad;
  volatile int32_t slots[1];  // tok[n] then ctx[n] (slot requests)
};
constexpr uint32_t kSvcFeatures = 0xffffffu;
constexpr uint64_t kSvcTagMask = 0xffffULL << 48;

// TWB_SVC_SLEEP_NS: back-off between polls (A/B; 0 = spin)
#ifndef TWB_SVC_SLEEP_NS
#define TWB_SVC_SLEEP_NS 0
#endif
__global__ void __launch_bounds__(32) k_predict_service(const char* __restrict__ pset_g, uint32_t pset_bytes,
                                                       uint32_t staged, tw_service_mailbox* mb) {
  extern __shared__ __align__(128) char smem[];
  const int lane = threadIdx.x;
  // the blob stays in shared memory for the service's life when it fits (one lookup is a
  // chain of dependent reads: shared memory instead of L2 on every step)
  if (staged) tma_stage_to_smem(smem + 128, pset_g, pset_bytes, reinterpret_cast<uint64_t*>(smem));
  const char* ps = staged ? static_cast<const char*>(smem + 128) : pset_g;
  const tw_pset_header* h = reinterpret_cast<const tw_pset_header*>(ps);
  const bool fast = h->fast_off > 0 && pset_bytes >= (uint32_t)h->total_bytes;
  const int n_desc = pset_ndesc(ps);
  uint64_t seen = 0;
  for (;;) {
    uint64_t v = 0, w = 0;
    for (;;) {
      if (lane < 4) v = mb->q[lane];  // one 32-byte read
      w = __shfl_sync(kFull, v, 0);
      if (w == seen) {
#if TWB_SVC_SLEEP_NS > 0
        __nanosleep(TWB_SVC_SLEEP_NS);
#endif
        continue;
      }
      if ((w & 0xffffffu) != kSvcFeatures) break;
      const uint64_t tag = (w >> 40) << 48;  // the counter's low 16 bits
      if (__all_sync(kFull, lane < 1 || lane >= 4 || (v & kSvcTagMask) == tag)) break;  // not torn
    }
    const int32_t desc = (int32_t)((w >> 24) & 0xffffu);
    if (desc == 0xffff) return;  // stop
    const uint32_t n = (uint32_t)(w & 0xffffffu);
    int64_t Pt = 0, Dn = 0, Ct = 0;
    if (n == kSvcFeatures) {  // P, D, C extracted on the host (the batch's three sums)
      Pt = (int64_t)(__shfl_sync(kFull, v, 1) & ~kSvcTagMask);
      Dn = (int64_t)(__shfl_sync(kFull, v, 2) & ~kSvcTagMask);
      Ct = (int64_t)(__shfl_sync(kFull, v, 3) & ~kSvcTagMask);
    } else {
      for (uint32_t i = lane; i < n; i += 32) {
        const int32_t x = mb->slots[i], c = mb->slots[n + i];  // one round of PCIe reads
        if (x >= 0) Pt += x; else Dn += 1;  // PrefillChunk / DecodeSlot (predictor.py:69-81)
        Ct += c;
      }
      Pt = warp_sum_i64(Pt);
      Dn = warp_sum_i64(Dn);
      Ct = warp_sum_i64(Ct);
    }
    if (lane == 0) {
      int64_t r;
      if (n == 0) r = TW_PRED_EMPTY_BATCH;
      else if (fast && ((Pt | Dn) >> 31) == 0 && Ct >= 0 &&
               (staged ? predict_fast<true>(ps, pset_qhdr(ps), n_desc, (int32_t)Pt, (int32_t)Dn, desc, r)
                       : predict_fast<false>(ps, pset_qhdr(ps), n_desc, (int32_t)Pt, (int32_t)Dn, desc, r))) {
      } else {
        r = predict_scalar(ps, desc, Pt, Dn, Ct);
      }
      mb->result = r;
      // the result before the acknowledgement, system-wide (a release store: no full fence)
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&mb->ack), "l"(w) : "memory");
    }
    seen = w;
    __syncwarp();
  }
}

struct tw_service {
  tw_service_mailbox* host;
  tw_service_mailbox* dev;
  cudaStream_t stream;
  uint64_t seq;
  int32_t cap;
};

extern "C" int tw_service_start(const void* pset, int64_t pset_bytes, int32_t max_slots, tw_service** out) {
  if (!pset || !out || max_slots < 1 || pset_bytes < (int64_t)sizeof(tw_pset_header)) {
    set_error("tw_service_start: bad arguments");
    return TW_EINVAL;
  }
  tw_service* sv = new tw_service();
  const size_t bytes = sizeof(tw_service_mailbox) + 8 * (size_t)max_slots;
  void* h = nullptr;
  if (cudaHostAlloc(&h, bytes, cudaHostAllocMapped) != cudaSuccess) {
    delete sv;
    set_error("tw_service_start: cudaHostAlloc failed");
    return TW_ECUDA;
  }
  memset(h, 0, bytes);
  sv->host = static_cast<tw_service_mailbox*>(h);
  sv->host->cap = max_slots;
  void* d = nullptr;
  cudaHostGetDevicePointer(&d, h, 0);
  sv->dev = static_cast<tw_service_mailbox*>(d);
  sv->seq = 0;
  sv->cap = max_slots;
  cudaStreamCreateWithFlags(&sv->stream, cudaStreamNonBlocking);
  int dev = 0, max_optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t stage_bytes = 128 + (((size_t)pset_bytes + 127) & ~(size_t)127);
  const uint32_t staged = ((pset_bytes & 15) == 0 && stage_bytes <= (size_t)max_optin) ? 1u : 0u;
  if (staged) cudaFuncSetAttribute(k_predict_service, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stage_bytes);
  k_predict_service<<<1, 32, staged ? stage_bytes : 0, sv->stream>>>(static_cast<const char*>(pset),
                                                                     (uint32_t)pset_bytes, staged, sv->dev);
  count_launch();
  const int rc = check_launch("tw_service_start");
  if (rc != TW_OK) {
    cudaStreamDestroy(sv->stream);
    cudaFreeHost(h);
    delete sv;
    return rc;
  }
  *out = sv;
  return TW_OK;
}

extern "C" int tw_service_predict(tw_service* sv, const int32_t* host_slots, int32_t n_slots, int32_t desc_id,
                                  int64_t* out_ns) {
  if (!sv || !out_ns || n_slots < 0 || n_slots > sv->cap || (n_slots > 0 && !host_slots)) {
    set_error("tw_service_predict: bad arguments (n_slots %d, capacity %d)", n_slots, sv ? sv->cap : 0);
    return TW_EINVAL;
  }
  if (desc_id < 0 || desc_id >= 0xffff || n_slots >= (1 << 24)) {
    set_error("tw_service_predict: descriptor %d or slot count %d out of range", desc_id, n_slots);
    return TW_EINVAL;
  }
  tw_service_mailbox* mb = sv->host;
  for (int i = 0; i < 2 * n_slots; i++) mb->slots[i] = host_slots[i];
  __sync_synchronize();  // the slots before the request word
  const uint64_t w = ((uint64_t)(++sv->seq & 0xffffff) << 40) | ((uint64_t)desc_id << 24) | (uint64_t)n_slots;
  mb->q[0] = w;
  for (int64_t spins = 0; mb->ack != w; spins++) {
    if ((spins & 0xfffff) == 0xfffff && cudaStreamQuery(sv->stream) != cudaErrorNotReady) {
      set_error("tw_service_predict: the service kernel is not running");
      return TW_ECUDA;
    }
  }
  __sync_synchronize();
  *out_ns = mb->result;
  return TW_OK;
}

extern "C" int tw_service_predict_features(tw_service* sv, int64_t total_prefill_tokens, int64_t num_decodes,
                                           int64_t total_context, int32_t desc_id, int64_t* out_ns) {
  if (!sv || !out_ns || desc_id < 0 || desc_id >= 0xffff || total_prefill_tokens < 0 || num_decodes < 0 ||
      total_context < 0 || ((total_prefill_tokens | num_decodes | total_context) >> 48) != 0) {
    set_error("tw_service_predict_features: bad arguments");
    return TW_EINVAL;
  }
  tw_service_mailbox* mb = sv->host;
  const uint64_t seq = ++sv->seq & 0xffffff;
  const uint64_t tag = (seq & 0xffff) << 48;
  mb->q[1] = tag | (uint64_t)total_prefill_tokens;
  mb->q[2] = tag | (uint64_t)num_decodes;
  mb->q[3] = tag | (uint64_t)total_context;
  __sync_synchronize();  // the features before the request word
  const uint64_t w = (seq << 40) | ((uint64_t)desc_id << 24) | (uint64_t)kSvcFeatures;
  mb->q[0] = w;
  for (int64_t spins = 0; mb->ack != w; spins++) {
    if ((spins & 0xfffff) == 0xfffff && cudaStreamQuery(sv->stream) != cudaErrorNotReady) {
      set_error("tw_service_predict_features: the service kernel is not running");
      return TW_ECUDA;
    }
  }
  __sync_synchronize();
  *out_ns = mb->result;
  return TW_OK;
}

extern "C" int tw_service_stop(tw_service* sv) {
  if (!sv) return TW_OK;
  __sync_synchronize();
  sv->host->q[0] = ((uint64_t)(++sv->seq & 0xffffff) << 40) | (0xffffULL << 24);  // stop
  const cudaError_t e = cudaStreamSynchronize(sv->stream);
  cudaStreamDestroy(sv->stream);
  cudaFreeHost(sv->host);
  delete sv;
  if (e != cudaSuccess) {
    set_error("tw_service_stop: %s", cudaGetErrorString(e));
    return TW_ECUDA;
  }
  return TW_OK;
}
#endif  // TWB_PRED_GLOBAL_TU
