// workload.cu — bulk Poisson workload generation on device.
//
// Reference: generate_arrivals / _poisson_arrivals (pkg/src/timewarp/workload.py:
// 118-144): one numpy Generator per workload (np.random.default_rng(seed)), draws
// interleaved per request in the frozen order gap -> prompt -> output:
//     gap_s = rng.exponential(1 / qps); clock += int(round(gap_s * 1e9))
//     prompt = int(rng.integers(low, high + 1))   (or a fixed value: no draw)
//     output = int(rng.integers(low, high + 1))
// restated over numpy's own algorithms (numpy 2.x, the reference's only dependency):
//   * bit generator PCG64 (XSL-RR 128/64): state = state * M + inc, output
//     rotr64(hi ^ lo, hi >> 58); next_uint32 returns the low half of a 64-bit draw and
//     buffers the high half; next_double = (next_uint64 >> 11) * 2^-53;
//   * Generator.exponential(scale) = scale * random_standard_exponential: the 256-layer
//     ziggurat with numpy's tables (ziggurat_tables.h, extracted from the installed
//     numpy by scripts/gen_ziggurat.py), tail r - log1p(-U), wedge test
//     (fe[i-1] - fe[i]) * U + fe[i] < exp(-x), else retry;
//   * Generator.integers(low, high + 1) for int64: Lemire's bounded method on 32-bit
//     draws (random_bounded_uint64 -> buffered_bounded_lemire_uint32).
// The host seeds each workload (default_rng(seed).bit_generator.state) and the device
// runs the sequential draw stream, one thread per workload. The rare ziggurat
// slow paths use CUDA's log1p / exp, which may differ from glibc's in the last ulp;
// that can only matter when a result sits on a rounding or comparison boundary
// (never observed against the fixtures; tests/test_gpu_parity.py).
#include <cmath>

#include "common.cuh"
#include "ziggurat_tables.h"

namespace twb {

constexpr int kWlThreads = 128;
constexpr uint64_t kPcgMultHi = 0x2360ED051FC65DA4ULL, kPcgMultLo = 0x4385DF649FCCF645ULL;
constexpr double kZigExpR = 7.69711747013104972;  // ziggurat_exp_r

struct Pcg64 {
  uint64_t hi, lo, inc_hi, inc_lo;
  bool has32;
  uint32_t u32;
  __device__ __forceinline__ uint64_t next64() {
    // state = state * M + inc (mod 2^128)
    const uint64_t l = lo * kPcgMultLo;
    uint64_t h = __umul64hi(lo, kPcgMultLo) + hi * kPcgMultLo + lo * kPcgMultHi;
    uint64_t nl = l + inc_lo;
    h += inc_hi + (nl < l ? 1ULL : 0ULL);
    lo = nl;
    hi = h;
    const uint64_t x = hi ^ lo;
    const unsigned rot = (unsigned)(hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  __device__ __forceinline__ uint32_t next32() {
    if (has32) {
      has32 = false;
      return u32;
    }
    const uint64_t n = next64();
    has32 = true;
    u32 = (uint32_t)(n >> 32);
    return (uint32_t)n;
  }
  __device__ __forceinline__ double next_double() {
    return __dmul_rn((double)(next64() >> 11), 1.0 / 9007199254740992.0);
  }
};

// Generator.integers(low, high + 1): off + buffered_bounded_lemire_uint32(rng = high - low)
__device__ __forceinline__ int32_t bounded(Pcg64& g, int32_t low, int32_t high) {
  const uint32_t rng = (uint32_t)((int64_t)high - (int64_t)low);
  if (rng == 0) return low;
  if (rng == 0xFFFFFFFFu) return (int32_t)((int64_t)low + g.next32());
  const uint32_t excl = rng + 1u;
  uint64_t m = (uint64_t)g.next32() * excl;
  uint32_t left = (uint32_t)m;
  if (left < excl) {
    const uint32_t threshold = (0xFFFFFFFFu - rng) % excl;
    while (left < threshold) {
      m = (uint64_t)g.next32() * excl;
      left = (uint32_t)m;
    }
  }
  return (int32_t)((int64_t)low + (int64_t)(m >> 32));
}

__device__ __forceinline__ int32_t sample_tokens(Pcg64& g, int32_t kind, int32_t a, int32_t b) {
  return kind == TW_TOKENS_FIXED ? a : bounded(g, a, b);  // TokenDist.sample (workload.py:39-44)
}

// Laid out for the memory system (profiles/README.md: 2.49 -> 0.85 ms for 65,536 x 1,000):
//  * the ziggurat's (ke, we) pair is one 16-byte shared-memory record: one LDS.128 per
//    draw instead of two randomly indexed LDS.64;
//  * each warp generates its 32 workloads in blocks of 16 requests into a padded
//    shared-memory tile, then writes every workload's block as one coalesced row
//    (storing each draw directly touched 32 cache lines per instruction).
struct ZigPair {
  uint64_t ke;
  double we;
};

// random_standard_exponential (numpy distributions.c)
__device__ double std_exponential(Pcg64& g, const ZigPair* __restrict__ zp, const double* __restrict__ fe) {
  for (;;) {
    uint64_t ri = g.next64() >> 3;
    const int idx = (int)(ri & 0xff);
    ri >>= 8;
    const ZigPair z = zp[idx];
    const double x = __dmul_rn((double)ri, z.we);
    if (ri < z.ke) return x;  // 98.9% of draws
    if (idx == 0) return __dsub_rn(kZigExpR, log1p(-g.next_double()));
    const double u = g.next_double();
    if (__dadd_rn(__dmul_rn(__dsub_rn(fe[idx - 1], fe[idx]), u), fe[idx]) < exp(-x)) return x;
  }
}

constexpr int kWlBlock = 16;  // requests per thread per staged block (41 KB of shared memory per CTA)
__global__ void __launch_bounds__(kWlThreads) k_generate_poisson(
    const tw_wl_spec* __restrict__ specs, int32_t n_wl, const int64_t* __restrict__ wl_off,
    int64_t* __restrict__ offset_ns, int32_t* __restrict__ prompt, int32_t* __restrict__ output,
    int32_t* __restrict__ status) {
  __shared__ ZigPair zp[256];
  __shared__ double fe[256];
  __shared__ int64_t t_off[kWlThreads / 32][32][kWlBlock + 1];
  __shared__ int32_t t_pr[kWlThreads / 32][32][kWlBlock + 1];
  __shared__ int32_t t_op[kWlThreads / 32][32][kWlBlock + 1];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    zp[i].ke = kZigKe[i];
    zp[i].we = kZigWe[i];
    fe[i] = kZigFe[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = w < n_wl;
  tw_wl_spec sp;
  int64_t base = 0, n = 0;
  if (live) {
    sp = specs[w];
    base = wl_off[w];
    n = wl_off[w + 1] - base;
  } else {
    sp = specs[0];  // any valid spec; nothing is generated or stored
  }
  Pcg64 g{sp.state_hi, sp.state_lo, sp.inc_hi, sp.inc_lo, sp.has_uint32 != 0, sp.uinteger};
  int64_t nmax = n;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t v = __shfl_xor_sync(0xffffffffu, nmax, o);
    nmax = v > nmax ? v : nmax;
  }
  int64_t clock = 0;
  int32_t st = 0;
  for (int64_t b0 = 0; b0 < nmax; b0 += kWlBlock) {
    const int cnt = (int)(n - b0 < kWlBlock ? (n - b0 > 0 ? n - b0 : 0) : kWlBlock);
    for (int k = 0; k < cnt; k++) {
      const double gap_s = __dmul_rn(sp.scale, std_exponential(g, zp, fe));
      clock += __double2ll_rn(__dmul_rn(gap_s, 1e9));  // int(round(gap_s * NS_PER_S))
      const int32_t p = sample_tokens(g, sp.prompt_kind, sp.prompt_a, sp.prompt_b);
      const int32_t o = sample_tokens(g, sp.output_kind, sp.output_a, sp.output_b);
      if ((p <= 0 || o <= 0) && st == 0) st = (int32_t)(b0 + k + 1);  // WorkloadError at request i
      t_off[warp][lane][k] = clock;
      t_pr[warp][lane][k] = p;
      t_op[warp][lane][k] = o;
    }
    __syncwarp();
    // rows r, r + 1 = the blocks of the warp's r-th and (r+1)-th workloads: half-warp h
    // stores row r + h, lane j of it request j
    const int h = lane >> 4, j = lane & 15;
    for (int r = 0; r < 32; r += 2) {
      const int64_t nr = __shfl_sync(0xffffffffu, n, r + h), br = __shfl_sync(0xffffffffu, base, r + h);
      if (b0 + j < nr) {
        offset_ns[br + b0 + j] = t_off[warp][r + h][j];
        prompt[br + b0 + j] = t_pr[warp][r + h][j];
        output[br + b0 + j] = t_op[warp][r + h][j];
      }
    }
    __syncwarp();
  }
  if (live) status[w] = st;
}

}  // namespace twb

using namespace twb;

extern "C" int tw_generate_poisson(const tw_wl_spec* specs, int32_t n_wl, const int64_t* wl_off,
                                   int64_t* offset_ns, int32_t* prompt, int32_t* output, int32_t* status,
                                   void* stream) {
  if (n_wl < 0 || (n_wl > 0 && (!specs || !wl_off || !offset_ns || !prompt || !output || !status))) {
    set_error("tw_generate_poisson: bad arguments");
    return TW_EINVAL;
  }
  if (n_wl == 0) return TW_OK;
  const int grid = (n_wl + kWlThreads - 1) / kWlThreads;
  k_generate_poisson<<<grid, kWlThreads, 0, (cudaStream_t)stream>>>(specs, n_wl, wl_off, offset_ns, prompt, output,
                                                                    status);
  count_launch();
  return check_launch("tw_generate_poisson");
}
