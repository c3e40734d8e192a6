// Performance-gap diagnosis (PAPER §VII-B):
// gap = y_p80 - t_theory / measured, underperforming <=> gap > 0.1, with
// per-spec counts and a per-spec gap histogram (Fig. 7's CDF).  HBM-bound
// streaming pass; per-spec tallies are aggregated across the warp (spec-major
// pairs give runs of equal (spec, bin) keys), into a per-block shared-memory
// copy when the G x (n_bins + 2) tallies fit in 48 KB (global atomics on ~1,000
// counters measured 267 GB/s), else straight into the global counters.
#include <cuda_runtime.h>

#include <cmath>

#include "ctx.h"
#include "sp_internal.h"
#include "synperf.h"

using namespace sp;

namespace {

struct GapArgs {
  const float *tt;       // t_theory_us row of the features
  const uint8_t *status;
  const float *p80, *meas;
  int64_t n;
  int32_t cross;         // 1: spec = p / n_configs; 0: spec_idx[p] (absolute) - spec_base
  int64_t n_configs;
  const int32_t *spec_idx;
  int32_t G, n_bins;
  float lo, hi;
  float *gap;
  unsigned long long *counts, *hist;
};

__device__ __forceinline__ void warp_add(unsigned long long *dst, uint32_t key, bool on) {
  const unsigned act = __ballot_sync(0xffffffffu, on);
  if (!on) return;
  const unsigned peers = __match_any_sync(act, key);
  if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(dst, (unsigned long long)__popc(peers));
}

// SMEM: the block's private copy of counts [G][2] and hist [G][n_bins]
// (flushed once per block), when it fits; else global atomics.
template <bool PRIV>
__global__ void __launch_bounds__(256) perf_gap_kernel(GapArgs a) {
  extern __shared__ uint32_t priv[];  // 32-bit block tallies (a block sees < 2^32 pairs)
  const int64_t n_priv = 2 * (int64_t)a.G + (int64_t)a.G * a.n_bins;
  if (PRIV) {
    for (int64_t i = threadIdx.x; i < n_priv; i += blockDim.x) priv[i] = 0;
    __syncthreads();
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n_round = (a.n + 31) / 32 * 32;  // whole warps stay in the loop (warp-level tallies)
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n_round; p += stride) {
    bool valid = false;
    int32_t g = 0;
    float gp = __int_as_float(0x7fc00000);
    if (p < a.n) {
      g = a.cross ? (int32_t)(p / a.n_configs) : __ldg(a.spec_idx + p);
      const float t = __ldg(a.tt + p), m = __ldg(a.meas + p), y80 = __ldg(a.p80 + p);
      if (__ldg(a.status + p) == 0 && g >= 0 && g < a.G && m > 0.f && !isnan(t) && !isnan(y80)) {
        const float y = __fdiv_rn(t, m);  // y_actual (IEEE division)
        gp = __fsub_rn(y80, y);
        valid = !isnan(gp);
      }
      if (a.gap) a.gap[p] = valid ? gp : __int_as_float(0x7fc00000);
    }
    const bool under = valid && gp > SP_GAP_THRESHOLD;
    int32_t bin = 0;
    if (valid) {
      const float f = (gp - a.lo) / (a.hi - a.lo) * (float)a.n_bins;
      bin = f < 0.f ? 0 : (f >= (float)a.n_bins ? a.n_bins - 1 : (int32_t)f);
    }
    if (PRIV) {  // shared-memory atomics: native 32-bit, no aggregation needed
      if (valid) {
        atomicAdd(priv + 2 * g, 1u);
        if (under) atomicAdd(priv + 2 * g + 1, 1u);
        atomicAdd(priv + 2 * (int64_t)a.G + (int64_t)g * a.n_bins + bin, 1u);
      }
    } else {
      warp_add(a.counts + 2 * (int64_t)g, (uint32_t)g, valid);
      warp_add(a.counts + 2 * (int64_t)g + 1, (uint32_t)g, under);
      warp_add(a.hist + (int64_t)g * a.n_bins + bin, (uint32_t)(g * a.n_bins + bin), valid);
    }
  }
  if (PRIV) {
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n_priv; i += blockDim.x) {
      const unsigned long long v = priv[i];
      if (!v) continue;  // flush the block's tallies
      if (i < 2 * (int64_t)a.G) atomicAdd(a.counts + i, v);
      else atomicAdd(a.hist + (i - 2 * (int64_t)a.G), v);
    }
  }
}

}  // namespace

extern "C" sp_status sp_perf_gap(sp_ctx *ctx, const sp_features *in, const float *eff_p80, const float *measured_us,
                                 const sp_pairing *pairs, int64_t n_configs, int32_t n_specs, int32_t n_bins,
                                 float gap_lo, float gap_hi, float *gap, int64_t *counts, int64_t *hist,
                                 void *stream) {
  if (!ctx) return fail(nullptr, SP_E_ARG, "sp_perf_gap: ctx is NULL");
  if (!in || !pairs || !counts || !hist) return fail(ctx, SP_E_ARG, "sp_perf_gap: NULL argument");
  if (n_bins < 1 || !(gap_hi > gap_lo) || !std::isfinite(gap_lo) || !std::isfinite(gap_hi))
    return fail(ctx, SP_E_ARG, "sp_perf_gap: need n_bins >= 1 and a finite gap_lo < gap_hi");
  const int64_t n = in->n_pairs;
  if (n < 0 || in->ld < n) return fail(ctx, SP_E_ARG, "sp_perf_gap: bad n_pairs / ld");
  GapArgs a{};
  if (pairs->kind == SP_PAIRS_CROSS) {
    if (pairs->spec_end < pairs->spec_begin || n_configs < 0) return fail(ctx, SP_E_ARG, "sp_perf_gap: bad spec range");
    a.G = pairs->spec_end - pairs->spec_begin;
    if ((int64_t)a.G * n_configs != n) return fail(ctx, SP_E_ARG, "sp_perf_gap: n_pairs != specs x n_configs");
    a.cross = 1;
    a.n_configs = n_configs > 0 ? n_configs : 1;
  } else if (pairs->kind == SP_PAIRS_LIST) {
    if (pairs->n_pairs != n || (n > 0 && !pairs->spec_idx) || n_specs < 0)
      return fail(ctx, SP_E_ARG, "sp_perf_gap: pair list does not match the features");
    a.G = n_specs;
    a.spec_idx = pairs->spec_idx;
  } else {
    return fail(ctx, SP_E_ARG, "sp_perf_gap: unknown pairing kind");
  }
  ctx->err.clear();
  cudaSetDevice(ctx->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (a.G > 0) {
    if ((e = cudaMemsetAsync(counts, 0, sizeof(int64_t) * 2 * (size_t)a.G, st)) != cudaSuccess ||
        (e = cudaMemsetAsync(hist, 0, sizeof(int64_t) * (size_t)n_bins * a.G, st)) != cudaSuccess)
      return cuda_fail(ctx, e, "sp_perf_gap: clear");
  }
  if (n == 0) return SP_OK;
  if (!eff_p80 || !measured_us || !in->flts || !in->status) return fail(ctx, SP_E_ARG, "sp_perf_gap: NULL buffer");
  a.tt = in->flts + (int64_t)F_TTHEORY * in->ld;
  a.status = in->status;
  a.p80 = eff_p80;
  a.meas = measured_us;
  a.n = n;
  a.n_bins = n_bins;
  a.lo = gap_lo;
  a.hi = gap_hi;
  a.gap = gap;
  a.counts = reinterpret_cast<unsigned long long *>(counts);
  a.hist = reinterpret_cast<unsigned long long *>(hist);
  const size_t priv = sizeof(uint32_t) * (2 * (size_t)a.G + (size_t)a.G * n_bins);
  const bool use_priv = priv <= 48 * 1024;
  // privatised tallies: fewer blocks, each over many pairs, so the flush is amortised
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * (use_priv ? 2 : 8));
  const LaunchHook hk = ctx->hook();
  hk.on_begin("perf_gap", stream);
  if (use_priv) perf_gap_kernel<true><<<(unsigned)blocks, 256, priv, st>>>(a);
  else perf_gap_kernel<false><<<(unsigned)blocks, 256, 0, st>>>(a);
  hk.on_end(stream);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(ctx, e, "sp_perf_gap: launch");
  return SP_OK;
}
