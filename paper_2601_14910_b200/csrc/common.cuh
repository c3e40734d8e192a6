// Device helpers shared by the feature kernels: field loads, the occupancy /
// waves closed form (a4), the cycle features (a7-a8) and the record store (a9).
#pragma once

#include <cstdint>

#include "sp_internal.h"

namespace sp {

__device__ __forceinline__ int64_t cdiv64(int64_t a, int64_t b) { return (a + b - 1) / b; }
__device__ __forceinline__ int32_t cdiv32(int32_t a, int32_t b) { return (a + b - 1) / b; }

__device__ __forceinline__ int bytes_per_elem(int dtype) {
  return (dtype == SP_BF16 || dtype == SP_FP16) ? 2 : (dtype == SP_FP32 ? 4 : 0);
}

// Unsigned 32-bit division by a runtime-invariant divisor d >= 1 via a
// multiply-high (round-up method): q = (umulhi(n, m) + n) >> s, computed in
// 64 bits so it is exact for every n < 2^32.
// Magic multiplier of d (not a power of two), s = ceil(log2 d):
// m = floor(2^(32+s) / d) - 2^32 + 1.  The quotient comes from an fp64 division
// (within one of the exact value) corrected by a 64-bit multiply check: a few
// instructions instead of the ~100 of the 64-bit integer division subroutine.
__device__ __forceinline__ uint32_t fastdiv_magic(uint32_t d, uint32_t s) {
  if (s >= 32) return (uint32_t)((((1ull << s) - d) << 32) / d + 1);  // d > 2^31: integer path
  const uint64_t num = 1ull << (32 + s);
  uint64_t q = (uint64_t)__ddiv_rz((double)num, (double)d);
  if (q * d > num) --q;                // q < 2^33, d < 2^32: no overflow
  else if ((q + 1) * d <= num) ++q;
  return (uint32_t)(q - (1ull << 32) + 1);
}

struct FastDiv {
  uint32_t d, m, s;
  __device__ __forceinline__ void init(uint32_t div) {
    d = div;
    s = div <= 1 ? 0 : 32 - __clz(div - 1);
    m = (div & (div - 1)) ? fastdiv_magic(div, s) : 1u;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    uint64_t t = (uint64_t)__umulhi(n, m) + n;
    return (uint32_t)(t >> s);
  }
  __device__ __forceinline__ uint32_t mod(uint32_t n) const { return n - div(n) * d; }
  // n < 2^31: the sum umulhi(n, m) + n < 2n stays in 32 bits
  __device__ __forceinline__ uint32_t div31(uint32_t n) const { return (__umulhi(n, m) + n) >> s; }
};

// Footprint of one task (O2 inputs) and the per-pair accumulated demands.
struct Footprint {
  int64_t smem;   // bytes per task (0: no smem quota, R6)
  int64_t warps;
  int64_t regs;
};

struct PairDemand {
  int64_t T;        // tasks
  int64_t tot[4];   // GPU totals: Tensor, FMA, XU ops, load bytes
  int64_t mx[4];    // max over SMs per quantity (R7)
};

// floor(a / b), b >= 1, exact: for a < 2^24 an fp32 reciprocal estimate
// corrected by one either way (the integer division is ~20 instructions);
// larger a take the integer division.
__device__ __forceinline__ uint32_t udiv_q(uint32_t a, uint32_t b) {
  if (a >= (1u << 24)) return a / b;
  uint32_t q = (uint32_t)__fmul_rz((float)a, __frcp_rn((float)b));  // within one of floor(a/b)
  if (q * b > a) --q;                                                 // (q + 1) b <= a + b < 2^25
  else if ((q + 1) * b <= a) ++q;
  return q;
}

template <bool FAST>
__device__ __forceinline__ uint32_t udiv(uint32_t a, uint32_t b) {
  return FAST ? udiv_q(a, b) : a / b;
}

// a4: occ = max(1, min(smem quota, RF quota, warp quota, CTA limit)) (R6).
template <bool FAST = false>
__device__ __forceinline__ int64_t occupancy(const Footprint &fp, const DevSpec &s) {
  int64_t occ = s.max_ctas;
  if (fp.smem > 0) occ = min(occ, fp.smem > s.smem_per_sm ? 0 : (int64_t)udiv<FAST>((uint32_t)s.smem_per_sm, (uint32_t)fp.smem));
  int64_t rden = fp.regs * 32 * fp.warps;
  occ = min(occ, rden > s.regs_per_sm ? 0 : (int64_t)udiv<FAST>((uint32_t)s.regs_per_sm, (uint32_t)rden));
  occ = min(occ, fp.warps > s.max_warps ? 0 : (int64_t)udiv<FAST>((uint32_t)s.max_warps, (uint32_t)fp.warps));
  return occ < 1 ? 1 : occ;
}

// waves = ceil(T / (N_SM * occ)) with T < 2^31.
template <bool FAST = false>
__device__ __forceinline__ int64_t waves_of(int64_t T, int64_t nsm, int64_t occ) {
  int64_t den = nsm * occ;
  if (T == 0) return 0;
  if (den >= T) return 1;
  return (int64_t)udiv<FAST>((uint32_t)T + (uint32_t)den - 1u, (uint32_t)den);
}

// a7-a9: cycles from the exact integers in fp64, one rounding to fp32 (R20),
// and the record store.  tdt = tensor dtype index (0 bf16, 1 fp16, 2 fp8).
// fv (optional): receives the 12 float slots as stored (the fused predictor
// normalises them without reading the record back).
// FAST: fp32-reciprocal quotients (udiv_q) -- the fused predictor's producers
// use them for every family (round 2: 1.7% faster on cfg3 once layer 3 moved to
// TMEM; earlier it had slowed the MoE instantiation at the 80-register cap).
template <bool FAST = false>
__device__ __forceinline__ void emit_pair(const FeatOut &o, int64_t p, const PairDemand &d,
                                          const Footprint &fp, const DevSpec &s, int pipes,
                                          int tdt, float *fv = nullptr) {
  const int64_t ld = o.ld;
  int64_t occ = occupancy<FAST>(fp, s);
  int64_t *I = o.ints + p;
  float *F = o.flts + p;
  I[I_NTASKS * ld] = d.T;
  I[I_OCC * ld] = occ;
  I[I_WAVES * ld] = waves_of<FAST>(d.T, s.num_sms, occ);
  I[I_TOT_T * ld] = d.tot[0];
  I[I_TOT_F * ld] = d.tot[1];
  I[I_TOT_X * ld] = d.tot[2];
  I[I_MAX_T * ld] = d.mx[0];
  I[I_MAX_F * ld] = d.mx[1];
  I[I_MAX_X * ld] = d.mx[2];
  I[I_BYTES * ld] = d.tot[3];
  I[I_BYTES_MAX * ld] = d.mx[3];
  // Eq.5 and Eq.4 per pipe present
  double cg[3] = {0.0, 0.0, 0.0}, cs[3] = {0.0, 0.0, 0.0};
  if (pipes & 1) { cg[0] = (double)d.tot[0] * s.cg_tensor[tdt]; cs[0] = (double)d.mx[0] * s.cs_tensor[tdt]; }
  if (pipes & 2) { cg[1] = (double)d.tot[1] * s.cg_fma; cs[1] = (double)d.mx[1] * s.cs_fma; }
  if (pipes & 4) { cg[2] = (double)d.tot[2] * s.cg_xu; cs[2] = (double)d.mx[2] * s.cs_xu; }
  const double B = (double)d.tot[3], Bm = (double)d.mx[3];
  const double glob_g = B * s.glob_g, l2_g = B * s.l2_g;
  double roof = fmax(glob_g, l2_g);
  roof = fmax(roof, fmax(cg[0], fmax(cg[1], cg[2])));
  const float f[kNumFlts] = {(float)cg[0], (float)cg[1], (float)cg[2], (float)cs[0], (float)cs[1], (float)cs[2],
                             (float)glob_g, (float)l2_g, (float)(Bm * s.glob_s), (float)(Bm * s.l2_s),
                             (float)(Bm * s.smem_s), (float)(roof * s.inv_f)};
#pragma unroll
  for (int k = 0; k < kNumFlts; ++k) {
    F[k * ld] = f[k];
    if (fv) fv[k] = f[k];
  }
  o.status[p] = 0;
}

__device__ __forceinline__ void emit_error(const FeatOut &o, int64_t p, int status) {
  const int64_t ld = o.ld;
#pragma unroll
  for (int k = 0; k < kNumInts; ++k) o.ints[p + k * ld] = -1;
#pragma unroll
  for (int k = 0; k < kNumFlts; ++k) o.flts[p + k * ld] = __int_as_float(0x7fc00000);
  o.status[p] = (uint8_t)status;
}

}  // namespace sp
