// Predictor stage, tcgen05/TMEM path with 16-bit operands -- fp16 (default)
// or bf16 -- and fp32 accumulation (steps a10-a12, R17-R18).
//
// The MLP 256-128-64 is a chain of three GEMMs per tile of 128 pairs:
//   D1[128x256] = X [128x16]  . W1^T   (x in cols 0..n_in-1, col 15 = 1 carries b1)
//   D2[128x128] = H1[128x256] . W2'^T  (W2' = W2 diag(s1): BN1 folded, R18)
//   D3[128x64]  = H2[128x128] . W3'^T  (W3' = W3 diag(s2))
// issued by one thread as tcgen05.mma (M = 128, 16-bit in, fp32 accumulate in
// TMEM).  The folded BatchNorm shifts become biases (b2' = b2 + W2 t1, ...)
// that the epilogue writes into the D2/D3 accumulators (tcgen05.st) before the
// MMAs accumulate onto them, and the last BN goes into the output layer
// (w4' = w4 s3, b4' = b4 + w4.t3).  Each hidden epilogue is therefore only
// TMEM load -> cvt.rn.relu.{f16,bf16}x2 -> 16-byte st.shared, and the final
// 64 -> 1 layer is 64 FMAs per row on CUDA cores.
//
// CTA = 16 epilogue warps (4 warpgroups: 2 tile slots x 2 column halves) + 1
// MMA warp, persistent over tiles.  Weights (88 KB, UMMA no-swizzle K-major
// layout prepacked on the host) stay resident in shared memory; each slot owns
// 256 TMEM columns (D1, then D2/D3 reusing them) and 68 KB of activation
// buffers (X, then H1, with H2 aliasing H1).  The two slots interleave so the
// tensor pipe works on one tile while the other tile's epilogue runs.  The
// feature loads of a slot's next tile are issued one tile ahead.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "tcgen05.cuh"

namespace sp {
namespace {

constexpr int kTile = 128;
constexpr int kEpiWarps = 16;
constexpr int kThreads = (kEpiWarps + 1) * 32;
constexpr int kK1 = 16;  // n_in padded; column 15 is the constant-1 bias column

// Shared-memory image, bytes.  Operand layout (K-major, no swizzle):
//   off(r, k) = (r / 8) * SBO + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2,  SBO = 16 * K
constexpr uint32_t kW1Bytes = 256 * kK1 * 2;   //  8 KB
constexpr uint32_t kW2Bytes = 128 * 256 * 2;   // 64 KB
constexpr uint32_t kW3Bytes = 64 * 128 * 2;    // 16 KB
constexpr uint32_t kWBytes = kW1Bytes + kW2Bytes + kW3Bytes;
constexpr uint32_t kXBytes = kTile * kK1 * 2;  //  4 KB
constexpr uint32_t kHBytes = kTile * 256 * 2;  // 64 KB (H1; H2 = 32 KB aliases it)
constexpr uint32_t kSlotBytes = kXBytes + kHBytes;
// fp32 vectors: b2'[128] b3'[64] w4'[64] na[16] nc[16]  (x = log2(1+v) * na + nc)
constexpr int kVB2 = 0, kVB3 = 128, kVW4 = 192, kVNA = 256, kVNC = 272, kVecFloats = 288;
constexpr uint32_t kVecBytes = kVecFloats * 4;
constexpr uint32_t kOffW1 = 0, kOffW2 = kW1Bytes, kOffW3 = kW1Bytes + kW2Bytes;
constexpr uint32_t kOffSlot0 = kWBytes;
constexpr uint32_t kOffVec = kWBytes + 2 * kSlotBytes;
constexpr uint32_t kOffZx = kOffVec + kVecBytes;  // [2][128] fp32 partial logits
constexpr uint32_t kOffBar = kOffZx + 2 * kTile * 4;
constexpr uint32_t kSmemBytes = kOffBar + 64;
static_assert(kSmemBytes <= 232448, "shared memory budget");

__host__ __device__ constexpr uint32_t op_off(uint32_t r, uint32_t k, uint32_t K) {
  return (r / 8) * (16 * K) + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2;
}

// Table IV order (O8): per pipe present (Tensor, FMA, XU) [total ops, C^GPU,
// max-SM ops, C^SM], then the 7 MIO features.  Record slot, +16 for a float slot.
__host__ __device__ constexpr int in_slot(int fam, int k) {
  const int pipes = (fam == SP_GEMM || fam == SP_FUSED_MOE) ? 1 : (fam == SP_ATTENTION ? 5 : 6);
  int n = 0;
  for (int p = 0; p < 3; ++p) {
    if (!(pipes & (1 << p))) continue;
    if (k == n) return I_TOT_T + p;
    if (k == n + 1) return 16 + F_CG_T + p;
    if (k == n + 2) return I_MAX_T + p;
    if (k == n + 3) return 16 + F_CS_T + p;
    n += 4;
  }
  const int mio[7] = {I_BYTES, 16 + F_GLOB_G, 16 + F_L2_G, I_BYTES_MAX, 16 + F_GLOB_S, 16 + F_L2_S, 16 + F_SMEM_S};
  return k - n < 7 ? mio[k - n] : -1;
}
__host__ __device__ constexpr int n_in_of(int fam) { return (fam == SP_GEMM || fam == SP_FUSED_MOE) ? 11 : 15; }

struct Params {
  MlpBf16 m;
  sp_features in;
  float *latency;
  float *eff;
  int64_t n_tiles;
};

// Half a row's raw MLP inputs (features 8h..8h+7), loaded unconditionally
// (row index clamped) so the loads never wait on each other; int64 slots as
// raw bits, float slots in the low word.  Decoded at use time.
struct TileIn {
  uint64_t raw[8];
  float t_theory;
  uint32_t status;
  bool in_range;
};

template <int FAM>
__device__ __forceinline__ TileIn load_tile_in(const Params &P, int64_t t, uint32_t row, int h) {
  TileIn r;
  int64_t p = t * kTile + row;
  r.in_range = t < P.n_tiles && p < P.in.n_pairs;
  p = r.in_range ? p : 0;
  const int64_t ld = P.in.ld;
  const unsigned long long *ints = reinterpret_cast<const unsigned long long *>(P.in.ints);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    r.raw[i] = 0;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {  // h is warp-uniform; both variants are compile-time slots
      const int sl = in_slot(FAM, 8 * hh + i);
      if (hh == h && 8 * hh + i < n_in_of(FAM))
        r.raw[i] = sl >= 16 ? (uint64_t)__float_as_uint(__ldg(P.in.flts + (int64_t)(sl - 16) * ld + p))
                            : (uint64_t)__ldg(ints + (int64_t)sl * ld + p);
    }
  }
  r.t_theory = h == 0 ? __ldg(P.in.flts + (int64_t)F_TTHEORY * ld + p) : 0.f;
  r.status = __ldg(P.in.status + p);
  return r;
}

template <int FAM>
__device__ __forceinline__ float decode_in(const TileIn &r, int i, int h) {
  const int sl0 = in_slot(FAM, i), sl1 = in_slot(FAM, 8 + i);
  const bool is_f = h == 0 ? sl0 >= 16 : sl1 >= 16;
  return is_f ? __uint_as_float((uint32_t)r.raw[i]) : (float)(int64_t)r.raw[i];
}

// Hidden epilogue: TMEM columns [c_begin, c_begin + NC) of this lane's row ->
// ReLU -> 16-bit -> next operand (K = KN) columns [c_begin, ...) in shared memory.
template <int NC, int KN, bool BF16>
__device__ __forceinline__ void epi_hidden(uint32_t tmem_row, uint32_t c_begin, uint32_t dst, uint32_t row) {
#pragma unroll 1
  for (int c00 = 0; c00 < NC; c00 += 64) {
    uint32_t vv[2][32];  // two TMEM loads in flight per wait
    tc::tmem_ld32(tmem_row + c_begin + c00, vv[0]);
    tc::tmem_ld32(tmem_row + c_begin + c00 + 32, vv[1]);
    tc::tmem_wait_ld();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // 4 chunks of 8 columns = 16 bytes
        const uint32_t *v = vv[h] + q * 8;
        tc::st_shared_v4(dst + op_off(row, c_begin + c00 + 32 * h + q * 8, KN),
                         tc::relu_x2<BF16>(__uint_as_float(v[0]), __uint_as_float(v[1])),
                         tc::relu_x2<BF16>(__uint_as_float(v[2]), __uint_as_float(v[3])),
                         tc::relu_x2<BF16>(__uint_as_float(v[4]), __uint_as_float(v[5])),
                         tc::relu_x2<BF16>(__uint_as_float(v[6]), __uint_as_float(v[7])));
      }
    }
  }
}

// Write a bias vector (broadcast over rows) into TMEM columns [c, c + NC).
template <int NC>
__device__ __forceinline__ void bias_to_tmem(uint32_t tmem_row, uint32_t c, const float *bias) {
#pragma unroll 1
  for (int c0 = 0; c0 < NC; c0 += 32) {
    uint32_t v[32];
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      const float4 b = *reinterpret_cast<const float4 *>(bias + c0 + j);
      v[j] = __float_as_uint(b.x);
      v[j + 1] = __float_as_uint(b.y);
      v[j + 2] = __float_as_uint(b.z);
      v[j + 3] = __float_as_uint(b.w);
    }
    tc::tmem_st32(tmem_row + c + c0, v);
  }
}

template <bool BF16, int FAM>
__global__ void __launch_bounds__(kThreads, 1) predict_tcgen05_kernel(Params P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sbase = tc::smem_u32(smem);
  float *vec = reinterpret_cast<float *>(smem + kOffVec);
  float *zx = reinterpret_cast<float *>(smem + kOffZx);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kOffBar);  // a_full[2], d_full[2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + kOffBar + 32);
  const uint32_t bar_a[2] = {tc::smem_u32(bars + 0), tc::smem_u32(bars + 1)};
  const uint32_t bar_d[2] = {tc::smem_u32(bars + 2), tc::smem_u32(bars + 3)};

  // ---- one-time setup: weights + vectors to smem, barriers, TMEM
  {
    const uint4 *src = reinterpret_cast<const uint4 *>(P.m.wpack);
    uint4 *dst = reinterpret_cast<uint4 *>(smem);
    for (int i = threadIdx.x; i < (int)(kWBytes / 16); i += kThreads) dst[i] = __ldg(src + i);
    for (int i = threadIdx.x; i < kVecFloats; i += kThreads) vec[i] = __ldg(P.m.vecs + i);
  }
  if (threadIdx.x == 0) {
    tc::mbar_init(bar_a[0], 256);
    tc::mbar_init(bar_a[1], 256);
    tc::mbar_init(bar_d[0], 1);
    tc::mbar_init(bar_d[1], 1);
    tc::mbar_init_fence();
  }
  if (warp == kEpiWarps) tc::tmem_alloc<512>(tc::smem_u32(tmem_slot));
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  const int64_t G = gridDim.x;
  if (warp == kEpiWarps) {
    // ================= MMA issuer (one thread) =================
    if (lane == 0) {
      const uint32_t i1 = tc::idesc_f16kind_f32(128, 256, BF16), i2 = tc::idesc_f16kind_f32(128, 128, BF16),
                     i3 = tc::idesc_f16kind_f32(128, 64, BF16);
      uint32_t pa[2] = {0, 0};
      for (int64_t k = 0;; k += 2) {
        const int64_t t0 = blockIdx.x + k * G;
        if (t0 >= P.n_tiles) break;
        const int nslots = (t0 + G < P.n_tiles) ? 2 : 1;
        for (int layer = 0; layer < 3; ++layer) {
          for (int s = 0; s < nslots; ++s) {
            const uint32_t slot = sbase + kOffSlot0 + s * kSlotBytes;
            const uint32_t dcol = tmem + (uint32_t)(s * 256);
            tc::mbar_wait(bar_a[s], pa[s]);
            pa[s] ^= 1;
            tc::fence_after();
            if (layer == 0) {  // bias b1 rides on X's constant-1 column: no accumulate
              tc::mma_f16kind(dcol, tc::smem_desc(slot, 128, 16 * kK1), tc::smem_desc(sbase + kOffW1, 128, 16 * kK1),
                              i1, 0);
            } else if (layer == 1) {  // D2 was preset to b2' by the epilogue: accumulate onto it
#pragma unroll
              for (int ks = 0; ks < 256 / 16; ++ks)
                tc::mma_f16kind(dcol, tc::smem_desc(slot + kXBytes + ks * 256, 128, 16 * 256),
                                tc::smem_desc(sbase + kOffW2 + ks * 256, 128, 16 * 256), i2, 1);
            } else {
#pragma unroll
              for (int ks = 0; ks < 128 / 16; ++ks)
                tc::mma_f16kind(dcol + 128, tc::smem_desc(slot + kXBytes + ks * 256, 128, 16 * 128),
                                tc::smem_desc(sbase + kOffW3 + ks * 256, 128, 16 * 128), i3, 1);
            }
            tc::commit(bar_d[s]);
          }
        }
      }
    }
  } else {
    // ================= epilogue warpgroups =================
    const int grp = warp >> 2;                    // 0..3
    const int s = grp >> 1, h = grp & 1;          // tile slot, column half
    const uint32_t row = (warp & 3) * 32 + lane;  // TMEM lane == tile row
    const uint32_t tmem_row = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(s * 256);
    const uint32_t xbuf = sbase + kOffSlot0 + s * kSlotBytes, hbuf = xbuf + kXBytes;
    const float *na = vec + kVNA, *nc = vec + kVNC, *w4 = vec + kVW4;
    const int64_t n_pairs = P.in.n_pairs;
    uint32_t pd = 0;
    TileIn cur = load_tile_in<FAM>(P, blockIdx.x + (int64_t)s * G, row, h);
    for (int64_t k = s;; k += 2) {
      const int64_t t = blockIdx.x + k * G;
      if (t >= P.n_tiles) break;
      const int64_t p = t * kTile + row;
      const bool valid = cur.in_range && cur.status == 0;
      const float t_theory = cur.t_theory;
      // a10: x = (ln(1+v) - mu) / sigma = log2(1+v) * (ln2/sigma) - mu/sigma;
      // this half writes X columns 8h..8h+7 (column 15 = 1 for the bias b1).
      float x[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int j = 8 * h + i;
        x[i] = j == 15 ? 1.f
                       : ((valid && j < n_in_of(FAM)) ? fmaf(__log2f(1.f + decode_in<FAM>(cur, i, h)), na[j], nc[j]) : 0.f);
      }
      cur = load_tile_in<FAM>(P, t + 2 * G, row, h);  // prefetch this slot's next tile
      tc::st_shared_v4(xbuf + op_off(row, 8 * h, kK1), tc::pack_x2<BF16>(x[0], x[1]), tc::pack_x2<BF16>(x[2], x[3]),
                       tc::pack_x2<BF16>(x[4], x[5]), tc::pack_x2<BF16>(x[6], x[7]));
      tc::fence_proxy_async();
      tc::mbar_arrive(bar_a[s]);
      // layer 1: D1 cols [128h, 128h+128) -> H1; then preset the next accumulators:
      // half 0 read D1[0,128) and presets D2 = b2' there; half 1 read D1[128,256)
      // and presets D3 = b3' in [128,192).
      tc::mbar_wait(bar_d[s], pd);
      pd ^= 1;
      tc::fence_after();
      epi_hidden<128, 256, BF16>(tmem_row, 128 * h, hbuf, row);
      if (h == 0) bias_to_tmem<128>(tmem_row, 0, vec + kVB2);
      else bias_to_tmem<64>(tmem_row, 128, vec + kVB3);
      tc::tmem_wait_st();
      tc::fence_before();
      tc::fence_proxy_async();
      tc::mbar_arrive(bar_a[s]);
      // layer 2: D2 cols [64h, 64h+64) -> H2 (aliases H1)
      tc::mbar_wait(bar_d[s], pd);
      pd ^= 1;
      tc::fence_after();
      epi_hidden<64, 128, BF16>(tmem_row, 64 * h, hbuf, row);
      tc::fence_before();
      tc::fence_proxy_async();
      tc::mbar_arrive(bar_a[s]);
      // layer 3 + output layer: z = b4' + sum_j w4'_j relu(D3_j); this half sums 32 columns
      tc::mbar_wait(bar_d[s], pd);
      pd ^= 1;
      tc::fence_after();
      float zp;
      {
        uint32_t v[32];
        tc::tmem_ld32(tmem_row + 128 + 32 * h, v);
        tc::tmem_wait_ld();
        float zz[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const float4 w = *reinterpret_cast<const float4 *>(w4 + 32 * h + j);
          zz[0] = fmaf(w.x, fmaxf(__uint_as_float(v[j + 0]), 0.f), zz[0]);
          zz[1] = fmaf(w.y, fmaxf(__uint_as_float(v[j + 1]), 0.f), zz[1]);
          zz[2] = fmaf(w.z, fmaxf(__uint_as_float(v[j + 2]), 0.f), zz[2]);
          zz[3] = fmaf(w.w, fmaxf(__uint_as_float(v[j + 3]), 0.f), zz[3]);
        }
        zp = (zz[0] + zz[1]) + (zz[2] + zz[3]);
      }
      tc::fence_before();
      if (h == 1) zx[s * kTile + row] = zp;
      asm volatile("bar.sync %0, 256;" ::"r"(1 + s) : "memory");  // the slot's two halves
      if (h == 0 && p < n_pairs) {
        const float z = P.m.b4 + zp + zx[s * kTile + row];
        float lat, e;
        if (!valid) {
          lat = e = __int_as_float(0x7fc00000);
        } else {
          const float ez = __expf(-z);
          e = 1.f / (1.f + ez);
          lat = t_theory * (1.f + ez);
        }
        P.latency[p] = lat;
        if (P.eff) P.eff[p] = e;
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == kEpiWarps) {
    tc::fence_after();
    tc::tmem_dealloc<512>(tmem);
  }
}

}  // namespace

// ---------------------------------------------------------------- host side

// fp64 -> 16-bit operand bits, round to nearest even.
static uint16_t to_bits16(double v, bool bf16) {
  uint16_t u;
  if (bf16) {
    __nv_bfloat16 h = __double2bfloat16(v);
    std::memcpy(&u, &h, 2);
  } else {
    __half h = __double2half(v);
    std::memcpy(&u, &h, 2);
  }
  return u;
}

bool pack_mlp_16bit(const sp_mlp_desc &d, const std::vector<double> *s, const std::vector<double> *t, bool bf16,
                    std::vector<uint16_t> &wpack, std::vector<float> &vecs, float &b4) {
  const int n_in = d.n_in;
  if (n_in > kK1 - 1) return false;  // column 15 carries the bias
  wpack.assign(kWBytes / 2, 0);
  auto put = [&](uint32_t base, uint32_t r, uint32_t k, uint32_t K, double v) {
    wpack[(base + op_off(r, k, K)) / 2] = to_bits16(v, bf16);
  };
  for (int n = 0; n < 256; ++n) {
    for (int k = 0; k < n_in; ++k) put(kOffW1, n, k, kK1, d.w1[n * n_in + k]);
    put(kOffW1, n, kK1 - 1, kK1, d.b1[n]);  // x[15] = 1
  }
  // W2' = W2 diag(s1), W3' = W3 diag(s2)  (BN folded into the next layer, R18)
  for (int n = 0; n < 128; ++n)
    for (int k = 0; k < 256; ++k) put(kOffW2, n, k, 256, (double)d.w2[n * 256 + k] * s[0][k]);
  for (int n = 0; n < 64; ++n)
    for (int k = 0; k < 128; ++k) put(kOffW3, n, k, 128, (double)d.w3[n * 128 + k] * s[1][k]);
  vecs.assign(kVecFloats, 0.f);
  for (int n = 0; n < 128; ++n) {
    double acc = d.b2[n];
    for (int k = 0; k < 256; ++k) acc += (double)d.w2[n * 256 + k] * t[0][k];
    vecs[kVB2 + n] = (float)acc;
  }
  for (int n = 0; n < 64; ++n) {
    double acc = d.b3[n];
    for (int k = 0; k < 128; ++k) acc += (double)d.w3[n * 128 + k] * t[1][k];
    vecs[kVB3 + n] = (float)acc;
  }
  double bb = d.b4;
  for (int k = 0; k < 64; ++k) {
    vecs[kVW4 + k] = (float)((double)d.w4[k] * s[2][k]);
    bb += (double)d.w4[k] * t[2][k];
  }
  // x_k = (ln(1+v) - mu_k) / sigma_k = log2(1+v) * (ln2 / sigma_k) - mu_k / sigma_k  (R17)
  for (int k = 0; k < n_in; ++k) {
    const double sg = std::fmax((double)d.sigma[k], 1e-8);
    vecs[kVNA + k] = (float)(0.69314718055994530942 / sg);
    vecs[kVNC + k] = (float)(-(double)d.mu[k] / sg);
  }
  b4 = (float)bb;
  return true;
}

template <bool BF16>
static cudaError_t launch_fam(int fam, const Params &P, unsigned grid, cudaStream_t st) {
  void (*kern)(Params) = nullptr;
  switch (fam) {
    case SP_GEMM: kern = predict_tcgen05_kernel<BF16, SP_GEMM>; break;
    case SP_ATTENTION: kern = predict_tcgen05_kernel<BF16, SP_ATTENTION>; break;
    case SP_FUSED_MOE: kern = predict_tcgen05_kernel<BF16, SP_FUSED_MOE>; break;
    case SP_RMSNORM: kern = predict_tcgen05_kernel<BF16, SP_RMSNORM>; break;
    default: kern = predict_tcgen05_kernel<BF16, SP_SILU_MUL>; break;
  }
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreads, kSmemBytes, st>>>(P);
  return cudaGetLastError();
}

int launch_predict_tcgen05(const MlpBf16 &m, const sp_features &in, float *latency, float *eff,
                           int num_device_sms, void *stream) {
  if (in.n_pairs == 0) return 0;
  Params P;
  P.m = m;
  P.in = in;
  P.latency = latency;
  P.eff = eff;
  P.n_tiles = (in.n_pairs + kTile - 1) / kTile;
  const int64_t grid = P.n_tiles < num_device_sms ? P.n_tiles : num_device_sms;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return (int)(m.bf16 ? launch_fam<true>(m.family, P, (unsigned)grid, st)
                      : launch_fam<false>(m.family, P, (unsigned)grid, st));
}

}  // namespace sp
