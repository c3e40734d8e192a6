// Predictor stage, tcgen05/TMEM path with 16-bit operands -- fp16 (default,
// parity ~3e-3) or bf16 (parity ~1e-2) -- and fp32 accumulation (steps
// a10-a12, R17-R18).
//
// The MLP 256-128-64 is a chain of three GEMMs per tile of 128 pairs:
//   D1[128x256] = X [128x16]  . W1^T   (K = n_in padded to 16)
//   D2[128x128] = H1[128x256] . W2'^T  (W2' = W2 diag(s1): BN1 folded, R18)
//   D3[128x64]  = H2[128x128] . W3'^T  (W3' = W3 diag(s2))
// issued by one thread as tcgen05.mma (M = 128, bf16 in, fp32 accumulate in
// TMEM).  The folded BatchNorm shifts become biases (b2' = b2 + W2 t1, ...)
// and the last BN goes into the output layer (w4' = w4 s3, b4' = b4 + w4.t3),
// so every epilogue is bias + ReLU + bf16 pack (one cvt.rn.relu.bf16x2 per
// two values), and the final 64 -> 1 layer is 64 FMAs per row on CUDA cores.
//
// CTA = 8 epilogue warps (two warpgroups, one per tile slot) + 1 MMA warp,
// persistent over tiles.  Weights (bf16, 88 KB, UMMA no-swizzle K-major
// layout prepacked on the host) stay resident in shared memory; each slot owns
// 256 TMEM columns (D1, then D2/D3 reusing them) and 68 KB of activation
// buffers (X, then H1, with H2 aliasing H1).  The two slots interleave so the
// tensor pipe works on one tile while the other tile's epilogue runs.
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
constexpr int kEpiWarps = 8;
constexpr int kThreads = (kEpiWarps + 1) * 32;
constexpr int kK1 = 16;  // n_in padded

// Shared-memory image, bytes.  Operand layout (K-major, no swizzle):
//   off(r, k) = (r / 8) * SBO + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2,  SBO = 16 * K
constexpr uint32_t kW1Bytes = 256 * kK1 * 2;   //  8 KB
constexpr uint32_t kW2Bytes = 128 * 256 * 2;   // 64 KB
constexpr uint32_t kW3Bytes = 64 * 128 * 2;    // 16 KB
constexpr uint32_t kWBytes = kW1Bytes + kW2Bytes + kW3Bytes;
constexpr uint32_t kXBytes = kTile * kK1 * 2;  //  4 KB
constexpr uint32_t kHBytes = kTile * 256 * 2;  // 64 KB (H1; H2 = 32 KB aliases it)
constexpr uint32_t kSlotBytes = kXBytes + kHBytes;
// fp32 vectors: b1[256] b2'[128] b3'[64] w4'[64] mu[16] inv_sigma[16]
constexpr int kVecFloats = 256 + 128 + 64 + 64 + 16 + 16;
constexpr uint32_t kVecBytes = kVecFloats * 4;
constexpr uint32_t kOffW1 = 0, kOffW2 = kW1Bytes, kOffW3 = kW1Bytes + kW2Bytes;
constexpr uint32_t kOffSlot0 = kWBytes;
constexpr uint32_t kOffVec = kWBytes + 2 * kSlotBytes;
constexpr uint32_t kOffBar = kOffVec + kVecBytes;
constexpr uint32_t kSmemBytes = kOffBar + 64;
static_assert(kSmemBytes <= 232448, "shared memory budget");

__host__ __device__ constexpr uint32_t op_off(uint32_t r, uint32_t k, uint32_t K) {
  return (r / 8) * (16 * K) + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2;
}

// Table IV order (O8): per pipe present (Tensor, FMA, XU) [total ops, C^GPU,
// max-SM ops, C^SM], then the 7 MIO features.  Record slot, +16 for a float slot.
static int feature_slot_host(int pipes, int k) {
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
  return mio[k - n];
}

struct Params {
  MlpBf16 m;
  sp_features in;
  float *latency;
  float *eff;
  int64_t n_tiles;
  int32_t n_in;
  int32_t slot[kK1];  // Table IV order (O8): feature j -> record slot; +16 marks a float slot
};

// One row's raw MLP inputs (features as fp32), validity and t_theory.
struct TileIn {
  float v[kK1];
  float t_theory;
  bool valid;
};

__device__ __forceinline__ TileIn load_tile_in(const Params &P, int64_t t, uint32_t row) {
  TileIn r;
  const int64_t p = t * kTile + row;
  r.valid = t < P.n_tiles && p < P.in.n_pairs && P.in.status[p] == 0;
  const int64_t ld = P.in.ld;
#pragma unroll
  for (int j = 0; j < kK1; ++j) {
    r.v[j] = 0.f;
    if (r.valid && j < P.n_in) {
      const int sl = P.slot[j];
      r.v[j] = sl >= 16 ? __ldg(P.in.flts + (int64_t)(sl - 16) * ld + p) : (float)__ldg(P.in.ints + (int64_t)sl * ld + p);
    }
  }
  r.t_theory = r.valid ? __ldg(P.in.flts + (int64_t)F_TTHEORY * ld + p) : 0.f;
  return r;
}

// Epilogue of one hidden layer: rows of D (TMEM columns [col0, col0+ncols))
// + bias, ReLU, 16-bit -> next operand (K = ncols) in shared memory.
template <int NCOLS, bool BF16>
__device__ __forceinline__ void epi_hidden(uint32_t tmem_row, uint32_t col0, const float *bias, uint32_t dst,
                                           uint32_t row) {
#pragma unroll 1
  for (int c0 = 0; c0 < NCOLS; c0 += 32) {
    uint32_t v[32];
    tc::tmem_ld32(tmem_row + col0 + c0, v);
    tc::tmem_wait_ld();
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // 4 chunks of 8 columns = 16 bytes
      const float4 b0 = *reinterpret_cast<const float4 *>(bias + c0 + q * 8);
      const float4 b1 = *reinterpret_cast<const float4 *>(bias + c0 + q * 8 + 4);
      const uint32_t w0 = tc::relu_x2<BF16>(__uint_as_float(v[q * 8 + 0]) + b0.x, __uint_as_float(v[q * 8 + 1]) + b0.y);
      const uint32_t w1 = tc::relu_x2<BF16>(__uint_as_float(v[q * 8 + 2]) + b0.z, __uint_as_float(v[q * 8 + 3]) + b0.w);
      const uint32_t w2 = tc::relu_x2<BF16>(__uint_as_float(v[q * 8 + 4]) + b1.x, __uint_as_float(v[q * 8 + 5]) + b1.y);
      const uint32_t w3 = tc::relu_x2<BF16>(__uint_as_float(v[q * 8 + 6]) + b1.z, __uint_as_float(v[q * 8 + 7]) + b1.w);
      tc::st_shared_v4(dst + op_off(row, c0 + q * 8, NCOLS), w0, w1, w2, w3);
    }
  }
}

template <bool BF16>
__global__ void __launch_bounds__(kThreads, 1) predict_tcgen05_kernel(Params P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sbase = tc::smem_u32(smem);
  float *vec = reinterpret_cast<float *>(smem + kOffVec);
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
    tc::mbar_init(bar_a[0], 128);
    tc::mbar_init(bar_a[1], 128);
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
            if (layer == 0) {
              tc::mma_bf16(dcol, tc::smem_desc(slot, 128, 16 * kK1), tc::smem_desc(sbase + kOffW1, 128, 16 * kK1),
                           i1, 0);
            } else if (layer == 1) {
#pragma unroll
              for (int ks = 0; ks < 256 / 16; ++ks)
                tc::mma_bf16(dcol, tc::smem_desc(slot + kXBytes + ks * 256, 128, 16 * 256),
                             tc::smem_desc(sbase + kOffW2 + ks * 256, 128, 16 * 256), i2, ks > 0);
            } else {
#pragma unroll
              for (int ks = 0; ks < 128 / 16; ++ks)
                tc::mma_bf16(dcol + 128, tc::smem_desc(slot + kXBytes + ks * 256, 128, 16 * 128),
                             tc::smem_desc(sbase + kOffW3 + ks * 256, 128, 16 * 128), i3, ks > 0);
            }
            tc::commit(bar_d[s]);
          }
        }
      }
    }
  } else {
    // ================= epilogue warpgroups =================
    const int s = warp >> 2;                  // slot
    const uint32_t row = (warp & 3) * 32 + lane;  // TMEM lane == tile row
    const uint32_t tmem_row = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(s * 256);
    const uint32_t slot = sbase + kOffSlot0 + s * kSlotBytes;
    const uint32_t xbuf = slot, hbuf = slot + kXBytes;
    const float *b1 = vec, *b2 = vec + 256, *b3 = vec + 384, *w4 = vec + 448, *na = vec + 512,
                *nc = vec + 528;
    const int64_t n_pairs = P.in.n_pairs;
    uint32_t pd = 0;
    // Inputs of this slot's next tile are loaded one tile ahead, so their HBM
    // latency hides behind the current tile's epilogues.
    TileIn cur = load_tile_in(P, blockIdx.x + (int64_t)s * G, row);
    for (int64_t k = s;; k += 2) {
      const int64_t t = blockIdx.x + k * G;
      if (t >= P.n_tiles) break;
      const int64_t p = t * kTile + row;
      const bool valid = cur.valid;
      const float t_theory = cur.t_theory;
      // a10: x = (ln(1+v) - mu) / sigma = log2(1+v) * (ln2/sigma) - mu/sigma, K padded to 16
      float x[kK1];
#pragma unroll
      for (int j = 0; j < kK1; ++j)
        x[j] = (valid && j < P.n_in) ? fmaf(__log2f(1.f + cur.v[j]), na[j], nc[j]) : 0.f;
      cur = load_tile_in(P, t + 2 * G, row);  // prefetch
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        uint32_t w[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) w[h] = tc::pack_x2<BF16>(x[q * 8 + 2 * h], x[q * 8 + 2 * h + 1]);
        tc::st_shared_v4(xbuf + op_off(row, q * 8, kK1), w[0], w[1], w[2], w[3]);
      }
      tc::fence_proxy_async();
      tc::mbar_arrive(bar_a[s]);
      // layer 1 epilogue: D1 (256 cols) -> H1
      tc::mbar_wait(bar_d[s], pd);
      pd ^= 1;
      tc::fence_after();
      epi_hidden<256, BF16>(tmem_row, 0, b1, hbuf, row);
      tc::fence_before();
      tc::fence_proxy_async();
      tc::mbar_arrive(bar_a[s]);
      // layer 2 epilogue: D2 (cols 0..127) -> H2 (aliases H1)
      tc::mbar_wait(bar_d[s], pd);
      pd ^= 1;
      tc::fence_after();
      epi_hidden<128, BF16>(tmem_row, 0, b2, hbuf, row);
      tc::fence_before();
      tc::fence_proxy_async();
      tc::mbar_arrive(bar_a[s]);
      // layer 3 epilogue + output layer: z = w4'.relu(D3 + b3') + b4'
      tc::mbar_wait(bar_d[s], pd);
      pd ^= 1;
      tc::fence_after();
      float z = P.m.b4;
#pragma unroll 1
      for (int c0 = 0; c0 < 64; c0 += 32) {
        uint32_t v[32];
        tc::tmem_ld32(tmem_row + 128 + c0, v);
        tc::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const float4 w = *reinterpret_cast<const float4 *>(w4 + c0 + j);
          const float4 bb = *reinterpret_cast<const float4 *>(b3 + c0 + j);
          z = fmaf(w.x, fmaxf(__uint_as_float(v[j + 0]) + bb.x, 0.f), z);
          z = fmaf(w.y, fmaxf(__uint_as_float(v[j + 1]) + bb.y, 0.f), z);
          z = fmaf(w.z, fmaxf(__uint_as_float(v[j + 2]) + bb.z, 0.f), z);
          z = fmaf(w.w, fmaxf(__uint_as_float(v[j + 3]) + bb.w, 0.f), z);
        }
      }
      tc::fence_before();
      if (p < n_pairs) {
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

// fp64 -> 16-bit operand bits, round to nearest even (via fp32 for the bf16 case:
// the double-rounding window is far below the bf16 ulp of these weights).
static uint16_t to_bits16(double v, bool bf16) {
  if (bf16) {
    __nv_bfloat16 h = __float2bfloat16_rn((float)v);
    uint16_t u;
    std::memcpy(&u, &h, 2);
    return u;
  }
  __half h = __double2half(v);
  uint16_t u;
  std::memcpy(&u, &h, 2);
  return u;
}

bool pack_mlp_16bit(const sp_mlp_desc &d, const std::vector<double> *s, const std::vector<double> *t, bool bf16,
                    std::vector<uint16_t> &wpack, std::vector<float> &vecs, float &b4) {
  const int n_in = d.n_in;
  if (n_in > kK1) return false;
  wpack.assign(kWBytes / 2, 0);
  auto put = [&](uint32_t base, uint32_t r, uint32_t k, uint32_t K, double v) {
    wpack[(base + op_off(r, k, K)) / 2] = to_bits16(v, bf16);
  };
  for (int n = 0; n < 256; ++n)
    for (int k = 0; k < n_in; ++k) put(kOffW1, n, k, kK1, d.w1[n * n_in + k]);
  // W2' = W2 diag(s1), W3' = W3 diag(s2)  (BN folded into the next layer, R18)
  for (int n = 0; n < 128; ++n)
    for (int k = 0; k < 256; ++k) put(kOffW2, n, k, 256, (double)d.w2[n * 256 + k] * s[0][k]);
  for (int n = 0; n < 64; ++n)
    for (int k = 0; k < 128; ++k) put(kOffW3, n, k, 128, (double)d.w3[n * 128 + k] * s[1][k]);
  vecs.assign(kVecFloats, 0.f);
  for (int n = 0; n < 256; ++n) vecs[n] = d.b1[n];
  for (int n = 0; n < 128; ++n) {
    double acc = d.b2[n];
    for (int k = 0; k < 256; ++k) acc += (double)d.w2[n * 256 + k] * t[0][k];
    vecs[256 + n] = (float)acc;
  }
  for (int n = 0; n < 64; ++n) {
    double acc = d.b3[n];
    for (int k = 0; k < 128; ++k) acc += (double)d.w3[n * 128 + k] * t[1][k];
    vecs[384 + n] = (float)acc;
  }
  double bb = d.b4;
  for (int k = 0; k < 64; ++k) {
    vecs[448 + k] = (float)((double)d.w4[k] * s[2][k]);
    bb += (double)d.w4[k] * t[2][k];
  }
  // x_k = (ln(1+v) - mu_k) / sigma_k = log2(1+v) * (ln2 / sigma_k) - mu_k / sigma_k  (R17)
  for (int k = 0; k < n_in; ++k) {
    const double sg = std::fmax((double)d.sigma[k], 1e-8);
    vecs[512 + k] = (float)(0.69314718055994530942 / sg);
    vecs[528 + k] = (float)(-(double)d.mu[k] / sg);
  }
  b4 = (float)bb;
  return true;
}

int launch_predict_tcgen05(const MlpBf16 &m, const sp_features &in, float *latency, float *eff,
                           int num_device_sms, void *stream) {
  if (in.n_pairs == 0) return 0;
  auto kern = m.bf16 ? predict_tcgen05_kernel<true> : predict_tcgen05_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
  if (e != cudaSuccess) return (int)e;
  Params P;
  P.m = m;
  P.in = in;
  P.latency = latency;
  P.eff = eff;
  P.n_tiles = (in.n_pairs + kTile - 1) / kTile;
  P.n_in = m.n_in;
  for (int j = 0; j < kK1; ++j) P.slot[j] = j < m.n_in ? feature_slot_host(family_pipes(m.family), j) : 0;
  const int64_t grid = P.n_tiles < num_device_sms ? P.n_tiles : num_device_sms;
  kern<<<(unsigned)grid, kThreads, kSmemBytes, reinterpret_cast<cudaStream_t>(stream)>>>(P);
  return (int)cudaGetLastError();
}

}  // namespace sp
