// Estimator training on the GPU (PAPER §V-C, §VII-A; SURVEY
// §8(f) NEXT-4): one minibatch step of the per-category MLP -- gather and
// normalise the minibatch's Table IV vectors and efficiency targets from the
// feature records, train-mode forward (Linear -> ReLU -> batch-statistics
// BatchNorm -> inverted Dropout, sigmoid output), MAPE or pinball loss,
// backward, running statistics, AdamW.  Readings T1..T9 in DESIGN.md §3c.
//
// fp32 on CUDA cores.  The work per step is small (B x ~44k MAC forward, twice
// that backward) and a chain of dependent stages; every reduction runs in a
// fixed order, so steps are deterministic:
//   gather | 3 x (sgemm, bn_stats, bn_apply) | out_fwd + out_red |
//   3 x (bn_bwd_stats + bn_bwd_apply, dW sgemm [+ split-K reduce], dX sgemm) | adamw
// BatchNorm kernels split the batch rows into up to 64 chunks (grid columns/32
// x chunks; per-chunk partial sums merged in chunk order by the consumer), and
// GEMMs whose tile grid would not fill the GPU -- the dW products, K = batch
// rows -- are split along K into slices summed in order.  GEMMs are 64x64x16
// shared-memory tiles, 4x4 outputs per thread.  tcgen05 would need TF32
// operands; at these sizes the step is latency-bound, not tensor-bound.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <new>
#include <vector>

#include "ctx.h"

using namespace sp;

namespace {

constexpr int kHid[3] = {256, 128, 64};
constexpr int kColThreadsX = 32, kColThreadsY = 16;
constexpr int kGemmT = 64, kGemmK = 16;

// ------------------------------------------------------------------ dropout generator (T3)

__device__ __forceinline__ uint64_t splitmix_fin(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

struct DropParams {
  uint64_t seed;
  const int64_t *step;  // DEVICE step counter (so a captured step graph replays correctly)
  uint32_t thr;  // keep iff bits 63..40 >= thr = round(p * 2^24)
  float scale;   // 1 / (1 - p)
};

__device__ __forceinline__ bool keep_unit(const DropParams &d, int layer, int64_t row, int col) {
  const uint64_t ctr = (((((uint64_t)(*d.step) * 4u + (uint64_t)layer) << 20) + (uint64_t)row) << 8) + (uint64_t)col;
  return (uint32_t)(splitmix_fin(d.seed + ctr * 0x9E3779B97F4A7C15ULL) >> 40) >= d.thr;
}

// ------------------------------------------------------------------ minibatch gather (O8-O9, P:489 target)

// Table IV order (O8), slot | (is_float << 8).
__device__ __forceinline__ int feature_slot(int pipes, int k) {
  int n = 0;
  for (int p = 0; p < 3; ++p) {
    if (!(pipes & (1 << p))) continue;
    if (k == n) return I_TOT_T + p;
    if (k == n + 1) return (F_CG_T + p) | 256;
    if (k == n + 2) return I_MAX_T + p;
    if (k == n + 3) return (F_CS_T + p) | 256;
    n += 4;
  }
  const int mio[7] = {I_BYTES, F_GLOB_G | 256, F_L2_G | 256, I_BYTES_MAX, F_GLOB_S | 256,
                      F_L2_S | 256, F_SMEM_S | 256};
  return mio[k - n];
}

// x[r][k] = (ln(1 + v) - mu_k) / max(sigma_k, 1e-8) in fp64, rounded once (R17);
// t[r] = t_theory / measured in fp32 (P:489's efficiency).
__global__ void train_gather(sp_features f, int pipes, int n_in, const float *__restrict__ mu,
                             const float *__restrict__ sigma, const float *__restrict__ measured,
                             const int64_t *__restrict__ idx, int64_t B, float *__restrict__ x,
                             float *__restrict__ t) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * (n_in + 1)) return;
  const int64_t r = i / (n_in + 1);
  const int k = (int)(i - r * (n_in + 1));
  const int64_t p = __ldg(idx + r);
  if (k == n_in) {
    t[r] = __fdiv_rn(__ldg(f.flts + (int64_t)F_TTHEORY * f.ld + p), __ldg(measured + p));
    return;
  }
  const int s = feature_slot(pipes, k);
  const double v = (s & 256) ? (double)__ldg(f.flts + (int64_t)(s & 255) * f.ld + p)
                             : (double)__ldg(f.ints + (int64_t)s * f.ld + p);
  x[r * n_in + k] = (float)((log1p(v) - (double)mu[k]) / fmax((double)sigma[k], 1e-8));
}

// ------------------------------------------------------------------ SGEMM

// C[M][N] (row-major, ldc = N) = sum_k A(m,k) B(k,n) (+ bias[n]), with
// A(m,k) = A[m*sam + k*sak], B(k,n) = B[k*sbk + n*sbn].  k summed in order.
__global__ void __launch_bounds__(256) train_sgemm(int M, int N, int K, const float *__restrict__ A,
                                                   int64_t sam, int64_t sak, const float *__restrict__ Bm,
                                                   int64_t sbk, int64_t sbn, const float *bias, float *C) {
  __shared__ float As[kGemmK][kGemmT + 4];
  __shared__ float Bs[kGemmK][kGemmT + 4];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * kGemmT, n0 = blockIdx.x * kGemmT;
  // split-K: slice blockIdx.z covers k in [kb, ke) and writes its own partial C
  const int kslice = (K + (int)gridDim.z - 1) / (int)gridDim.z;
  const int kb = (int)blockIdx.z * kslice, ke = min(K, kb + kslice);
  if (gridDim.z > 1) {
    C += (int64_t)blockIdx.z * M * N;
    bias = nullptr;
  }
  float acc[4][4] = {};
  for (int k0 = kb; k0 < ke; k0 += kGemmK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + i * 256;
      // contiguous-k operands read 16 consecutive k per row; otherwise 64 consecutive rows
      const int am = sak == 1 ? e >> 4 : e & 63, ak = sak == 1 ? e & 15 : e >> 6;
      const int bn = sbk == 1 ? e >> 4 : e & 63, bk = sbk == 1 ? e & 15 : e >> 6;
      const int gm = m0 + am, gk = k0 + ak, gn = n0 + bn, gk2 = k0 + bk;
      As[ak][am] = (gm < M && gk < ke) ? __ldg(A + gm * sam + gk * sak) : 0.f;
      Bs[bk][bn] = (gn < N && gk2 < ke) ? __ldg(Bm + gk2 * sbk + gn * sbn) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kGemmK; ++k) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[k][ty * 4 + i];
        b[i] = Bs[k][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n < N) C[(int64_t)m * N + n] = acc[i][j] + (bias ? __ldg(bias + n) : 0.f);
    }
  }
}

// ------------------------------------------------------------------ column reductions

// Fixed-order fold of the 16 row lanes of one column (sm: [16][33]).
__device__ __forceinline__ float fold_lanes(float (*sm)[kColThreadsX + 1], float v) {
  const int tx = threadIdx.x, ty = threadIdx.y;
  sm[ty][tx] = v;
  __syncthreads();
  float s = 0.f;
  for (int l = 0; l < kColThreadsY; ++l) s += sm[l][tx];
  __syncthreads();
  return s;
}

// Row chunks of the BatchNorm kernels: block (32 columns x 16 row lanes),
// grid (columns / 32, R chunks); each statistic is a per-chunk partial in
// scratch, merged by the consumer in chunk order (deterministic).
__host__ __device__ inline int bn_chunks(int B) { return B <= 256 ? 1 : (B + 255) / 256 < 64 ? (B + 255) / 256 : 64; }
__device__ __forceinline__ void chunk_rows(int B, int R, int rc, int &r0, int &r1) {
  const int per = (B + R - 1) / R;
  r0 = min(B, rc * per);
  r1 = min(B, r0 + per);
}

// Forward statistics (T2), shifted sums: with K = relu(z[0][c]), per chunk
// S1 = sum (a - K), S2 = sum (a - K)^2 (the shift keeps S2 - S1^2/B free of
// cancellation).  part: [2][R][w].
__global__ void __launch_bounds__(512) train_bn_stats(int B, int w, int R, const float *__restrict__ z,
                                                      float *__restrict__ part) {
  __shared__ float sm[kColThreadsY][kColThreadsX + 1];
  const int tx = threadIdx.x, ty = threadIdx.y, rc = blockIdx.y;
  const int c = blockIdx.x * kColThreadsX + tx;
  const bool ok = c < w;
  int r0, r1;
  chunk_rows(B, R, rc, r0, r1);
  float s1 = 0.f, s2 = 0.f;
  if (ok) {
    const float K = fmaxf(z[c], 0.f);
    for (int r = r0 + ty; r < r1; r += kColThreadsY) {
      const float d = fmaxf(z[(int64_t)r * w + c], 0.f) - K;
      s1 += d;
      s2 = fmaf(d, d, s2);
    }
  }
  s1 = fold_lanes(sm, s1);
  s2 = fold_lanes(sm, s2);
  if (ok && ty == 0) {
    part[(int64_t)rc * w + c] = s1;
    part[(int64_t)(R + rc) * w + c] = s2;
  }
}

// Hidden-layer epilogue, forward.  Train (T2): merge the chunk statistics into
// the batch mean and biased variance, a_hat, y = gamma a_hat + beta, inverted
// dropout (T3); chunk 0 updates the running statistics (T6).  Eval: running
// statistics, no dropout.
__global__ void __launch_bounds__(512) train_bn_apply(int B, int w, int R, const float *__restrict__ z,
                                                      const float *__restrict__ part, const float *__restrict__ gamma,
                                                      const float *__restrict__ beta, float *__restrict__ rmean,
                                                      float *__restrict__ rvar, float *__restrict__ ahat,
                                                      float *__restrict__ h, float *__restrict__ inv_std, float eps,
                                                      float mom, int train, DropParams dp, int layer) {
  const int tx = threadIdx.x, ty = threadIdx.y, rc = blockIdx.y;
  const int c = blockIdx.x * kColThreadsX + tx;
  if (c >= w) return;
  int r0, r1;
  chunk_rows(B, R, rc, r0, r1);
  const float g = gamma[c], b = beta[c];
  if (!train) {
    const float m = rmean[c], inv = 1.0f / sqrtf(rvar[c] + eps);
    for (int r = r0 + ty; r < r1; r += kColThreadsY) {
      const float a = fmaxf(z[(int64_t)r * w + c], 0.f);
      h[(int64_t)r * w + c] = g * ((a - m) * inv) + b;
    }
    return;
  }
  float S1 = 0.f, S2 = 0.f;
  for (int k = 0; k < R; ++k) {
    S1 += part[(int64_t)k * w + c];
    S2 += part[(int64_t)(R + k) * w + c];
  }
  const float K = fmaxf(z[c], 0.f);
  const float d1 = S1 / (float)B;
  const float mean = K + d1;
  const float var = fmaxf(S2 / (float)B - d1 * d1, 0.f);
  const float inv = 1.0f / sqrtf(var + eps);
  for (int r = r0 + ty; r < r1; r += kColThreadsY) {
    const int64_t o = (int64_t)r * w + c;
    const float ah = (fmaxf(z[o], 0.f) - mean) * inv;
    ahat[o] = ah;
    h[o] = keep_unit(dp, layer, r, c) ? (g * ah + b) * dp.scale : 0.f;
  }
  if (rc == 0 && ty == 0) {
    inv_std[c] = inv;
    rmean[c] = (1.f - mom) * rmean[c] + mom * mean;
    rvar[c] = (1.f - mom) * rvar[c] + mom * (var * ((float)B / (float)(B - 1)));
  }
}

// Backward statistics per chunk (dy = dh * keep * scale): sum dy, sum dy a_hat,
// and over the active rows (z > 0): sum dy, sum a_hat, count.  part: [5][R][w].
__global__ void __launch_bounds__(512) train_bn_bwd_stats(int B, int w, int R, const float *__restrict__ dh,
                                                          const float *__restrict__ z, const float *__restrict__ ahat,
                                                          DropParams dp, int layer, float *__restrict__ part) {
  __shared__ float sm[kColThreadsY][kColThreadsX + 1];
  const int tx = threadIdx.x, ty = threadIdx.y, rc = blockIdx.y;
  const int c = blockIdx.x * kColThreadsX + tx;
  const bool ok = c < w;
  int r0, r1;
  chunk_rows(B, R, rc, r0, r1);
  float v[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
  if (ok)
    for (int r = r0 + ty; r < r1; r += kColThreadsY) {
      const int64_t o = (int64_t)r * w + c;
      const float dy = keep_unit(dp, layer, r, c) ? dh[o] * dp.scale : 0.f;
      const float ah = ahat[o];
      v[0] += dy;
      v[1] = fmaf(dy, ah, v[1]);
      if (z[o] > 0.f) {
        v[2] += dy;
        v[3] += ah;
        v[4] += 1.f;
      }
    }
#pragma unroll
  for (int k = 0; k < 5; ++k) v[k] = fold_lanes(sm, v[k]);
  if (ok && ty == 0)
#pragma unroll
    for (int k = 0; k < 5; ++k) part[(int64_t)(k * R + rc) * w + c] = v[k];
}

// Hidden-layer epilogue, backward: dgamma = sum dy a_hat, dbeta = sum dy;
// dz = inv_std (gamma dy - gamma mean(dy) - a_hat gamma mean(dy a_hat)) [z > 0];
// dbias = sum dz = inv_std (gamma sum_act dy - n_act m1 - m2 sum_act a_hat).
__global__ void __launch_bounds__(512) train_bn_bwd_apply(int B, int w, int R, const float *__restrict__ dh,
                                                          const float *__restrict__ z,
                                                          const float *__restrict__ ahat,
                                                          const float *__restrict__ part,
                                                          const float *__restrict__ gamma,
                                                          const float *__restrict__ inv_std, DropParams dp,
                                                          int layer, float *__restrict__ dz,
                                                          float *__restrict__ dgamma, float *__restrict__ dbeta,
                                                          float *__restrict__ dbias) {
  const int tx = threadIdx.x, ty = threadIdx.y, rc = blockIdx.y;
  const int c = blockIdx.x * kColThreadsX + tx;
  if (c >= w) return;
  int r0, r1;
  chunk_rows(B, R, rc, r0, r1);
  float S[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
  for (int k = 0; k < R; ++k)
#pragma unroll
    for (int q = 0; q < 5; ++q) S[q] += part[(int64_t)(q * R + k) * w + c];
  const float g = gamma[c], inv = inv_std[c];
  const float m1 = g * S[0] / (float)B, m2 = g * S[1] / (float)B;
  for (int r = r0 + ty; r < r1; r += kColThreadsY) {
    const int64_t o = (int64_t)r * w + c;
    const float dy = keep_unit(dp, layer, r, c) ? dh[o] * dp.scale : 0.f;
    dz[o] = z[o] > 0.f ? inv * (g * dy - m1 - ahat[o] * m2) : 0.f;
  }
  if (rc == 0 && ty == 0) {
    dgamma[c] = S[1];
    dbeta[c] = S[0];
    dbias[c] = inv * (g * S[2] - S[4] * m1 - m2 * S[3]);
  }
}

// Split-K partials of train_sgemm summed in slice order, plus the bias.
__global__ void train_splitk_reduce(int64_t MN, int N, int S, const float *__restrict__ part,
                                    const float *__restrict__ bias, float *__restrict__ C) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= MN) return;
  float v = 0.f;
  for (int z = 0; z < S; ++z) v += part[(int64_t)z * MN + i];
  C[i] = v + (bias ? bias[i % N] : 0.f);
}

// ------------------------------------------------------------------ output layer and loss (T4)

// Warp per row: e = sigmoid(h3 . w4 + b4), per-row loss; train: dz4 = dL/de e (1 - e)
// (with the 1/B of the mean) and dh3 = dz4 w4.
__global__ void train_out_fwd(int B, const float *__restrict__ h3, const float *__restrict__ w4,
                              const float *__restrict__ b4, const float *__restrict__ t, int loss, float q,
                              int train, float *__restrict__ dz4, float *__restrict__ dh3,
                              float *__restrict__ loss_r) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= B) return;
  const float *hr = h3 + (int64_t)r * 64;
  float z = hr[lane] * w4[lane] + hr[lane + 32] * w4[lane + 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
  z += b4[0];
  const float e = 1.0f / (1.0f + expf(-z));
  const float tr = t[r];
  float lr, dl;
  if (loss == SP_LOSS_MAPE) {
    const float tc = fmaxf(tr, 1e-6f);
    lr = fabsf(e - tr) / tc;
    dl = (e > tr ? 1.f : e < tr ? -1.f : 0.f) / tc;
  } else {
    const float d = tr - e;
    lr = fmaxf(q * d, (q - 1.f) * d);
    dl = e > tr ? 1.f - q : tr > e ? -q : 0.f;
  }
  if (lane == 0) loss_r[r] = lr;
  if (!train) return;
  const float dz = dl / (float)B * e * (1.f - e);
  if (lane == 0) dz4[r] = dz;
  dh3[(int64_t)r * 64 + lane] = dz * w4[lane];
  dh3[(int64_t)r * 64 + lane + 32] = dz * w4[lane + 32];
}

// One block (64 columns x 16 row lanes): dw4 = sum_r dz4 h3, db4 = sum dz4,
// loss = sum_r loss_r / B (train), or the chunk's loss sum into partial (eval).
__global__ void __launch_bounds__(1024) train_out_red(int B, const float *__restrict__ h3,
                                                      const float *__restrict__ dz4,
                                                      const float *__restrict__ loss_r, int train,
                                                      float *__restrict__ dw4, float *__restrict__ db4,
                                                      float *__restrict__ loss_out) {
  __shared__ float sm[16][65];
  const int c = threadIdx.x & 63, ly = threadIdx.x >> 6;
  if (train) {
    float s = 0.f;
    for (int r = ly; r < B; r += 16) s = fmaf(dz4[r], h3[(int64_t)r * 64 + c], s);
    sm[ly][c] = s;
  }
  // loss and db4: 16 x 32 lanes over rows in a fixed interleave
  const int lx = threadIdx.x & 31, lyy = threadIdx.x >> 5;  // 32 x 32 threads
  float sl_ = 0.f, sd = 0.f;
  for (int r = lyy * 32 + lx; r < B; r += 1024) {
    sl_ += loss_r[r];
    if (train) sd += dz4[r];
  }
  __shared__ float sll[1024], sdd[1024];
  sll[threadIdx.x] = sl_;
  sdd[threadIdx.x] = sd;
  __syncthreads();
  if (train && ly == 0) {
    float s = 0.f;
    for (int l = 0; l < 16; ++l) s += sm[l][c];
    dw4[c] = s;
  }
  if (threadIdx.x == 0) {
    float a = 0.f, d = 0.f;
    for (int i = 0; i < 1024; ++i) {
      a += sll[i];
      d += sdd[i];
    }
    if (train) {
      db4[0] = d;
      loss_out[0] = a / (float)B;
    } else {
      loss_out[0] = a;
    }
  }
}

__global__ void train_loss_finalize(int n_chunks, const float *__restrict__ partial, int64_t n,
                                    float *__restrict__ loss_out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  float s = 0.f;
  for (int i = 0; i < n_chunks; ++i) s += partial[i];
  loss_out[0] = s / (float)n;
}

__global__ void train_copy_scalar(const float *__restrict__ src, float *__restrict__ dst) {
  if (threadIdx.x == 0 && blockIdx.x == 0) dst[0] = src[0];
}

// ------------------------------------------------------------------ AdamW (T5)

__global__ void train_adamw(int64_t n, float *__restrict__ p, const float *__restrict__ g, float *__restrict__ m,
                            float *__restrict__ v, float lr, float wd, float b1, float b2, float eps,
                            const int64_t *__restrict__ step) {
  // bias corrections 1 - beta^t in fp64 (t = the step being taken), rounded once
  const double t = (double)(*step + 1);
  const float bc1 = (float)(1.0 - pow((double)b1, t)), bc2 = (float)(1.0 - pow((double)b2, t));
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float gi = g[i];
  const float mi = b1 * m[i] + (1.f - b1) * gi;
  const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
  m[i] = mi;
  v[i] = vi;
  const float mh = mi / bc1, vh = vi / bc2;
  p[i] = p[i] - lr * (wd * p[i] + mh / (sqrtf(vh) + eps));
}

__global__ void train_step_end(int64_t *step) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *step += 1;
}

// ------------------------------------------------------------------ normalisation fit (T7)

// Block per feature; fp64 sums over the rows in a fixed order (thread i takes
// rows i, i+256, ...; then a sequential fold of the 256 partials).
__global__ void __launch_bounds__(256) fit_norm_kernel(sp_features f, int pipes, const int64_t *__restrict__ idx,
                                                       int64_t n, double *__restrict__ out) {
  __shared__ double part[256];
  __shared__ double mean_s;
  const int k = blockIdx.x;
  const int s = feature_slot(pipes, k);
  auto val = [&](int64_t r) {
    const int64_t p = __ldg(idx + r);
    const double v = (s & 256) ? (double)__ldg(f.flts + (int64_t)(s & 255) * f.ld + p)
                               : (double)__ldg(f.ints + (int64_t)s * f.ld + p);
    return log1p(v);
  };
  double a = 0.0;
  for (int64_t r = threadIdx.x; r < n; r += 256) a += val(r);
  part[threadIdx.x] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < 256; ++i) t += part[i];
    mean_s = t / (double)n;
  }
  __syncthreads();
  const double mu = mean_s;
  double b = 0.0;
  for (int64_t r = threadIdx.x; r < n; r += 256) {
    const double d = val(r) - mu;
    b += d * d;
  }
  __syncthreads();
  part[threadIdx.x] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < 256; ++i) t += part[i];
    out[2 * k] = mu;
    out[2 * k + 1] = sqrt(t / (double)n);
  }
}

int pipes_count(int fam) {
  const int p = family_pipes(fam);
  return (p & 1) + ((p >> 1) & 1) + ((p >> 2) & 1);
}

bool family_ok(int fam) { return fam >= SP_GEMM && fam <= SP_GEMM_SPLITK; }

}  // namespace

// ------------------------------------------------------------------ trainer

struct sp_trainer {
  sp_ctx *ctx = nullptr;
  int family = 0, n_in = 0, pipes = 0;
  sp_train_config cfg{};
  float bn_eps = 1e-5f;
  int64_t step = 0;
  int64_t n_params = 0;
  // offsets into the flat parameter vector: layer l = 0..2 w, b, g, be; then w4, b4
  int64_t ow[4] = {}, ob[4] = {}, og[3] = {}, obe[3] = {};
  DevBuf params, grads, mom1, mom2, running, norm, act, partial, scratch;
  float *bn_part = nullptr;  // BatchNorm chunk partials [5][64][256]
  int64_t *dstep = nullptr;  // DEVICE step counter (dropout counter, AdamW t - 1)
  float *kpart = nullptr;    // split-K GEMM partials
  int64_t kpart_cap = 0;     // floats
  size_t partial_cap = 0;
  int B = 0;  // max batch
  float *x = nullptr, *t = nullptr, *z[3] = {}, *ah[3] = {}, *h[3] = {}, *inv[3] = {}, *dz4 = nullptr,
        *loss_r = nullptr, *dh = nullptr, *dzb = nullptr, *loss = nullptr;
  float *rm[3] = {}, *rv[3] = {};
};

namespace {

sp_status check_features(sp_trainer *tr, const sp_features *in, const float *measured, const int64_t *idx,
                         int64_t n) {
  if (!in || !measured || !idx) return fail(tr->ctx, SP_E_ARG, "training: NULL argument");
  if (in->family != tr->family) return fail(tr->ctx, SP_E_ARG, "training: features/model family mismatch");
  if (!in->ints || !in->flts || in->ld < in->n_pairs) return fail(tr->ctx, SP_E_ARG, "training: bad features");
  if (n < 0) return fail(tr->ctx, SP_E_ARG, "training: negative row count");
  return SP_OK;
}

DropParams drop_params(const sp_trainer *tr) {
  DropParams d;
  d.seed = tr->cfg.seed;
  d.step = tr->dstep;
  d.thr = (uint32_t)std::llround((double)tr->cfg.dropout * 16777216.0);
  d.scale = 1.0f / (1.0f - tr->cfg.dropout);
  return d;
}

// C[M][N] = A . B (+ bias) with train_sgemm; GEMMs whose tile grid would not
// fill the GPU (the dW products: K = batch rows) are split along K into S
// slices summed in order by train_splitk_reduce.
void gemm(sp_trainer *tr, int M, int N, int K, const float *A, int64_t sam, int64_t sak, const float *Bm, int64_t sbk,
          int64_t sbn, const float *bias, float *C, cudaStream_t st, const LaunchHook &hk) {
  const int gx = (N + kGemmT - 1) / kGemmT, gy = (M + kGemmT - 1) / kGemmT;
  const int target = 2 * tr->ctx->num_sms;
  int S = 1;
  if (gx * gy < target && K >= 4 * kGemmK) {
    S = std::min((target + gx * gy - 1) / (gx * gy), K / (2 * kGemmK));
    S = (int)std::min<int64_t>(S, tr->kpart_cap / ((int64_t)M * N));
    S = std::max(S, 1);
  }
  hk.on_begin("train_sgemm", st);
  train_sgemm<<<dim3(gx, gy, S), 256, 0, st>>>(M, N, K, A, sam, sak, Bm, sbk, sbn, bias, S > 1 ? tr->kpart : C);
  hk.on_end(st);
  if (S > 1) {
    const int64_t MN = (int64_t)M * N;
    hk.on_begin("train_splitk_reduce", st);
    train_splitk_reduce<<<(unsigned)((MN + 255) / 256), 256, 0, st>>>(MN, N, S, tr->kpart, bias, C);
    hk.on_end(st);
  }
}

// Forward of rows [0, B) already gathered into tr->x / tr->t.
void forward(sp_trainer *tr, int B, bool train, const DropParams &dp, cudaStream_t st, const LaunchHook &hk) {
  const float *P = (const float *)tr->params.p;
  const float *hin = tr->x;
  int fan = tr->n_in;
  const int R = bn_chunks(B);
  for (int l = 0; l < 3; ++l) {
    const int w = kHid[l];
    gemm(tr, B, w, fan, hin, fan, 1, P + tr->ow[l], 1, fan, P + tr->ob[l], tr->z[l], st, hk);
    const dim3 cg((w + kColThreadsX - 1) / kColThreadsX, R), cb(kColThreadsX, kColThreadsY);
    if (train) {
      hk.on_begin("train_bn_stats", st);
      train_bn_stats<<<cg, cb, 0, st>>>(B, w, R, tr->z[l], tr->bn_part);
      hk.on_end(st);
    }
    hk.on_begin("train_bn_apply", st);
    train_bn_apply<<<cg, cb, 0, st>>>(B, w, R, tr->z[l], tr->bn_part, P + tr->og[l], P + tr->obe[l], tr->rm[l],
                                      tr->rv[l], tr->ah[l], tr->h[l], tr->inv[l], tr->bn_eps, tr->cfg.bn_momentum,
                                      train ? 1 : 0, dp, l);
    hk.on_end(st);
    hin = tr->h[l];
    fan = w;
  }
}

}  // namespace

extern "C" sp_status sp_train_create(sp_ctx *ctx, const sp_mlp_desc *d, const sp_train_config *cfg,
                                     sp_trainer **out) {
  if (!ctx || !d || !cfg || !out) return fail(ctx, SP_E_ARG, "sp_train_create: NULL argument");
  *out = nullptr;
  if (!family_ok(d->family)) return fail(ctx, SP_E_ARG, "sp_train_create: unknown family");
  const int n_in = d->n_in;
  if (n_in != 4 * pipes_count(d->family) + 7)
    return fail(ctx, SP_E_DATA, "sp_train_create: n_in does not match the family's Table IV layout");
  if (cfg->max_batch < 2 || cfg->max_batch > (1 << 20))
    return fail(ctx, SP_E_ARG, "sp_train_create: max_batch must be in [2, 2^20]");
  if (!(cfg->lr > 0.f) || !(cfg->dropout >= 0.f && cfg->dropout < 1.f) || !(cfg->beta1 >= 0.f && cfg->beta1 < 1.f) ||
      !(cfg->beta2 >= 0.f && cfg->beta2 < 1.f) || !(cfg->adam_eps > 0.f) || !(cfg->weight_decay >= 0.f) ||
      !(cfg->bn_momentum >= 0.f && cfg->bn_momentum <= 1.f) ||
      (cfg->loss != SP_LOSS_MAPE && cfg->loss != SP_LOSS_PINBALL) ||
      (cfg->loss == SP_LOSS_PINBALL && !(cfg->quantile > 0.f && cfg->quantile < 1.f)))
    return fail(ctx, SP_E_ARG, "sp_train_create: invalid training configuration");
  if (!(d->bn_eps > 0.f)) return fail(ctx, SP_E_DATA, "sp_train_create: bn_eps must be > 0");
  const float *vecs[] = {d->mu, d->sigma, d->w1, d->b1, d->g1, d->be1, d->m1, d->v1, d->w2, d->b2, d->g2,
                         d->be2, d->m2, d->v2, d->w3, d->b3, d->g3, d->be3, d->m3, d->v3, d->w4};
  for (const float *v : vecs)
    if (!v) return fail(ctx, SP_E_ARG, "sp_train_create: NULL weight pointer");

  sp_trainer *tr = new (std::nothrow) sp_trainer;
  if (!tr) return fail(ctx, SP_E_INTERNAL, "sp_train_create: out of host memory");
  tr->ctx = ctx;
  tr->family = d->family;
  tr->n_in = n_in;
  tr->pipes = family_pipes(d->family);
  tr->cfg = *cfg;
  tr->bn_eps = d->bn_eps;
  tr->B = cfg->max_batch;

  // flat parameter vector
  std::vector<float> P;
  auto put = [&](const float *src, int64_t n) {
    const int64_t o = (int64_t)P.size();
    P.insert(P.end(), src, src + n);
    return o;
  };
  const float *W[3] = {d->w1, d->w2, d->w3}, *Bv[3] = {d->b1, d->b2, d->b3}, *G[3] = {d->g1, d->g2, d->g3},
              *BE[3] = {d->be1, d->be2, d->be3}, *RM[3] = {d->m1, d->m2, d->m3}, *RV[3] = {d->v1, d->v2, d->v3};
  int fan = n_in;
  for (int l = 0; l < 3; ++l) {
    tr->ow[l] = put(W[l], (int64_t)kHid[l] * fan);
    tr->ob[l] = put(Bv[l], kHid[l]);
    tr->og[l] = put(G[l], kHid[l]);
    tr->obe[l] = put(BE[l], kHid[l]);
    fan = kHid[l];
  }
  tr->ow[3] = put(d->w4, 64);
  tr->ob[3] = put(&d->b4, 1);
  tr->n_params = (int64_t)P.size();
  for (float v : P)
    if (!std::isfinite(v)) {
      delete tr;
      return fail(ctx, SP_E_DATA, "sp_train_create: non-finite initial weight");
    }
  std::vector<float> R;  // running statistics m1 v1 m2 v2 m3 v3
  for (int l = 0; l < 3; ++l) {
    R.insert(R.end(), RM[l], RM[l] + kHid[l]);
    R.insert(R.end(), RV[l], RV[l] + kHid[l]);
  }
  std::vector<float> N(d->mu, d->mu + n_in);
  N.insert(N.end(), d->sigma, d->sigma + n_in);
  std::vector<float> zeros(P.size(), 0.f);
  const size_t pb = P.size() * sizeof(float);
  cudaSetDevice(ctx->device);
  cudaError_t e;
  if ((e = tr->params.alloc_copy(P.data(), pb)) != cudaSuccess || (e = tr->grads.alloc_copy(zeros.data(), pb)) ||
      (e = tr->mom1.alloc_copy(zeros.data(), pb)) || (e = tr->mom2.alloc_copy(zeros.data(), pb)) ||
      (e = tr->running.alloc_copy(R.data(), R.size() * sizeof(float))) ||
      (e = tr->norm.alloc_copy(N.data(), N.size() * sizeof(float)))) {
    delete tr;
    return cuda_fail(ctx, e, "sp_train_create: parameter buffers");
  }
  // activations for max_batch rows
  const int64_t B = tr->B;
  const int64_t n_act = B * n_in + B + 3 * B * (256 + 128 + 64) + (256 + 128 + 64) + B + B + 2 * B * 256 + 4;
  e = cudaMalloc(&tr->act.p, (size_t)n_act * sizeof(float));
  if (e != cudaSuccess) {
    tr->act.p = nullptr;
    delete tr;
    return cuda_fail(ctx, e, "sp_train_create: activation buffers");
  }
  float *a = (float *)tr->act.p;
  auto take = [&](int64_t n) {
    float *r = a;
    a += n;
    return r;
  };
  tr->x = take(B * n_in);
  tr->t = take(B);
  for (int l = 0; l < 3; ++l) {
    tr->z[l] = take(B * kHid[l]);
    tr->ah[l] = take(B * kHid[l]);
    tr->h[l] = take(B * kHid[l]);
    tr->inv[l] = take(kHid[l]);
  }
  tr->dz4 = take(B);
  tr->loss_r = take(B);
  tr->dh = take(B * 256);
  tr->dzb = take(B * 256);
  tr->loss = take(4);
  // BatchNorm partials and split-K partials (no allocation inside a step)
  tr->kpart_cap = (int64_t)32 * 256 * 256;
  const size_t scratch_floats = (size_t)5 * 64 * 256 + (size_t)tr->kpart_cap;  // even: the step counter is 8-aligned
  e = cudaMalloc(&tr->scratch.p, scratch_floats * sizeof(float) + sizeof(int64_t));
  if (e == cudaSuccess) e = cudaMemset(tr->scratch.p, 0, scratch_floats * sizeof(float) + sizeof(int64_t));
  if (e != cudaSuccess) {
    tr->scratch.p = nullptr;
    delete tr;
    return cuda_fail(ctx, e, "sp_train_create: scratch");
  }
  tr->bn_part = (float *)tr->scratch.p;
  tr->dstep = reinterpret_cast<int64_t *>(tr->bn_part + scratch_floats);
  tr->kpart = tr->bn_part + (size_t)5 * 64 * 256;
  float *rs = (float *)tr->running.p;
  for (int l = 0, o = 0; l < 3; ++l) {
    tr->rm[l] = rs + o;
    tr->rv[l] = rs + o + kHid[l];
    o += 2 * kHid[l];
  }
  *out = tr;
  return SP_OK;
}

extern "C" void sp_train_destroy(sp_trainer *tr) { delete tr; }

extern "C" sp_status sp_train_step(sp_trainer *tr, const sp_features *in, const float *measured,
                                   const int64_t *batch_idx, int64_t B, float *loss_out, void *stream) {
  if (!tr) return fail(nullptr, SP_E_ARG, "sp_train_step: NULL trainer");
  sp_status s = check_features(tr, in, measured, batch_idx, B);
  if (s != SP_OK) return s;
  if (B < 2 || B > tr->B) return fail(tr->ctx, SP_E_ARG, "sp_train_step: B must be in [2, max_batch]");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const LaunchHook hk = tr->ctx->hook();
  const int b = (int)B, n_in = tr->n_in;
  const DropParams dp = drop_params(tr);
  float *P = (float *)tr->params.p, *G = (float *)tr->grads.p;
  const float *mu = (const float *)tr->norm.p, *sg = mu + n_in;

  hk.on_begin("train_gather", st);
  const int64_t ng = B * (n_in + 1);
  train_gather<<<(unsigned)((ng + 255) / 256), 256, 0, st>>>(*in, tr->pipes, n_in, mu, sg, measured, batch_idx, B,
                                                             tr->x, tr->t);
  hk.on_end(st);
  forward(tr, b, true, dp, st, hk);
  // output layer: dh3 into tr->dh ([B][64])
  hk.on_begin("train_out", st);
  train_out_fwd<<<(b + 7) / 8, 256, 0, st>>>(b, tr->h[2], P + tr->ow[3], P + tr->ob[3], tr->t, tr->cfg.loss,
                                             tr->cfg.quantile, 1, tr->dz4, tr->dh, tr->loss_r);
  train_out_red<<<1, 1024, 0, st>>>(b, tr->h[2], tr->dz4, tr->loss_r, 1, G + tr->ow[3], G + tr->ob[3], tr->loss);
  hk.on_end(st);
  // backward through the hidden layers: dh (layer l's output grad) -> dzb -> dW, dh(l-1)
  const int R = bn_chunks(b);
  for (int l = 2; l >= 0; --l) {
    const int w = kHid[l], fan = l ? kHid[l - 1] : n_in;
    const dim3 cg((w + kColThreadsX - 1) / kColThreadsX, R), cb(kColThreadsX, kColThreadsY);
    hk.on_begin("train_bn_bwd", st);
    train_bn_bwd_stats<<<cg, cb, 0, st>>>(b, w, R, tr->dh, tr->z[l], tr->ah[l], dp, l, tr->bn_part);
    train_bn_bwd_apply<<<cg, cb, 0, st>>>(b, w, R, tr->dh, tr->z[l], tr->ah[l], tr->bn_part, P + tr->og[l],
                                          tr->inv[l], dp, l, tr->dzb, G + tr->og[l], G + tr->obe[l], G + tr->ob[l]);
    hk.on_end(st);
    const float *hprev = l ? tr->h[l - 1] : tr->x;
    // dW[w][fan] = dZ^T H: A(m=unit, k=row) = dzb[row*w + unit], B(k=row, n) = hprev[row*fan + n]
    gemm(tr, w, fan, b, tr->dzb, 1, w, hprev, fan, 1, nullptr, G + tr->ow[l], st, hk);
    // dH[B][fan] = dZ W: A(m=row, k=unit) = dzb[row*w + unit], B(k=unit, n) = W[unit*fan + n]
    if (l) gemm(tr, b, fan, w, tr->dzb, w, 1, P + tr->ow[l], fan, 1, nullptr, tr->dh, st, hk);
  }
  tr->step += 1;
  hk.on_begin("train_adamw", st);
  train_adamw<<<(unsigned)((tr->n_params + 255) / 256), 256, 0, st>>>(
      tr->n_params, P, G, (float *)tr->mom1.p, (float *)tr->mom2.p, tr->cfg.lr, tr->cfg.weight_decay,
      tr->cfg.beta1, tr->cfg.beta2, tr->cfg.adam_eps, tr->dstep);
  hk.on_end(st);
  train_step_end<<<1, 32, 0, st>>>(tr->dstep);
  if (loss_out) train_copy_scalar<<<1, 32, 0, st>>>(tr->loss, loss_out);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(tr->ctx, e, "sp_train_step: launch");
  return SP_OK;
}

extern "C" sp_status sp_train_eval(sp_trainer *tr, const sp_features *in, const float *measured,
                                   const int64_t *idx, int64_t n, float *loss_out, void *stream) {
  if (!tr) return fail(nullptr, SP_E_ARG, "sp_train_eval: NULL trainer");
  sp_status s = check_features(tr, in, measured, idx, n);
  if (s != SP_OK) return s;
  if (n < 1 || !loss_out) return fail(tr->ctx, SP_E_ARG, "sp_train_eval: n must be >= 1 and loss_out non-NULL");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const LaunchHook hk = tr->ctx->hook();
  const int64_t chunks = (n + tr->B - 1) / tr->B;
  if ((size_t)chunks > tr->partial_cap) {
    // grow-only scratch; validation sets are set up once
    if (tr->partial.p) cudaFree(tr->partial.p);
    tr->partial.p = nullptr;
    tr->partial_cap = 0;
    cudaError_t e = cudaMalloc(&tr->partial.p, (size_t)chunks * sizeof(float));
    if (e != cudaSuccess) {
      tr->partial.p = nullptr;
      return cuda_fail(tr->ctx, e, "sp_train_eval: scratch");
    }
    tr->partial_cap = (size_t)chunks;
  }
  const float *P = (const float *)tr->params.p;
  const float *mu = (const float *)tr->norm.p, *sg = mu + tr->n_in;
  const DropParams dp = drop_params(tr);
  for (int64_t c = 0; c < chunks; ++c) {
    const int64_t r0 = c * tr->B, b = std::min<int64_t>(tr->B, n - r0);
    const int64_t ng = b * (tr->n_in + 1);
    hk.on_begin("train_gather", st);
    train_gather<<<(unsigned)((ng + 255) / 256), 256, 0, st>>>(*in, tr->pipes, tr->n_in, mu, sg, measured, idx + r0,
                                                               b, tr->x, tr->t);
    hk.on_end(st);
    forward(tr, (int)b, false, dp, st, hk);
    hk.on_begin("train_out", st);
    train_out_fwd<<<(unsigned)((b + 7) / 8), 256, 0, st>>>((int)b, tr->h[2], P + tr->ow[3], P + tr->ob[3], tr->t,
                                                          tr->cfg.loss, tr->cfg.quantile, 0, nullptr, nullptr,
                                                          tr->loss_r);
    train_out_red<<<1, 1024, 0, st>>>((int)b, tr->h[2], nullptr, tr->loss_r, 0, nullptr, nullptr,
                                      (float *)tr->partial.p + c);
    hk.on_end(st);
  }
  train_loss_finalize<<<1, 32, 0, st>>>((int)chunks, (const float *)tr->partial.p, n, loss_out);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(tr->ctx, e, "sp_train_eval: launch");
  return SP_OK;
}

extern "C" int64_t sp_train_export_count(const sp_trainer *tr) {
  return tr ? tr->n_params + 2 * (256 + 128 + 64) : -1;
}

extern "C" sp_status sp_train_export(sp_trainer *tr, float *host_out, void *stream) {
  if (!tr || !host_out) return fail(tr ? tr->ctx : nullptr, SP_E_ARG, "sp_train_export: NULL argument");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(host_out, tr->params.p, tr->n_params * sizeof(float), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(host_out + tr->n_params, tr->running.p, 2 * (256 + 128 + 64) * sizeof(float),
                        cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(tr->ctx, e, "sp_train_export");
  return SP_OK;
}

extern "C" sp_status sp_train_export_grads(sp_trainer *tr, float *host_out, void *stream) {
  if (!tr || !host_out) return fail(tr ? tr->ctx : nullptr, SP_E_ARG, "sp_train_export_grads: NULL argument");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(host_out, tr->grads.p, tr->n_params * sizeof(float), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(tr->ctx, e, "sp_train_export_grads");
  return SP_OK;
}

extern "C" sp_status sp_fit_norm(sp_ctx *ctx, const sp_features *in, const int64_t *idx, int64_t n, float *mu_out,
                                 float *sigma_out, void *stream) {
  if (!ctx || !in || !idx || !mu_out || !sigma_out) return fail(ctx, SP_E_ARG, "sp_fit_norm: NULL argument");
  if (!family_ok(in->family)) return fail(ctx, SP_E_ARG, "sp_fit_norm: unknown family");
  if (n < 1) return fail(ctx, SP_E_ARG, "sp_fit_norm: n must be >= 1");
  const int n_in = 4 * pipes_count(in->family) + 7;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  DevBuf out;
  cudaError_t e = cudaMalloc(&out.p, 2 * n_in * sizeof(double));
  if (e != cudaSuccess) {
    out.p = nullptr;
    return cuda_fail(ctx, e, "sp_fit_norm: scratch");
  }
  const LaunchHook hk = ctx->hook();
  hk.on_begin("fit_norm", st);
  fit_norm_kernel<<<n_in, 256, 0, st>>>(*in, family_pipes(in->family), idx, n, (double *)out.p);
  hk.on_end(st);
  double h[2 * 16];
  e = cudaMemcpyAsync(h, out.p, 2 * n_in * sizeof(double), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "sp_fit_norm");
  for (int k = 0; k < n_in; ++k) {
    mu_out[k] = (float)h[2 * k];
    sigma_out[k] = (float)h[2 * k + 1];
  }
  return SP_OK;
}
