// Probe: do UMMA shared-memory descriptors with a zero stride alias as plain
// strides would (SBO = 0: every 8-row group reads the same rows; LBO = 0: both
// K core matrices of a K = 16 step read the same 16 bytes per row)?  One CTA,
// D[128 x 128] = A[128 x 16] . B[128 x 16]^T, fp16 operands, fp32 in TMEM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I. -o umma_alias_probe umma_alias_probe.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

#include "../paper_2601_14910_b200/csrc/tcgen05.cuh"

using namespace sp;
constexpr int M = 128, N = 128, K = 16;

__global__ void probe(const __half *Ag, const __half *Bg, float *D, int a_alias, int b_alias) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  uint8_t *sA = sm, *sB = sm + M * K * 2;
  // A: full layout off(r,k) = (r/8)*256 + (k/8)*128 + (r%8)*16 + (k%8)*2, or with
  // a_alias only rows 0..7 stored (SBO = 0).  B: full (LBO 128, SBO 256) or with
  // b_alias only K 0..7 stored per row (LBO = 0, SBO = 128).
  for (int i = threadIdx.x; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    if (a_alias && r >= 8) continue;
    *reinterpret_cast<__half *>(sA + (r / 8) * 256 + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2) = Ag[i];
  }
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    if (b_alias) {
      if (k >= 8) continue;
      *reinterpret_cast<__half *>(sB + (r / 8) * 128 + (r % 8) * 16 + k * 2) = Bg[i];
    } else {
      *reinterpret_cast<__half *>(sB + (r / 8) * 256 + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2) = Bg[i];
    }
  }
  tc::fence_proxy_async();
  const uint32_t mb = tc::smem_u32(&mbar);
  if (threadIdx.x == 0) {
    tc::mbar_init(mb, 1);
    tc::mbar_init_fence();
  }
  if (threadIdx.x < 32) tc::tmem_alloc<128>(tc::smem_u32(&tmem_base));
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  if (threadIdx.x == 0) {
    const uint64_t da = a_alias ? tc::smem_desc(tc::smem_u32(sA), 128, 0) : tc::smem_desc(tc::smem_u32(sA), 128, 256);
    const uint64_t db = b_alias ? tc::smem_desc(tc::smem_u32(sB), 0, 128) : tc::smem_desc(tc::smem_u32(sB), 128, 256);
    tc::mma_f16kind(tmem, da, db, tc::idesc_f16kind_f32(M, N, false), 0);
    tc::commit(mb);
  }
  tc::mbar_wait(mb, 0);
  tc::fence_after();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
    tc::tmem_wait_ld();
    for (int j = 0; j < 32; ++j) D[(warp * 32 + lane) * N + c0 + j] = __uint_as_float(v[j]);
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<128>(tmem);
}

int main() {
  std::vector<__half> A(M * K), B(N * K);
  std::vector<float> Af(M * K), Bf(N * K), D(M * N);
  srand(3);
  for (int i = 0; i < M * K; ++i) { Af[i] = (float)(rand() % 7 - 3); A[i] = __float2half(Af[i]); }
  for (int i = 0; i < N * K; ++i) { Bf[i] = (float)(rand() % 5 - 2); B[i] = __float2half(Bf[i]); }
  __half *dA, *dB;
  float *dD;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  const int smem = (M + N) * K * 2;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int v = 0; v < 4; ++v) {
    const int aa = v & 1, ba = v >> 1;
    cudaMemset(dD, 0, D.size() * 4);
    probe<<<1, 128, smem>>>(dA, dB, dD, aa, ba);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        float s = 0;  // the aliased operand as the descriptor should present it
        for (int k = 0; k < K; ++k) {
          const float a = Af[(aa ? m % 8 : m) * K + k];
          const float b = Bf[n * K + (ba ? k % 8 : k)];
          s += a * b;
        }
        bad += D[m * N + n] != s;
      }
    printf("A SBO=0: %d  B LBO=0: %d -> %s, mismatches %d / %d\n", aa, ba, cudaGetErrorString(e), bad, M * N);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
