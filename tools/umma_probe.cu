// Probe of the tcgen05 (UMMA) operand conventions on sm_100a: one CTA computes
// D[M x N] = A[M x K] * B[N x K]^T with bf16 operands in shared memory
// (K-major, no swizzle, core matrices of 8 rows x 16 bytes) and an fp32
// accumulator in TMEM, for every combination of core-matrix strides and
// descriptor LBO/SBO assignment; prints which combinations are exact.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_probe umma_probe.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>

constexpr int M = 128, N = 64, K = 64;

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm_100)
  return d;                 // layout type 0 = no swizzle
}

__device__ __forceinline__ uint32_t off_of(int r, int k, int cR, int cK) {
  return (r / 8) * cR + (k / 8) * cK + (r % 8) * 16 + (k % 8) * 2;
}

__global__ void probe(const __nv_bfloat16 *A, const __nv_bfloat16 *B, float *D, int variant) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  uint8_t *sA = sm, *sB = sm + M * K * 2;
  // variant bit0: layout (0: K-adjacent core matrices contiguous, 1: row-adjacent contiguous)
  // variant bit1: descriptor (0: LBO = K-direction stride, 1: LBO = row-direction stride)
  const int lay = variant & 1, swap = (variant >> 1) & 1;
  const int cK_A = lay ? (M / 8) * 128 : 128, cR_A = lay ? 128 : K * 16;
  const int cK_B = lay ? (N / 8) * 128 : 128, cR_B = lay ? 128 : K * 16;
  for (int i = threadIdx.x; i < M * K; i += blockDim.x) {
    int r = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16 *>(sA + off_of(r, k, cR_A, cK_A)) = A[i];
  }
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    int r = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16 *>(sB + off_of(r, k, cR_B, cK_B)) = B[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const uint32_t mbar_s = (uint32_t)__cvta_generic_to_shared(&mbar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar_s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&tmem_base);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(dst));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sA), b0 = (uint32_t)__cvta_generic_to_shared(sB);
    for (int ks = 0; ks < K / 16; ++ks) {
      const uint32_t la = swap ? cR_A : cK_A, sa = swap ? cK_A : cR_A;
      const uint32_t lb = swap ? cR_B : cK_B, sb = swap ? cK_B : cR_B;
      const uint64_t da = desc(a0 + ks * 2 * cK_A, la, sa);
      const uint64_t db = desc(b0 + ks * 2 * cK_B, lb, sb);
      const uint32_t acc = ks > 0;
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar_s));
  }
  // wait for the MMA
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done) : "r"(mbar_s), "r"(0u));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp < 4) {
    for (int c0 = 0; c0 < N; c0 += 16) {
      uint32_t v[16];
      const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 16; ++j) D[(warp * 32 + lane) * N + c0 + j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

int main() {
  std::vector<__nv_bfloat16> A(M * K), B(N * K);
  std::vector<float> Af(M * K), Bf(N * K), ref(M * N), D(M * N);
  srand(1);
  for (int i = 0; i < M * K; ++i) { Af[i] = (float)(rand() % 7 - 3); A[i] = __float2bfloat16(Af[i]); }
  for (int i = 0; i < N * K; ++i) { Bf[i] = (float)(rand() % 5 - 2); B[i] = __float2bfloat16(Bf[i]); }
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      float s = 0;
      for (int k = 0; k < K; ++k) s += Af[m * K + k] * Bf[n * K + k];
      ref[m * N + n] = s;
    }
  __nv_bfloat16 *dA, *dB;
  float *dD;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  const int smem = (M + N) * K * 2;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int v = 0; v < 4; ++v) {
    cudaMemset(dD, 0, D.size() * 4);
    probe<<<1, 128, smem>>>(dA, dB, dD, v);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < M * N; ++i) bad += D[i] != ref[i];
    printf("variant layout=%d swap=%d: %s, mismatches %d / %d (D[0]=%g ref %g)\n", v & 1, v >> 1,
           cudaGetErrorString(e), bad, M * N, D[0], ref[0]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
