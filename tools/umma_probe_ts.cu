// Probe of the tcgen05 "A from TMEM" form (kind::f16, cta_group::1, M = 128):
// A[128 x K] fp16 is written to TMEM by tcgen05.st, lane m = row m, 32-bit
// column c = (A[m][2c] low half, A[m][2c+1] high half); B[N x K] in shared
// memory (K-major, no swizzle, as tools/umma_probe.cu).  Checks D = A.B^T.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_probe_ts umma_probe_ts.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int M = 128, N = 64, K = 64;

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

__global__ void probe(const __half *A, const __half *B, float *D, int variant) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  uint8_t *sB = sm;
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    int r = i / K, k = i % K;
    *reinterpret_cast<__half *>(sB + (r / 8) * (K * 16) + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2) = B[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const uint32_t mbar_s = (uint32_t)__cvta_generic_to_shared(&mbar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar_s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&tmem_base);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(dst));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int row = warp * 32 + lane;
  // A -> TMEM columns [64, 64 + K/2): 32 columns of packed pairs
  const uint32_t a_col = 64;
  {
    uint32_t v[32];
    for (int c = 0; c < K / 2; ++c) {
      __half lo = A[row * K + 2 * c], hi = A[row * K + 2 * c + 1];
      if (variant == 1) { __half t = lo; lo = hi; hi = t; }  // swapped halves
      v[c] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
    }
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + a_col;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
        "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
        "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(sB);
    for (int ks = 0; ks < K / 16; ++ks) {
      const uint64_t db = desc(b0 + ks * 256, 128, K * 16);
      const uint32_t at = tmem + a_col + ks * 8;
      const uint32_t acc = ks > 0;
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
          "r"(at), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar_s));
  }
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done) : "r"(mbar_s), "r"(0u));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

int main() {
  std::vector<__half> A(M * K), B(N * K);
  std::vector<float> Af(M * K), Bf(N * K), ref(M * N), D(M * N);
  srand(2);
  for (int i = 0; i < M * K; ++i) { Af[i] = (float)(rand() % 7 - 3); A[i] = __float2half(Af[i]); }
  for (int i = 0; i < N * K; ++i) { Bf[i] = (float)(rand() % 5 - 2); B[i] = __float2half(Bf[i]); }
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      float s = 0;
      for (int k = 0; k < K; ++k) s += Af[m * K + k] * Bf[n * K + k];
      ref[m * N + n] = s;
    }
  __half *dA, *dB;
  float *dD;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  const int smem = N * K * 2;
  for (int v = 0; v < 2; ++v) {
    cudaMemset(dD, 0, D.size() * 4);
    probe<<<1, 128, smem>>>(dA, dB, dD, v);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < M * N; ++i) bad += D[i] != ref[i];
    printf("TS variant %d (%s): %s, mismatches %d / %d (D[0]=%g ref %g)\n", v,
           v ? "k odd in low half" : "k even in low half", cudaGetErrorString(e), bad, M * N, D[0], ref[0]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
