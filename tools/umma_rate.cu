// Issue-rate probe for tcgen05.mma kind::f16 (M = 128, cta_group::1): cycles
// per MMA for A from shared memory ("SS") or TMEM ("TS"), B from shared
// memory with no swizzle or 128B swizzle, N in {64, 128, 256}.  Values are
// garbage (rate only).  One CTA per SM, one issuing thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_rate umma_rate.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}

template <bool TS>
__global__ void rate(int N, int swz, int iters, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const uint32_t mbar_s = (uint32_t)__cvta_generic_to_shared(&mbar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar_s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&tmem_base);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(dst));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(sm);
    // B: N rows x K=64 (4 K-steps) region at s0 + 32 KB; A (SS): 128 x 64 at s0
    const uint32_t layout = swz ? 2u : 0u;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int ks = it & 3;
      uint64_t db, da;
      if (swz) {  // 128B swizzle K-major: 8-row atoms of 1024 B, K step = +32 B
        db = desc(s0 + 32768 + ks * 32, 16, 1024, layout);
        da = desc(s0 + ks * 32, 16, 1024, layout);
      } else {
        db = desc(s0 + 32768 + ks * 256, 128, 16 * 64, 0);
        da = desc(s0 + ks * 256, 128, 16 * 64, 0);
      }
      const uint32_t d = tmem + 256;
      if (TS) {
        const uint32_t a = tmem + ks * 8;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
            "r"(a), "l"(db), "r"(idesc), "r"(1));
      } else {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
            "l"(da), "l"(db), "r"(idesc), "r"(1));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar_s));
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(mbar_s), "r"(0u));
    }
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  long long *d_out;
  cudaMalloc(&d_out, 148 * sizeof(long long));
  const int smem = 96 * 1024;
  cudaFuncSetAttribute(rate<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(rate<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  for (int ts = 0; ts < 2; ++ts)
    for (int swz = 0; swz < 2; ++swz)
      for (int N = 64; N <= 256; N *= 2) {
        if (ts) rate<true><<<148, 128, smem>>>(N, swz, iters, d_out);
        else rate<false><<<148, 128, smem>>>(N, swz, iters, d_out);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 148; ++i) avg += (double)h[i];
        avg /= 148.0 * iters;
        const double floor_ = 128.0 * N / 256.0;
        printf("%s swz=%d N=%3d: %.1f cyc/MMA (floor %.0f, %.0f%%) %s\n", ts ? "TS" : "SS", swz, N, avg, floor_,
               100.0 * floor_ / avg, cudaGetErrorString(e));
      }
  return 0;
}
