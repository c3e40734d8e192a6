// Latency probes for the predictor's MMA <-> epilogue handoffs (values are garbage):
//  1. ping-pong: one thread issues k MMAs (N = 128, TS) + commit; a second warp
//     waits on the mbarrier and arrives on another one the issuer waits on.
//     Reports cycles per round trip minus the MMA floor.
//  2. TMEM load throughput of 4 warps (32x32b.x32) with and without a long MMA
//     stream running on other TMEM columns.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_handoff umma_handoff.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph, bool sleep) {
  uint32_t done = 0;
  while (!done) {
    if (sleep)
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000;\nselp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(bar), "r"(ph)
          : "memory");
    else
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(bar), "r"(ph)
          : "memory");
  }
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(1));
}

// mode 0: ping-pong; mode 1: tmem ld alone; mode 2: tmem ld during MMA stream
__global__ void probe(int mode, int k, int rounds, int sleep, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bars[2];
  __shared__ uint32_t tmem_base;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(&bars[0]), b1 = b0 + 8;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(b1));
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
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t idesc = (1u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(sm);
  if (mode == 0) {
    if (threadIdx.x == 0) {
      long long t0 = clock64();
      for (int r = 0; r < rounds; ++r) {
        for (int i = 0; i < k; ++i) mma_ts(tmem + 256, tmem + 8 * (i & 7), desc(s0 + (i & 3) * 256, 128, 16 * 64), idesc);
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b0));
        wait(b1, r & 1, false);
        asm volatile("tcgen05.fence::after_thread_sync;");
      }
      out[blockIdx.x] = clock64() - t0;
    } else if (warp == 1) {
      for (int r = 0; r < rounds; ++r) {
        wait(b0, r & 1, sleep);
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b1) : "memory");
      }
    }
  } else {
    // warps 0..3 load columns [0, 128) of their lane quadrant; warp 4 lane 0 issues MMAs into [256, 512)
    if (warp < 4) {
      uint32_t acc = 0;
      long long t0 = clock64();
      for (int r = 0; r < rounds; ++r) {
        uint32_t v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
              "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)((r & 3) * 32)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 32; ++j) acc += v[j];
      }
      long long t1 = clock64();
      if (lane == 0 && warp == 0) out[blockIdx.x] = t1 - t0;
      if (acc == 0x12345678u) out[0] = 0;
    } else if (warp == 4 && lane == 0 && mode == 2) {
      for (int i = 0; i < 4 * rounds; ++i)
        mma_ts(tmem + 256, tmem + 128 + 8 * (i & 7), desc(s0 + (i & 3) * 256, 128, 16 * 64), idesc);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b0));
      wait(b0, 0, false);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

static double run(int mode, int k, int rounds, int sleep) {
  static long long *d_out = nullptr;
  if (!d_out) cudaMalloc(&d_out, 148 * sizeof(long long));
  probe<<<148, 160, 64 * 1024>>>(mode, k, rounds, sleep, d_out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return -1;
  }
  long long h[148];
  cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += (double)h[i];
  return avg / 148.0 / rounds;
}

int main() {
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int sleep = 0; sleep < 2; ++sleep)
    for (int k : {1, 4, 16}) {
      const double c = run(0, k, 2000, sleep);
      printf("ping-pong k=%2d MMAs (N=128 TS, floor %4d) %s: %.0f cyc/round, overhead %.0f\n", k, 64 * k,
             sleep ? "sleep-wait" : "spin-wait ", c, c - 64 * k);
    }
  const double a = run(1, 0, 4000, 0), b = run(2, 0, 4000, 0);
  printf("tmem ld x32 (4 warps, 4 KB each): alone %.1f cyc/ld (%.0f B/clk/SMSP); during MMA stream %.1f cyc/ld\n", a,
         4096.0 / a, b);
  return 0;
}
