// tcgen05.ld throughput by shape (sm_100a): 32x32b.x32, 16x256b.x8, 16x128b.x16,
// 16x64b.x32 -- each 4 KB per warp-instruction, 32 registers per thread.  W warps
// (warp w: lane quadrant w % 4), one wait per load; prints B/clk per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tmem_shapes tmem_shapes.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define REGS32                                                                                               \
  "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28," \
  "%29,%30,%31}"
#define OUTS32                                                                                                 \
  "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), \
      "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),   \
      "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),  \
      "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])

template <int SHAPE>
__global__ void probe(int iters, long long *out, unsigned *sink) {
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&tmem_base);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(dst));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tmem_base;
  const uint32_t base = tm + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(((warp >> 2) * 64) & 511);
  uint32_t r[32];
  unsigned acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t a = base + (uint32_t)((it & 1) * 32);
    if (SHAPE == 0)
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " REGS32 ", [%32];" : OUTS32 : "r"(a));
    else if (SHAPE == 1)
      asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 " REGS32 ", [%32];" : OUTS32 : "r"(a));
    else if (SHAPE == 2)
      asm volatile("tcgen05.ld.sync.aligned.16x128b.x16.b32 " REGS32 ", [%32];" : OUTS32 : "r"(a));
    else
      asm volatile("tcgen05.ld.sync.aligned.16x64b.x32.b32 " REGS32 ", [%32];" : OUTS32 : "r"(a));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int q = 0; q < 32; ++q) acc ^= r[q];
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int SHAPE>
void run(int warps, const char *name) {
  long long *d;
  unsigned *sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 4);
  const int iters = 4000;
  probe<SHAPE><<<148, warps * 32>>>(10, d, sink);
  cudaDeviceSynchronize();
  probe<SHAPE><<<148, warps * 32>>>(iters, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < 148; ++i) cyc += (double)h[i];
  cyc /= 148;
  printf("%-14s warps=%2d: %.1f B/clk/SM, %.0f cyc per 4 KB load (%s)\n", name, warps,
         (double)warps * iters * 4096.0 / cyc, cyc / iters, cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  for (int w : {1, 4, 8, 16}) {
    run<0>(w, "32x32b.x32");
    run<1>(w, "16x256b.x8");
    run<2>(w, "16x128b.x16");
    run<3>(w, "16x64b.x32");
  }
  return 0;
}
