// TMEM load/store bandwidth probe (sm_100a): W warps per CTA (warp w reads
// lane quadrant w % 4), each doing `iters` rounds of NLD tcgen05.ld
// 32x32b.x32 (4 KB per warp-instruction) followed by one wait::ld; or the
// same with tcgen05.st.  One CTA per SM; prints bytes per SM clock.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tmem_bw tmem_bw.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define LD32(addr, r)                                                                                         \
  asm volatile(                                                                                               \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                          \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),        \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),  \
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), \
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])  \
      : "r"(addr))
#define ST32(addr, r)                                                                                          \
  asm volatile(                                                                                                \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17," \
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),                              \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),         \
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),  \
      "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), \
      "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]))

#define LD16(addr, r)                                                                                         \
  asm volatile(                                                                                               \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"   \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),        \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])   \
      : "r"(addr))

// NLD x16 loads (2 KB each) into distinct registers before one wait
template <int NLD>
__global__ void probe16(int iters, long long *out, unsigned *sink) {
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
  const uint32_t base = tm + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(((warp >> 2) * 128) & 511);
  uint32_t r[NLD][16];
  unsigned acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < NLD; ++k) LD16(base + (uint32_t)(16 * (k & 7)), r[k]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int k = 0; k < NLD; ++k)
#pragma unroll
      for (int q = 0; q < 16; ++q) acc ^= r[k][q];  // static indices: registers, not local memory
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int NLD>
void run16(int warps) {
  long long *d;
  unsigned *sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 4);
  const int iters = 2000;
  probe16<NLD><<<148, warps * 32>>>(10, d, sink);
  cudaDeviceSynchronize();
  probe16<NLD><<<148, warps * 32>>>(iters, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < 148; ++i) cyc += (double)h[i];
  cyc /= 148;
  const double bytes = (double)warps * iters * NLD * 2048.0;
  printf("ld16 warps=%2d per_wait=%d (%d KB/round): %.1f B/clk/SM, %.0f cyc/round (%s)\n", warps, NLD, NLD * 2,
         bytes / cyc, cyc / iters, cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(sink);
}

template <int NLD, bool ST>
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
  const int nw = blockDim.x >> 5;
  // warp w: quadrant w % 4, column block (w / 4) * 128 (distinct columns per warp of a quadrant)
  const uint32_t base = tm + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(((warp >> 2) * 128) & 511);
  uint32_t r[32];
  for (int i = 0; i < 32; ++i) r[i] = threadIdx.x + i;
  unsigned acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < NLD; ++k) {
      if (ST) {
        ST32(base + (uint32_t)(32 * (k & 3)), r);
      } else {
        LD32(base + (uint32_t)(32 * (k & 3)), r);
      }
    }
    if (ST) {
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int q = 0; q < 32; ++q) acc ^= r[q];  // static indices: registers, not local memory
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[0] = acc;
  (void)nw;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int NLD, bool ST>
void run(int warps) {
  long long *d;
  unsigned *sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 4);
  const int iters = 2000;
  probe<NLD, ST><<<148, warps * 32>>>(10, d, sink);
  cudaDeviceSynchronize();
  probe<NLD, ST><<<148, warps * 32>>>(iters, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < 148; ++i) cyc += (double)h[i];
  cyc /= 148;
  const double bytes = (double)warps * iters * NLD * 4096.0;
  printf("%s warps=%2d per_wait=%d: %.1f B/clk/SM (%s)\n", ST ? "st" : "ld", warps, NLD, bytes / cyc,
         cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  for (int w : {1, 2, 4, 8, 16}) {
    run<1, false>(w);
    run<2, false>(w);
    run<4, false>(w);
  }
  for (int w : {4, 8, 16}) {
    run<1, true>(w);
    run<4, true>(w);
  }
  for (int w : {1, 4, 8, 16}) {
    run16<1>(w);
    run16<2>(w);
    run16<4>(w);
    run16<8>(w);
    run16<16>(w);
  }
  return 0;
}
