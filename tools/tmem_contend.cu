// TMEM contention probe (sm_100a): one thread streams tcgen05.mma (M = 128,
// N = 128, K = 16 fp16; A from TMEM "TS" or shared memory "SS", B from shared
// memory) into TMEM columns [64, 192) while W other warps stream tcgen05.ld
// (32x32b.x32, one wait per load) or tcgen05.st on columns [256, 512) of their
// lane quadrant until the MMA stream is done.  Prints the MMA cycles per
// instruction (floor 64) and the loaders' bytes per SM clock, to see how much
// epilogue TMEM traffic slows a TS / SS MMA and vice versa.  Values are garbage.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tmem_contend tmem_contend.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

__global__ void probe(int ts, int n_load_warps, int op, int n_mma, int d_col, int a_col, int kb, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  __shared__ volatile int done;
  __shared__ unsigned long long bytes;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(&bar);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int mma_warp = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    done = 0;
    bytes = 0;
  }
  if (warp == mma_warp) {
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&tmem_base);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(dst));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(sm);
  if (warp == mma_warp) {
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const long long t0 = clock64();
      for (int i = 0; i < n_mma; ++i) {
        const uint64_t bd = desc(s0 + 32768 + (i & (kb / 16 - 1)) * 256, 128, 16 * kb);
        if (ts)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + d_col),
                       "r"(tmem + a_col + 8 * (i & 7)), "l"(bd), "r"(idesc), "r"(1));
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + d_col),
                       "l"(desc(s0 + (i & (kb / 16 - 1)) * 256, 128, 16 * kb)), "l"(bd), "r"(idesc), "r"(1));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b0));
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok)
                     : "r"(b0)
                     : "memory");
      const long long t1 = clock64();
      done = 1;
      out[2 * blockIdx.x] = t1 - t0;
    }
  } else if (warp < n_load_warps) {
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 384u + (uint32_t)(((warp >> 2) * 64) & 127);
    uint32_t v[32];
    for (int i = 0; i < 32; ++i) v[i] = threadIdx.x + i;
    unsigned acc = 0;
    unsigned long long n = 0;
    const long long t0 = clock64();
    while (!done) {
      if (op == 0) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
              "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(base + (uint32_t)((n & 1) * 32)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) acc ^= v[j];
      } else {
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
            "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(base + (uint32_t)((n & 1) * 32)),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
            "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
            "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
            "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      ++n;
    }
    const long long t1 = clock64();
    if (lane == 0) atomicAdd(&bytes, (unsigned long long)(n * 4096ull));
    if (warp == 0 && lane == 0) out[2 * blockIdx.x + 1] = t1 - t0;
    if (acc == 0x12345678u) out[0] = 0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x == 0 && n_load_warps > 0) out[2 * blockIdx.x + 1] = (long long)bytes * 1000 / (out[2 * blockIdx.x + 1] + 1);
  if (warp == mma_warp) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

static void run(int ts, int w, int op, int d_col, int a_col, int kb, long long *d_out) {
  const int n_mma = 4096;
  const int threads = (w == 0 ? 4 : w) * 32 + 32;
  probe<<<148, threads, 100 * 1024>>>(ts, w, op, n_mma, d_col, a_col, kb, d_out);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2 * 148];
  cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = 0, bw = 0;
  for (int i = 0; i < 148; ++i) {
    cyc += (double)h[2 * i];
    bw += (double)h[2 * i + 1] / 1000.0;
  }
  cyc /= 148.0 * n_mma;
  bw /= 148.0;
  printf("%s MMA N=128 D@%3d A@%3d K-region %3d + %2d warps of tcgen05.%s: %.1f cyc/MMA (floor 64), loaders %.0f B/clk/SM (%s)\n",
         ts ? "TS" : "SS", d_col, a_col, kb, w, op ? "st" : "ld", cyc, w ? bw : 0.0, cudaGetErrorString(e));
}

int main() {
  long long *d_out;
  cudaMalloc(&d_out, 2 * 148 * sizeof(long long));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  // placement / descriptor sweep, no loaders
  for (int ts = 0; ts < 2; ++ts)
    for (int kb : {64, 128})
      for (int d : {0, 64, 128, 256})
        run(ts, 0, 0, d, d == 0 ? 128 : 0, kb, d_out);
  // contention: D at 64 (the predictor's D2) and at 256
  for (int d : {64, 256})
    for (int ts = 0; ts < 2; ++ts)
      for (int op = 0; op < 2; ++op)
        for (int w : {4, 8, 16}) run(ts, w, op, d, d == 64 ? 0 : 0, 64, d_out);
  return 0;
}
