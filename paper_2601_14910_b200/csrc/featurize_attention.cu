// Feature stage for FlashInfer FA2 attention, prefill and decode (Table V
// P:413; non-uniform causal tasks P:262; readings R4, R10-R13).
//
// Tasks: kv-head h outermost, then request b, q-block i, kv-chunk c (R4).  A
// task's demands are affine in its kv units u = kv_eff/BKV:
//   Tensor = 4*BQ*hd*BKV*u, XU = BQ*(BKV+1)*u, bytes = bpe*hd*(BQ + 2*BKV*u),
// so per SM only two numbers matter: the task count n_j (closed form under
// cyclic dealing) and the unit sum S_j.  All nkv kv-heads repeat the same
// task sequence of length L, so with A[r] = sum of u over head-0 tasks k with
// k mod N = r, the per-SM sums are the rotations S_j = sum_h A[(j - h*L) mod N]
// (exact identity of t -> t mod N with t = h*L + k).
//
// Layout: one warp per config.  Lanes take 32 consecutive head-0 tasks per
// step; the 32 SM residues are then distinct (N >= 32), so each lane updates
// its own shared-memory accumulator with a plain load/add/store.  The task
// sequence does not depend on the spec, so in SP_PAIRS_CROSS mode a warp
// accumulates once per *distinct SM count* of the spec range (the 11 GPUs of
// Table VI have 7 distinct counts) and then emits every spec of the group.
// This kernel is ALU/issue bound (a handful of integer ops per task), not HBM
// bound.
#include <cuda_runtime.h>

#include "common.cuh"

namespace sp {
namespace {

constexpr int kWarps = 8;           // warps per block
constexpr int kMaxDistinct = 16;    // distinct SM counts per group
constexpr int64_t kI32Max = 2147483647LL;
constexpr int64_t kU32Max = 4294967295LL;
constexpr unsigned __int128 kI64Max = 9223372036854775807ULL;

// Field indices (include/synperf.h, SP_ATTENTION)
enum { BS, NH, NKV, HD, BQ, BKV, CHUNK, CAUSAL, WARPS, REGS, SMEM, DTYPE };

struct DistinctSet {
  int nd;
  const int32_t *N;     // [nd] SM counts
  const int32_t *off;   // [nd] word offsets in the warp's accumulator region
  const FastDiv *fd;    // [nd] divisors N
};

__device__ __forceinline__ int64_t warp_sum64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int64_t warp_max64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, (int64_t)__shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int64_t warp_min64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, (int64_t)__shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Per-config scalars shared by all lanes.
struct AttnCfg {
  int status;
  int64_t bs, nh, nkv, hd, bq, bkv, chunk, causal, dt, g;
  const int32_t *req;
  Footprint fp;
};

__device__ __forceinline__ AttnCfg load_cfg(const ConfigView &v, int64_t c, int lane) {
  AttnCfg a{};
  int32_t f = lane < 12 ? __ldg(v.fields + (int64_t)lane * v.ld + c) : 0;
  a.bs = __shfl_sync(0xffffffffu, f, BS);
  a.nh = __shfl_sync(0xffffffffu, f, NH);
  a.nkv = __shfl_sync(0xffffffffu, f, NKV);
  a.hd = __shfl_sync(0xffffffffu, f, HD);
  a.bq = __shfl_sync(0xffffffffu, f, BQ);
  a.bkv = __shfl_sync(0xffffffffu, f, BKV);
  a.chunk = __shfl_sync(0xffffffffu, f, CHUNK);
  a.causal = __shfl_sync(0xffffffffu, f, CAUSAL);
  const int64_t warps = __shfl_sync(0xffffffffu, f, WARPS);
  const int64_t regs = __shfl_sync(0xffffffffu, f, REGS);
  const int64_t smem = __shfl_sync(0xffffffffu, f, SMEM);
  a.dt = __shfl_sync(0xffffffffu, f, DTYPE);
  const int64_t off = v.ragged_off ? __ldg(v.ragged_off + c) : -1;
  // validation, in the oracle's order (a config without requests first)
  if (off < 0) { a.status = SP_PAIR_E_DIM; return a; }
  if (a.bs < 1 || a.nh < 1 || a.nkv < 1 || a.hd < 1) { a.status = SP_PAIR_E_DIM; return a; }
  if (a.bq < 1 || a.bkv < 1 || a.chunk < 0) { a.status = SP_PAIR_E_TILE; return a; }
  if (warps < 1 || regs < 1 || smem < 0) { a.status = SP_PAIR_E_RES; return a; }
  if (a.dt != SP_BF16 && a.dt != SP_FP16) { a.status = SP_PAIR_E_DTYPE; return a; }
  if (a.nh % a.nkv != 0) { a.status = SP_PAIR_E_HEADS; return a; }
  a.g = a.nh / a.nkv;
  a.req = v.ragged + off;
  // per-request checks: the first failing request decides (dim, causal, range)
  int64_t first = INT64_MAX;
  for (int64_t b = lane; b < a.bs; b += 32) {
    const int64_t q = __ldg(a.req + 2 * b), kv = __ldg(a.req + 2 * b + 1);
    int code = 0;
    if (q < 1 || kv < 1) code = SP_PAIR_E_DIM;
    else if (a.causal && kv < q) code = SP_PAIR_E_CAUSAL;
    else if (q * a.g > kI32Max) code = SP_PAIR_E_RANGE;
    if (code) { first = min(first, b * 16 + code); break; }
  }
  first = warp_min64(first);
  if (first != INT64_MAX) { a.status = (int)(first % 16); return a; }
  a.fp.smem = smem > 0 ? smem : (a.bq + 2 * a.bkv) * a.hd * 2;
  a.fp.warps = warps;
  a.fp.regs = regs;
  return a;
}

// Advance a residue by 32 modulo N.
__device__ __forceinline__ uint32_t step32(uint32_t r, uint32_t N, const FastDiv &fd) {
  r += 32u;
  if (r >= N) r -= N;
  if (r >= N) r = fd.mod(r);
  return r;
}

// Accumulate unit value u of head-0 task position `pos` (residues r[d]) into
// every distinct slot.  Lanes of one call hold distinct positions; when
// N >= 32 their residues are distinct so a plain RMW is race-free.
__device__ __forceinline__ void accumulate(uint32_t *acc, const DistinctSet &ds, const uint32_t *r,
                                           uint32_t u, bool active) {
#pragma unroll
  for (int d = 0; d < kMaxDistinct; ++d) {
    if (d < ds.nd && active) {
      uint32_t *a = acc + ds.off[d] + r[d];
      if (ds.N[d] >= 32) *a += u;
      else atomicAdd(a, u);
    }
  }
}

// Results per distinct SM count: max_j S_j and max_j (BQ*n_j + 2*BKV*S_j).
struct DistinctMax {
  int64_t maxS, maxB;
};

// Runs the task loop of one config for every distinct SM count; returns the
// per-head task count L and unit sum U (or a RANGE status), and fills res[d].
__device__ int attn_accumulate(const AttnCfg &a, uint32_t *acc, int words, const DistinctSet &ds,
                               int lane, int64_t &L_out, int64_t &U_out, DistinctMax *res) {
  for (int w = lane * 4; w < words; w += 128) *reinterpret_cast<uint4 *>(acc + w) = make_uint4(0, 0, 0, 0);
  __syncwarp();
  FastDiv fg, fbkv;
  fg.init((uint32_t)a.g);
  fbkv.init((uint32_t)a.bkv);
  int64_t base = 0;     // head-0 task index of the current request's first task
  int64_t usum = 0;     // per-lane partial of U
  int status = 0;
  uint32_t r[kMaxDistinct];
  for (int64_t b = 0; b < a.bs && status == 0; ++b) {
    const int64_t qlen = __ldg(a.req + 2 * b), kvlen = __ldg(a.req + 2 * b + 1);
    const int64_t rows = qlen * a.g;
    const int64_t nqb = cdiv64(rows, a.bq);
    const bool split = a.chunk > 0;
    if (!split || !a.causal) {
      // every q-block has the same chunk count (unsplit, or non-causal kv_need = kvlen)
      const int64_t n_ch = split ? cdiv64(kvlen, a.chunk) : 1;
      const int64_t tasks = nqb * n_ch;
      if (base + tasks > kI32Max) { status = SP_PAIR_E_RANGE; break; }
      FastDiv fch;
      fch.init((uint32_t)n_ch);
      const uint32_t u_full = split ? (uint32_t)cdiv64(min(a.chunk, kvlen), a.bkv) : 0;
      const uint32_t u_last = split ? (uint32_t)cdiv64(kvlen - (n_ch - 1) * a.chunk, a.bkv) : 0;
#pragma unroll
      for (int d = 0; d < kMaxDistinct; ++d)
        if (d < ds.nd) r[d] = ds.fd[d].mod((uint32_t)(base + lane));
      for (int64_t k0 = 0; k0 < tasks; k0 += 32) {
        const int64_t k = k0 + lane;
        const bool active = k < tasks;
        uint32_t u = 0;
        if (active) {
          if (split) {  // non-causal: kv_need = kvlen for every q-block
            const uint32_t ch = fch.mod((uint32_t)k);
            u = ch == (uint32_t)(n_ch - 1) ? u_last : u_full;
          } else {
            // q_last = floor((min((i+1)BQ, rows) - 1) / g); kv_need (causal) = min(kvlen, kvlen - qlen + q_last + 1)
            const int64_t end = min((k + 1) * a.bq, rows) - 1;
            const int64_t q_last = fg.div((uint32_t)end);
            const int64_t need = a.causal ? min(kvlen, kvlen - qlen + q_last + 1) : kvlen;
            u = fbkv.div((uint32_t)(need + a.bkv - 1));
          }
        }
        accumulate(acc, ds, r, u, active);
        usum += u;
        __syncwarp();
#pragma unroll
        for (int d = 0; d < kMaxDistinct; ++d)
          if (d < ds.nd) r[d] = step32(r[d], (uint32_t)ds.N[d], ds.fd[d]);
      }
      base += tasks;
    } else {
      // causal + split-KV: each q-block has its own chunk count.  Lanes take
      // 32 q-blocks, scan their chunk counts, then walk their own chunks
      // (positions are no longer lane-consecutive: atomic adds).
      for (int64_t i0 = 0; i0 < nqb && status == 0; i0 += 32) {
        const int64_t i = i0 + lane;
        int64_t need = 0, n_ch = 0;
        if (i < nqb) {
          const int64_t end = min((i + 1) * a.bq, rows) - 1;
          const int64_t q_last = fg.div((uint32_t)end);
          need = min(kvlen, kvlen - qlen + q_last + 1);
          n_ch = cdiv64(need, a.chunk);
        }
        int64_t incl = n_ch;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        const int64_t total = __shfl_sync(0xffffffffu, incl, 31);
        if (base + total > kI32Max) { status = SP_PAIR_E_RANGE; break; }
        const int64_t start = base + incl - n_ch;
        for (int64_t ch = 0; ch < n_ch; ++ch) {
          const int64_t len = min(a.chunk, need - ch * a.chunk);
          const uint32_t u = (uint32_t)cdiv64(len, a.bkv);
          const uint32_t pos = (uint32_t)(start + ch);
#pragma unroll
          for (int d = 0; d < kMaxDistinct; ++d)
            if (d < ds.nd) atomicAdd(acc + ds.off[d] + ds.fd[d].mod(pos), u);
          usum += u;
        }
        base += total;
        __syncwarp();
      }
    }
  }
  const int64_t U = warp_sum64(usum);
  const int64_t L = base;
  if (status == 0 && (U > kU32Max || L * a.nkv > kI32Max)) status = SP_PAIR_E_RANGE;
  L_out = L;
  U_out = U;
  if (status) return status;
  __syncwarp();
  // fold the nkv rotations and take the per-quantity maxima per distinct N
  const int64_t T = L * a.nkv;
  for (int d = 0; d < ds.nd; ++d) {
    const int64_t N = ds.N[d];
    const uint32_t Lm = ds.fd[d].mod((uint32_t)L);
    const uint32_t *A = acc + ds.off[d];
    int64_t mS = 0, mB = 0;
    for (int64_t s = lane; s < N; s += 32) {
      int64_t S = 0;
      int64_t o = 0;  // (h * L) mod N
      for (int64_t h = 0; h < a.nkv; ++h) {
        int64_t idx = s - o;
        if (idx < 0) idx += N;
        S += A[idx];
        o += Lm;
        if (o >= N) o -= N;
      }
      const int64_t n_s = s < T ? (T - s - 1) / N + 1 : 0;
      mS = max(mS, S);
      mB = max(mB, a.bq * n_s + 2 * a.bkv * S);
    }
    mS = warp_max64(mS);
    mB = warp_max64(mB);
    if (lane == 0) res[d] = DistinctMax{mS, mB};
  }
  __syncwarp();
  return 0;
}

typedef unsigned __int128 u128;

// a*b, flagging (bad = true) a product above INT64_MAX without overflowing:
// operands are each < 2^96 here, so either one exceeds 2^63 (and the other is
// nonzero) or the product is < 2^126.
__device__ __forceinline__ u128 mul_le_i64(u128 a, u128 b, bool &bad) {
  if (a == 0 || b == 0) return 0;
  if (a > kI64Max || b > kI64Max) { bad = true; return 0; }
  return a * b;
}

// One (config, spec) record from the accumulated per-distinct maxima.
__device__ __forceinline__ void attn_emit(const FeatOut &out, int64_t p, const AttnCfg &a, int cfg_status,
                                          int64_t L, int64_t U, const DistinctMax &m, const DevSpec &s) {
  if (cfg_status) { emit_error(out, p, cfg_status); return; }
  const int tdt = (int)a.dt;
  if (!s.tensor_ok[tdt]) { emit_error(out, p, SP_PAIR_E_DTYPE); return; }
  const int64_t T = L * a.nkv;
  const u128 Ua = (u128)U * (u128)a.nkv;  // < 2^63 (U < 2^32, nkv < 2^31)
  bool bad = false;
  const u128 totT = mul_le_i64((u128)(4 * a.bq) * (u128)a.hd * (u128)a.bkv, Ua, bad);
  const u128 totX = mul_le_i64((u128)a.bq * (u128)(a.bkv + 1), Ua, bad);
  const u128 totB = mul_le_i64((u128)(2 * a.hd), (u128)a.bq * (u128)T + (u128)(2 * a.bkv) * Ua, bad);
  if (bad || totT > kI64Max || totX > kI64Max || totB > kI64Max) { emit_error(out, p, SP_PAIR_E_RANGE); return; }
  PairDemand d;
  d.T = T;
  d.tot[0] = (int64_t)totT;
  d.tot[1] = 0;
  d.tot[2] = (int64_t)totX;
  d.tot[3] = (int64_t)totB;
  d.mx[0] = 4 * a.bq * a.hd * a.bkv * m.maxS;
  d.mx[1] = 0;
  d.mx[2] = a.bq * (a.bkv + 1) * m.maxS;
  d.mx[3] = 2 * a.hd * m.maxB;
  emit_pair(out, p, d, a.fp, s, 5, tdt);
}

__global__ void __launch_bounds__(kWarps * 32) featurize_attention_cross(ConfigView cfg,
                                                                         const DevSpec *__restrict__ specs,
                                                                         int g0, AttnPlan plan, FeatOut out) {
  extern __shared__ uint32_t smem[];
  __shared__ int32_t s_N[kMaxDistinct], s_off[kMaxDistinct];
  __shared__ FastDiv s_fd[kMaxDistinct];
  __shared__ DistinctMax s_res[kWarps][kMaxDistinct];
  const AttnGroup grp = plan.groups[blockIdx.y];
  if (threadIdx.x < grp.n_distinct) {
    const int n = plan.distinct_n[grp.distinct_first + threadIdx.x];
    s_N[threadIdx.x] = n;
    s_off[threadIdx.x] = plan.distinct_off[grp.distinct_first + threadIdx.x];
    s_fd[threadIdx.x].init((uint32_t)n);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t *acc = smem + (size_t)warp * plan.words_per_warp;
  const DistinctSet ds{grp.n_distinct, s_N, s_off, s_fd};
  int words = 0;
  for (int d = 0; d < grp.n_distinct; ++d) words = max(words, s_off[d] + s_N[d]);
  words = (words + 3) & ~3;
  const int64_t C = cfg.n_configs;
  for (int64_t c = (int64_t)blockIdx.x * kWarps + warp; c < C; c += (int64_t)gridDim.x * kWarps) {
    const AttnCfg a = load_cfg(cfg, c, lane);
    int st = a.status;
    int64_t L = 0, U = 0;
    if (st == 0) st = attn_accumulate(a, acc, words, ds, lane, L, U, s_res[warp]);
    for (int j = lane; j < grp.n_specs; j += 32) {
      const int g = plan.group_specs[grp.spec_first + j];
      const int d = plan.spec_dist[grp.spec_first + j] - grp.distinct_first;
      const int64_t p = (int64_t)(g - g0) * C + c;
      attn_emit(out, p, a, st, L, U, s_res[warp][d], specs[g]);
    }
    __syncwarp();
  }
}

__global__ void __launch_bounds__(kWarps * 32) featurize_attention_list(ConfigView cfg,
                                                                        const DevSpec *__restrict__ specs,
                                                                        int n_specs, int words_per_warp,
                                                                        int64_t n_pairs,
                                                                        const int64_t *__restrict__ cfg_idx,
                                                                        const int32_t *__restrict__ spec_idx,
                                                                        FeatOut out) {
  extern __shared__ uint32_t smem[];
  __shared__ int32_t s_N[kWarps], s_off[kWarps];
  __shared__ FastDiv s_fd[kWarps];
  __shared__ DistinctMax s_res[kWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t *acc = smem + (size_t)warp * words_per_warp;
  for (int64_t p = (int64_t)blockIdx.x * kWarps + warp; p < n_pairs; p += (int64_t)gridDim.x * kWarps) {
    const int64_t c = __ldg(cfg_idx + p);
    const int32_t g = __ldg(spec_idx + p);
    if (c < 0 || c >= cfg.n_configs || g < 0 || g >= n_specs) {
      if (lane == 0) emit_error(out, p, SP_PAIR_E_INDEX);
      continue;
    }
    const int N = specs[g].num_sms;
    if (lane == 0) {
      s_N[warp] = N;
      s_off[warp] = 0;
      s_fd[warp].init((uint32_t)N);
    }
    __syncwarp();
    const DistinctSet ds{1, s_N + warp, s_off + warp, s_fd + warp};
    const AttnCfg a = load_cfg(cfg, c, lane);
    int st = a.status;
    int64_t L = 0, U = 0;
    if (st == 0) st = attn_accumulate(a, acc, (N + 3) & ~3, ds, lane, L, U, s_res + warp);
    if (lane == 0) attn_emit(out, p, a, st, L, U, s_res[warp], specs[g]);
    __syncwarp();
  }
}

}  // namespace

int launch_featurize_attention(const ConfigView &cfg, const DevSpec *specs, int spec_begin,
                               int n_specs, const AttnPlan &plan, int64_t n_pairs, const int64_t *cfg_idx,
                               const int32_t *spec_idx, int32_t max_sms, const FeatOut &out,
                               int num_device_sms, void *stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (cfg_idx == nullptr) {
    if (cfg.n_configs == 0 || plan.n_groups == 0) return 0;
    const size_t smem = (size_t)kWarps * plan.words_per_warp * 4;
    cudaError_t e = cudaFuncSetAttribute(featurize_attention_cross,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    int64_t want = (cfg.n_configs + kWarps - 1) / kWarps;
    int64_t cap = (int64_t)num_device_sms * 16;
    dim3 grid((unsigned)(want < cap ? want : cap), (unsigned)plan.n_groups);
    featurize_attention_cross<<<grid, kWarps * 32, smem, st>>>(cfg, specs, spec_begin, plan, out);
  } else {
    if (n_pairs == 0) return 0;
    const int words = (max_sms + 3) & ~3;
    const size_t smem = (size_t)kWarps * words * 4;
    cudaError_t e = cudaFuncSetAttribute(featurize_attention_list,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    int64_t want = (n_pairs + kWarps - 1) / kWarps;
    int64_t cap = (int64_t)num_device_sms * 16;
    featurize_attention_list<<<(unsigned)(want < cap ? want : cap), kWarps * 32, smem, st>>>(
        cfg, specs, n_specs, words, n_pairs, cfg_idx, spec_idx, out);
  }
  return (int)cudaGetLastError();
}

}  // namespace sp
