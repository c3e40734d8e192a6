// Feature stage for the uniform-task families: GEMM (Table V), fused MoE
// (P:419), RMSNorm, SiLU&Mul.
//
// Every task of these kernels has the same demands (padded tiles R2, one task
// per row for the row-wise kernels), so the round-robin schedule (Eq.2, R5)
// has a closed form: SM j holds ceil((T - j)/N) tasks and the busiest SM holds
// ceil(T/N).  Per pair the work is O(1): no task list, no loop.
//
// Layout: one thread per config, looping over a tile of specs staged in shared
// memory; for each spec the thread writes pair p = (g - g0)*C + c, so a warp's
// stores to every SoA row are 32 consecutive elements (coalesced).  Config
// invariants (T, per-task demands, footprint, status) are computed once per
// config and reused across the spec tile.  The kernel is bound by the
// 137 B/pair record written to HBM.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>

#include "common.cuh"

namespace sp {
namespace {

constexpr int kThreads = 256;
constexpr int kSpecTile = 16;
constexpr int64_t kI32Max = 2147483647LL;
constexpr unsigned __int128 kI64Max = 9223372036854775807ULL;

struct UniformCfg {
  int status;       // config-level status (validation order of the oracle)
  int range_bad;    // totals do not fit in int64 (checked after the spec dtype check)
  int tdt;          // tensor dtype index: 0 bf16, 1 fp16, -1 none
  int64_t T;
  int64_t task[4];  // per-task Tensor, FMA, XU ops, load bytes
  int64_t tot[4];
  Footprint fp;
};

__device__ __forceinline__ int32_t fld(const ConfigView &v, int k, int64_t c) {
  return __ldg(v.fields + (int64_t)k * v.ld + c);
}

// ceil(a/b) for 1 <= a, b < 2^31 (config fields and their products checked
// below 2^31): one 32-bit division instead of the 64-bit software routine.
__device__ __forceinline__ int64_t cdiv31(int64_t a, int64_t b) {
  return (int64_t)(((uint32_t)a + (uint32_t)b - 1u) / (uint32_t)b);
}

__device__ __forceinline__ int64_t sat40(unsigned __int128 x) {
  const unsigned __int128 lim = (unsigned __int128)1 << 40;
  return (int64_t)(x > lim ? lim : x);
}

// Task demands and totals with the exact-range rule (R22): uniform tasks, so
// tot = T * task; all in 128-bit before narrowing.
__device__ __forceinline__ void finish_totals(UniformCfg &u, const unsigned __int128 task[4]) {
  u.range_bad = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    unsigned __int128 t = task[q] * (unsigned __int128)u.T;
    if (task[q] > kI64Max || t > kI64Max) u.range_bad = 1;
    u.task[q] = (int64_t)task[q];
    u.tot[q] = (int64_t)t;
  }
}

// GEMM: T = ceil(M/tm) * ceil(N/tn); task = 2*tm*tn*K_pad Tensor ops, (tm+tn)*K_pad*bpe bytes
// (Eq.3 alpha = 2; R1, R2); smem default stages*(tm+tn)*BK*bpe.
__device__ UniformCfg gemm_cfg(const ConfigView &v, int64_t c) {
  UniformCfg u{};
  const int64_t M = fld(v, 0, c), N = fld(v, 1, c), K = fld(v, 2, c), tm = fld(v, 3, c),
                tn = fld(v, 4, c), bk = fld(v, 5, c), stages = fld(v, 6, c), warps = fld(v, 7, c),
                regs = fld(v, 8, c), smem = fld(v, 9, c), dt = fld(v, 10, c);
  if (M < 1 || N < 1 || K < 1) { u.status = SP_PAIR_E_DIM; return u; }
  if (tm < 1 || tn < 1 || bk < 1 || stages < 1) { u.status = SP_PAIR_E_TILE; return u; }
  if (warps < 1 || regs < 1 || smem < 0) { u.status = SP_PAIR_E_RES; return u; }
  if (dt != SP_BF16 && dt != SP_FP16) { u.status = SP_PAIR_E_DTYPE; return u; }
  const int64_t T = cdiv31(M, tm) * cdiv31(N, tn);
  if (T > kI32Max) { u.status = SP_PAIR_E_RANGE; return u; }
  u.T = T;
  u.tdt = (int)dt;
  const int64_t kpad = cdiv31(K, bk) * bk;
  unsigned __int128 task[4] = {(unsigned __int128)(2 * tm * tn) * kpad, 0, 0,
                               (unsigned __int128)(tm + tn) * kpad * 2};
  finish_totals(u, task);
  u.fp.smem = smem > 0 ? smem : sat40((unsigned __int128)stages * (tm + tn) * bk * 2);
  u.fp.warps = warps;
  u.fp.regs = regs;
  return u;
}

// Histogram pass of a fused-MoE config (R16): sum of the per-expert token
// counts, any negative count, and sum_e ceil(t_e/BM).
struct MoeHist {
  int64_t sum = 0;
  int64_t mblocks = 0;
  int neg = 0;
};

// Warp-cooperative histogram pass for the (up to) 32 configs of a warp, lane j
// holding config c0 + j: the warp takes its configs four at a time, its lanes
// reading 32 consecutive counts per config (coalesced; the first 128 counts of
// all four configs are loaded before any is reduced, so four histograms are in
// flight instead of one), and reduces with REDUX (32-bit partials; see take()).
// A saturated or negative partial marks the histogram invalid (`neg`: moe_cfg
// reports SP_PAIR_E_HIST, as for a sum that differs from M topk).  Lane j
// receives config j's result.  All 32 lanes must call it.
__device__ __forceinline__ MoeHist moe_hist_warp(const ConfigView &v, int64_t c, bool valid) {
  const int lane = threadIdx.x & 31;
  int64_t off = -1;
  int32_t E = 0, bm = 0;
  if (valid && v.ragged_off) {
    off = __ldg(v.ragged_off + c);
    E = fld(v, 1, c);
    bm = fld(v, 5, c);
  }
  MoeHist mine;
  // FastDiv of this lane's own BM, once per lane (its init is a 64-bit division;
  // done warp-uniformly per config it was most of the pre-pass's instructions)
  FastDiv my_fbm{1u, 1u, 0u};
  if (off >= 0 && E >= 1 && bm >= 1) my_fbm.init((uint32_t)bm);
  unsigned need = __ballot_sync(0xffffffffu, off >= 0 && E >= 1 && bm >= 1);
  while (need) {
    int jj[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      jj[q] = need ? __ffs(need) - 1 : -1;
      need &= need - 1;
    }
    int64_t oj[4];
    int32_t Ej[4];
    int32_t t[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // issue every load first
      const int src = jj[q] < 0 ? 0 : jj[q];
      oj[q] = __shfl_sync(0xffffffffu, off, src);
      Ej[q] = jj[q] < 0 ? 0 : __shfl_sync(0xffffffffu, E, src);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int32_t e = lane + 32 * r;
        t[q][r] = e < Ej[q] ? __ldg(v.ragged + oj[q] + e) : 0;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (jj[q] < 0) break;  // warp-uniform
      const uint32_t bmj = (uint32_t)__shfl_sync(0xffffffffu, bm, jj[q]);
      // ceil(t_e / BM) = (max(t_e, 1) - 1) / BM + [t_e > 0] by multiply-high (operand < 2^31)
      const FastDiv fbm{bmj, __shfl_sync(0xffffffffu, my_fbm.m, jj[q]), __shfl_sync(0xffffffffu, my_fbm.s, jj[q])};
      // 32-bit lane partials: `ors` collects the sign bits (a negative count), `sum`
      // saturates at 2^31 (a valid histogram sums to M topk < 2^31, so a saturated
      // partial is an invalid one either way), `mb` is exact whenever the
      // histogram is valid (sum_e ceil(t_e/BM) <= sum_e t_e < 2^31)
      uint32_t ors = 0, sum = 0, mb = 0;
      auto take = [&](int32_t te) {
        ors |= (uint32_t)te;
        sum = min(sum + (uint32_t)te, 1u << 31);  // sum <= 2^31, te < 2^31 when ors keeps bit 31 clear
        mb += fbm.div31((uint32_t)max(te, 1) - 1u) + (te > 0 ? 1u : 0u);
      };
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (32 * r < Ej[q]) take(t[q][r]);  // warp-uniform: rows past E hold no counts
      for (int32_t e = lane + 128; e < Ej[q]; e += 32) take(__ldg(v.ragged + oj[q] + e));  // E > 128
      // warp totals by REDUX: the sum as two 16-bit halves (each total < 2^21), exact
      const int neg = __any_sync(0xffffffffu, (ors >> 31) != 0 || sum >= (1u << 31));
      const uint32_t s_hi = __reduce_add_sync(0xffffffffu, sum >> 16), s_lo = __reduce_add_sync(0xffffffffu, sum & 0xffffu);
      const uint32_t mbt = __reduce_add_sync(0xffffffffu, mb);
      if (lane == jj[q]) {
        mine.sum = ((int64_t)s_hi << 16) + (int64_t)s_lo;
        mine.mblocks = mbt;
        mine.neg = neg;
      }
    }
  }
  return mine;
}

// Scaled MM (reading R23): GEMM tiles with one-byte FP8 operands
// at the spec's FP8 tensor rate, plus the block-wise fp32 scales each task
// loads: A scales tm x ceil(K/128), B scales ceil(tn/128) x ceil(K/128).
__device__ UniformCfg scaled_mm_cfg(const ConfigView &v, int64_t c) {
  UniformCfg u{};
  const int64_t M = fld(v, 0, c), N = fld(v, 1, c), K = fld(v, 2, c), tm = fld(v, 3, c),
                tn = fld(v, 4, c), bk = fld(v, 5, c), stages = fld(v, 6, c), warps = fld(v, 7, c),
                regs = fld(v, 8, c), smem = fld(v, 9, c), dt = fld(v, 10, c);
  if (M < 1 || N < 1 || K < 1) { u.status = SP_PAIR_E_DIM; return u; }
  if (tm < 1 || tn < 1 || bk < 1 || stages < 1) { u.status = SP_PAIR_E_TILE; return u; }
  if (warps < 1 || regs < 1 || smem < 0) { u.status = SP_PAIR_E_RES; return u; }
  if (dt != SP_FP8) { u.status = SP_PAIR_E_DTYPE; return u; }
  const int64_t T = cdiv31(M, tm) * cdiv31(N, tn);
  if (T > kI32Max) { u.status = SP_PAIR_E_RANGE; return u; }
  u.T = T;
  u.tdt = 2;
  const int64_t kpad = cdiv31(K, bk) * bk, kb = cdiv31(K, 128);
  unsigned __int128 task[4] = {(unsigned __int128)(2 * tm * tn) * kpad, 0, 0,
                               (unsigned __int128)(tm + tn) * kpad +
                                   ((unsigned __int128)tm + (unsigned __int128)cdiv31(tn, 128)) * kb * 4};
  finish_totals(u, task);
  u.fp.smem = smem > 0 ? smem : sat40((unsigned __int128)stages * (tm + tn) * bk);
  u.fp.warps = warps;
  u.fp.regs = regs;
  return u;
}

// Split-K GEMM (reading R25; cuBLAS split-K): the kt = ceil(K/BK)
// k-tiles are cut into S' = ceil(kt/kps) slices of kps = ceil(kt/SPLIT_K); the
// task list is slice-major (grid z last), tiles row-major inside a slice.  Two
// task classes: the Ta = (S'-1)*tiles tasks of full slices (kps k-tiles) come
// first, then the `tiles` tasks of the last slice (kt - (S'-1)*kps k-tiles).
struct SplitKCfg {
  UniformCfg u;      // u.task = full-slice task, u.tot = totals over both classes
  int64_t Ta;        // tasks of the full slices (a prefix of the task list)
  int64_t taskb[4];  // last-slice task
};

__device__ SplitKCfg splitk_cfg(const ConfigView &v, int64_t c) {
  SplitKCfg r{};
  UniformCfg &u = r.u;
  const int64_t M = fld(v, 0, c), N = fld(v, 1, c), K = fld(v, 2, c), tm = fld(v, 3, c),
                tn = fld(v, 4, c), bk = fld(v, 5, c), split = fld(v, 6, c), stages = fld(v, 7, c),
                warps = fld(v, 8, c), regs = fld(v, 9, c), smem = fld(v, 10, c), dt = fld(v, 11, c);
  if (M < 1 || N < 1 || K < 1) { u.status = SP_PAIR_E_DIM; return r; }
  if (tm < 1 || tn < 1 || bk < 1 || split < 1 || stages < 1) { u.status = SP_PAIR_E_TILE; return r; }
  if (warps < 1 || regs < 1 || smem < 0) { u.status = SP_PAIR_E_RES; return r; }
  if (dt != SP_BF16 && dt != SP_FP16) { u.status = SP_PAIR_E_DTYPE; return r; }
  const int64_t kt = cdiv31(K, bk), kps = cdiv31(kt, split), slices = cdiv31(kt, kps);
  const int64_t tiles = cdiv31(M, tm) * cdiv31(N, tn);  // <= 2^31 * 2^31 / 1: fits in int64
  if ((unsigned __int128)tiles * (unsigned __int128)slices > (unsigned __int128)kI32Max) {
    u.status = SP_PAIR_E_RANGE;
    return r;
  }
  u.T = tiles * slices;
  u.tdt = (int)dt;
  r.Ta = tiles * (slices - 1);
  const int64_t klast = kt - (slices - 1) * kps;
  const unsigned __int128 ta[4] = {(unsigned __int128)(2 * tm * tn) * (kps * bk), 0, 0,
                                   (unsigned __int128)(tm + tn) * (kps * bk) * 2};
  const unsigned __int128 tb[4] = {(unsigned __int128)(2 * tm * tn) * (klast * bk), 0, 0,
                                   (unsigned __int128)(tm + tn) * (klast * bk) * 2};
  u.range_bad = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const unsigned __int128 t = ta[q] * (unsigned __int128)r.Ta + tb[q] * (unsigned __int128)tiles;
    if (ta[q] > kI64Max || t > kI64Max) u.range_bad = 1;
    u.task[q] = (int64_t)ta[q];
    r.taskb[q] = (int64_t)tb[q];
    u.tot[q] = (int64_t)t;
  }
  u.fp.smem = smem > 0 ? smem : sat40((unsigned __int128)stages * (tm + tn) * bk * 2);
  u.fp.warps = warps;
  u.fp.regs = regs;
  return r;
}

// Fused MoE (R16): t_e from the histogram or the balanced split; tasks are
// padded BM x BN x H_pad tiles: T = sum_e ceil(t_e/BM) * ceil(N/BN).
// `hist`: this config's histogram pass (moe_hist_warp), or nullptr to walk it here.
__device__ UniformCfg moe_cfg(const ConfigView &v, int64_t c, const MoeHist *hist) {
  UniformCfg u{};
  const int64_t M = fld(v, 0, c), E = fld(v, 1, c), topk = fld(v, 2, c), H = fld(v, 3, c),
                N = fld(v, 4, c), bm = fld(v, 5, c), bn = fld(v, 6, c), bk = fld(v, 7, c),
                stages = fld(v, 9, c), warps = fld(v, 10, c), regs = fld(v, 11, c),
                smem = fld(v, 12, c), dt = fld(v, 13, c);
  if (M < 1 || E < 1 || topk < 1 || H < 1 || N < 1) { u.status = SP_PAIR_E_DIM; return u; }
  if (bm < 1 || bn < 1 || bk < 1 || stages < 1) { u.status = SP_PAIR_E_TILE; return u; }
  if (warps < 1 || regs < 1 || smem < 0) { u.status = SP_PAIR_E_RES; return u; }
  if (dt != SP_BF16 && dt != SP_FP16) { u.status = SP_PAIR_E_DTYPE; return u; }
  const int64_t mt = M * topk;
  if (mt > kI32Max) { u.status = SP_PAIR_E_RANGE; return u; }
  const int64_t off = v.ragged_off ? __ldg(v.ragged_off + c) : -1;
  unsigned __int128 mblocks = 0;
  if (off >= 0 && hist) {
    if (hist->neg || hist->sum != mt) { u.status = SP_PAIR_E_HIST; return u; }
    mblocks = (unsigned __int128)hist->mblocks;
  } else if (off >= 0) {
    const int32_t *h = v.ragged + off;
    int64_t sum = 0;
    for (int64_t e = 0; e < E; ++e) {
      const int64_t te = __ldg(h + e);
      if (te < 0) { u.status = SP_PAIR_E_HIST; return u; }
      sum += te;
    }
    if (sum != mt) { u.status = SP_PAIR_E_HIST; return u; }
    for (int64_t e = 0; e < E; ++e) mblocks += cdiv64(__ldg(h + e), bm);
  } else {
    const int64_t q = (uint32_t)mt / (uint32_t)E, r = mt - q * E;  // mt < 2^31 (checked above)
    mblocks = (unsigned __int128)r * cdiv31(q + 1, bm) + (unsigned __int128)(E - r) * cdiv31(q, bm);
  }
  const unsigned __int128 T = mblocks * (unsigned __int128)cdiv31(N, bn);
  if (T > (unsigned __int128)kI32Max) { u.status = SP_PAIR_E_RANGE; return u; }
  u.T = (int64_t)T;
  u.tdt = (int)dt;
  const int64_t hpad = cdiv31(H, bk) * bk;
  unsigned __int128 task[4] = {(unsigned __int128)(2 * bm * bn) * hpad, 0, 0,
                               (unsigned __int128)(bm + bn) * hpad * 2};
  finish_totals(u, task);
  u.fp.smem = smem > 0 ? smem : sat40((unsigned __int128)stages * (bm + bn) * bk * 2);
  u.fp.warps = warps;
  u.fp.regs = regs;
  return u;
}

// RMSNorm (R14): per row FMA 3*dim, XU 1, bytes 2*dim*bpe.
// SiLU&Mul (R15): per row FMA 4*dim, XU 2*dim, bytes 2*dim*bpe.  One task per row.
__device__ UniformCfg rowwise_cfg(const ConfigView &v, int64_t c, bool silu) {
  UniformCfg u{};
  const int64_t seq = fld(v, 0, c), dim = fld(v, 1, c), warps = fld(v, 2, c), regs = fld(v, 3, c),
                smem = fld(v, 4, c), dt = fld(v, 5, c);
  if (seq < 1 || dim < 1) { u.status = SP_PAIR_E_DIM; return u; }
  if (warps < 1 || regs < 1 || smem < 0) { u.status = SP_PAIR_E_RES; return u; }
  const int bpe = bytes_per_elem((int)dt);
  if (bpe == 0) { u.status = SP_PAIR_E_DTYPE; return u; }
  u.T = seq;
  u.tdt = -1;
  unsigned __int128 task[4] = {0, (unsigned __int128)(silu ? 4 : 3) * dim,
                               silu ? (unsigned __int128)2 * dim : (unsigned __int128)1,
                               (unsigned __int128)2 * dim * bpe};
  finish_totals(u, task);
  u.fp.smem = smem > 0 ? smem : warps * 4;
  u.fp.warps = warps;
  u.fp.regs = regs;
  return u;
}

__device__ __forceinline__ UniformCfg config_of(int fam, const ConfigView &v, int64_t c,
                                                const MoeHist *hist = nullptr) {
  switch (fam) {
    case SP_GEMM: return gemm_cfg(v, c);
    case SP_FUSED_MOE: return moe_cfg(v, c, hist);
    case SP_RMSNORM: return rowwise_cfg(v, c, false);
    case SP_SCALED_MM: return scaled_mm_cfg(v, c);
    default: return rowwise_cfg(v, c, true);
  }
}

// One pair: spec-dependent checks in the oracle's order, then the closed-form
// schedule (busiest SM = ceil(T/N) tasks) and the record.
__device__ __forceinline__ void uniform_pair(const FeatOut &out, int64_t p, const UniformCfg &u,
                                             const DevSpec &s, int pipes) {
  if (u.status != 0) { emit_error(out, p, u.status); return; }
  if (u.tdt >= 0 && !s.tensor_ok[u.tdt]) { emit_error(out, p, SP_PAIR_E_DTYPE); return; }
  if (u.range_bad) { emit_error(out, p, SP_PAIR_E_RANGE); return; }
  PairDemand d;
  d.T = u.T;
  const int64_t per_sm = (int64_t)(((uint32_t)u.T + (uint32_t)s.num_sms - 1u) / (uint32_t)s.num_sms);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    d.tot[q] = u.tot[q];
    d.mx[q] = per_sm * u.task[q];
  }
  emit_pair(out, p, d, u.fp, s, pipes, u.tdt < 0 ? 0 : u.tdt);
}

// Split-K pair: cyclic dealing of two contiguous task classes.  SM j holds
// qa + [j < ra] full-slice tasks (ra = Ta mod N) and qb + [(j - Ta) mod N < rb]
// last-slice tasks; since Ta = ra (mod N) the second set is the cyclic
// interval [ra, ra + rb), which meets [0, ra) iff ra + rb > N.  Full-slice
// demands dominate last-slice ones (k_last <= kps), so the busiest SM is
//   qa*a + qb*b + (ra + rb > N ? a + b : ra > 0 ? a : rb > 0 ? b : 0)
// for every quantity at once (all are proportional to the slice's k extent).
__device__ __forceinline__ void splitk_pair(const FeatOut &out, int64_t p, const SplitKCfg &r,
                                            const DevSpec &s) {
  const UniformCfg &u = r.u;
  if (u.status != 0) { emit_error(out, p, u.status); return; }
  if (!s.tensor_ok[u.tdt]) { emit_error(out, p, SP_PAIR_E_DTYPE); return; }
  if (u.range_bad) { emit_error(out, p, SP_PAIR_E_RANGE); return; }
  const uint32_t N = (uint32_t)s.num_sms, Ta = (uint32_t)r.Ta, Tb = (uint32_t)(u.T - r.Ta);
  const uint32_t qa = Ta / N, ra = Ta - qa * N, qb = Tb / N, rb = Tb - qb * N;
  const int cls = ra + rb > N ? 3 : ra > 0 ? 1 : rb > 0 ? 2 : 0;  // bit 0: a, bit 1: b
  PairDemand d;
  d.T = u.T;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    d.tot[q] = u.tot[q];
    d.mx[q] = (int64_t)(qa + (cls & 1)) * u.task[q] + (int64_t)(qb + (cls >> 1)) * r.taskb[q];
  }
  emit_pair(out, p, d, u.fp, s, 1, u.tdt);
}

__global__ void __launch_bounds__(kThreads) featurize_splitk_cross(ConfigView cfg,
                                                                   const DevSpec *__restrict__ specs, int g0,
                                                                   int g1, FeatOut out) {
  __shared__ DevSpec s_spec[kSpecTile];
  const int gt0 = g0 + blockIdx.y * kSpecTile;
  const int gt1 = min(g1, gt0 + kSpecTile);
  {
    const int n_words = (gt1 - gt0) * (int)(sizeof(DevSpec) / 16);
    const int4 *src = reinterpret_cast<const int4 *>(specs + gt0);
    int4 *dst = reinterpret_cast<int4 *>(s_spec);
    for (int i = threadIdx.x; i < n_words; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (c >= cfg.n_configs) return;
  const SplitKCfg r = splitk_cfg(cfg, c);
  const int64_t C = cfg.n_configs;
  for (int g = gt0; g < gt1; ++g) splitk_pair(out, (int64_t)(g - g0) * C + c, r, s_spec[g - gt0]);
}

__global__ void __launch_bounds__(kThreads) featurize_splitk_list(ConfigView cfg, const DevSpec *__restrict__ specs,
                                                                  int n_specs, int64_t n_pairs,
                                                                  const int64_t *__restrict__ cfg_idx,
                                                                  const int32_t *__restrict__ spec_idx,
                                                                  FeatOut out) {
  const int64_t p = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (p >= n_pairs) return;
  const int64_t c = __ldg(cfg_idx + p);
  const int32_t g = __ldg(spec_idx + p);
  if (c < 0 || c >= cfg.n_configs || g < 0 || g >= n_specs) { emit_error(out, p, SP_PAIR_E_INDEX); return; }
  splitk_pair(out, p, splitk_cfg(cfg, c), specs[g]);
}

__global__ void __launch_bounds__(kThreads) featurize_uniform_cross(int fam, ConfigView cfg,
                                                                    const DevSpec *__restrict__ specs,
                                                                    int g0, int g1, FeatOut out) {
  __shared__ DevSpec s_spec[kSpecTile];
  const int gt0 = g0 + blockIdx.y * kSpecTile;
  const int gt1 = min(g1, gt0 + kSpecTile);
  {
    const int n_words = (gt1 - gt0) * (int)(sizeof(DevSpec) / 16);
    const int4 *src = reinterpret_cast<const int4 *>(specs + gt0);
    int4 *dst = reinterpret_cast<int4 *>(s_spec);
    for (int i = threadIdx.x; i < n_words; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  MoeHist hist;
  if (fam == SP_FUSED_MOE) hist = moe_hist_warp(cfg, c, c < cfg.n_configs);
  if (c >= cfg.n_configs) return;
  const UniformCfg u = config_of(fam, cfg, c, fam == SP_FUSED_MOE ? &hist : nullptr);
  const int pipes = family_pipes(fam);
  const int64_t C = cfg.n_configs;
  for (int g = gt0; g < gt1; ++g) uniform_pair(out, (int64_t)(g - g0) * C + c, u, s_spec[g - gt0], pipes);
}

__global__ void __launch_bounds__(kThreads) featurize_uniform_list(int fam, ConfigView cfg,
                                                                   const DevSpec *__restrict__ specs,
                                                                   int n_specs, int64_t n_pairs,
                                                                   const int64_t *__restrict__ cfg_idx,
                                                                   const int32_t *__restrict__ spec_idx,
                                                                   FeatOut out) {
  const int64_t p = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (p >= n_pairs) return;
  const int64_t c = __ldg(cfg_idx + p);
  const int32_t g = __ldg(spec_idx + p);
  if (c < 0 || c >= cfg.n_configs || g < 0 || g >= n_specs) { emit_error(out, p, SP_PAIR_E_INDEX); return; }
  const UniformCfg u = config_of(fam, cfg, c);
  uniform_pair(out, p, u, specs[g], family_pipes(fam));
}

// ------------------------------------------------------------------ config pre-pass (fused path)

// Spec-independent part of a uniform-family config for the fused
// featurize -> predict kernel: u64 SoA [kPreFields][ldc] (layout in
// sp_internal.h).  Thread per config; fused-MoE histograms by warp as above.
__global__ void __launch_bounds__(kThreads) uniform_prepass(int fam, ConfigView cfg, uint64_t *__restrict__ pre,
                                                            int64_t ldc) {
  const int64_t c = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  MoeHist hist;
  if (fam == SP_FUSED_MOE) hist = moe_hist_warp(cfg, c, c < cfg.n_configs);
  if (c >= cfg.n_configs) return;
  const UniformCfg u = config_of(fam, cfg, c, fam == SP_FUSED_MOE ? &hist : nullptr);
  uint64_t *o = pre + c;
  o[0] = (uint64_t)(uint32_t)u.status | ((uint64_t)u.range_bad << 8) | ((uint64_t)(u.tdt + 1) << 16) |
         ((uint64_t)(uint32_t)u.T << 32);
#pragma unroll
  for (int q = 0; q < 4; ++q) o[(1 + q) * ldc] = (uint64_t)u.task[q];
  // smem clamped to 32 bits: anything above any SM's capacity gives the same zero quota
  const uint64_t sm32 = u.fp.smem > 0xffffffffLL ? 0xffffffffull : (uint64_t)u.fp.smem;
  o[5 * ldc] = sm32 | ((uint64_t)(uint32_t)u.fp.warps << 32);
  o[6 * ldc] = (uint64_t)(uint32_t)u.fp.regs;
}

// ------------------------------------------------------------------ clamped edge tiles

// SPEC's clamped reading of edge tiles (the alternative to R2's
// padded tiles): an edge tile computes and loads only its
// in-range rows/columns, over the exact K (GEMM) or H (fused MoE).  Tasks are no
// longer uniform, so the busiest SM is not ceil(T/N) tasks.  GEMM has a closed
// form per SM (clamped_gemm_pair below).  For fused MoE the task list is a
// sequence of runs of equal tasks (per output-tile row: nt-1 full-width tiles,
// then the edge tile), and cyclic dealing sends a run [start, start+len) of
// weight w to SM j  q*w + w*[(j - start) mod N < r]  times (q = len/N, r = len%N).
// A warp per pair adds the q*w parts to a constant and the cyclic intervals to a
// per-warp difference array in shared memory (64-bit atomics: order-free
// integer sums), then a prefix scan gives every S_j and the max.  O(rows + N).
struct ClampRuns {
  unsigned __int128 tot[2] = {0, 0};  // this lane's totals: Tensor ops, bytes
  int64_t cst[2] = {0, 0};            // this lane's q*w parts
};

__device__ __forceinline__ void add_run(ClampRuns &cr, int64_t *D, int N, int64_t start, int64_t len,
                                        int64_t w_ops, int64_t w_bytes) {
  const int64_t w[2] = {w_ops, w_bytes};
  const int64_t q = len / N, r = len - q * N;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    cr.tot[k] += (unsigned __int128)len * (unsigned __int128)w[k];
    cr.cst[k] += q * w[k];
    if (r == 0) continue;
    unsigned long long *d = reinterpret_cast<unsigned long long *>(D + k * (N + 1));
    const int a = (int)(start % N), b = a + (int)r;
    atomicAdd(d + a, (unsigned long long)w[k]);
    if (b <= N) {
      atomicAdd(d + b, (unsigned long long)(-w[k]));
    } else {
      atomicAdd(d, (unsigned long long)w[k]);
      atomicAdd(d + (b - N), (unsigned long long)(-w[k]));
    }
  }
}

__device__ __forceinline__ int64_t warp_sum64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// GEMM clamped, closed form (no task list): with dh = tm - h_last, dw = tn - w_last,
//   ops(t)   = 2K (tm tn - tm dw [last column] - dh tn [last row] + dh dw [corner])
//   bytes(t) = K bpe (tm + tn - dw [last column] - dh [last row])
// so SM s holds  cnt_s, C_s, R_s, K_s  tasks of the four indicator classes:
//   cnt_s = all tasks (cyclic: q + [s < r]); R_s = the last row, a contiguous run;
//   K_s = the corner (t = T-1); C_s = the last column, the progression
//   (nt-1) + i nt, i < mt: with d = gcd(nt, N), P = N/d, residue s is hit iff
//   d | s - (nt-1), by i = i0 + kP, i0 = ((s - (nt-1))/d) inv(nt/d mod P) mod P,
//   that is mt/P + [i0 < mt mod P] times.
// Lanes take SMs; O(N/32) per pair.  Exact (128-bit products).
__device__ __forceinline__ uint32_t inv_mod(uint32_t a, uint32_t m) {  // gcd(a, m) = 1, m >= 1
  if (m == 1) return 0;
  int32_t t = 0, nt = 1;
  uint32_t r = m, nr = a % m;
  while (nr != 0) {
    const uint32_t q = r / nr, r2 = r - q * nr;
    const int32_t t2 = t - (int32_t)q * nt;
    t = nt; nt = t2; r = nr; nr = r2;
  }
  return t < 0 ? (uint32_t)(t + (int32_t)m) : (uint32_t)t;
}

__device__ void clamped_gemm_pair(const ConfigView &v, int64_t c, const UniformCfg &u, const DevSpec &s,
                                  const FeatOut &out, int64_t p) {
  const int lane = threadIdx.x & 31;
  const int64_t M = fld(v, 0, c), Nn = fld(v, 1, c), K = fld(v, 2, c), tm = fld(v, 3, c), tn = fld(v, 4, c);
  const int64_t bpe = bytes_per_elem((int)fld(v, 10, c));
  const int64_t mt = cdiv31(M, tm), nt = cdiv31(Nn, tn), T = mt * nt;
  const int64_t dh = tm - (M - (mt - 1) * tm), dw = tn - (Nn - (nt - 1) * tn);
  typedef __int128 i128;
  const i128 tot_ops = (i128)2 * K * M * Nn, tot_bytes = (i128)K * bpe * ((i128)nt * M + (i128)mt * Nn);
  if (tot_ops > (i128)kI64Max || tot_bytes > (i128)kI64Max) {
    if (lane == 0) emit_error(out, p, SP_PAIR_E_RANGE);
    return;
  }
  // T < 2^31 (validated) and N <= 4096: 32-bit counts
  const uint32_t N32 = (uint32_t)s.num_sms, T32 = (uint32_t)T, nt32 = (uint32_t)nt, mt32 = (uint32_t)mt;
  const int64_t q = T32 / N32, r = T32 % N32;
  const int64_t startR = (T32 - nt32) % N32, qR = nt32 / N32, rR = nt32 % N32;
  uint32_t d32 = nt32, e32 = N32;  // gcd(nt, N)
  while (e32 != 0) { const uint32_t t2 = d32 % e32; d32 = e32; e32 = t2; }
  const uint32_t P32 = N32 / d32, invn = inv_mod((nt32 / d32) % P32, P32);
  const int64_t a0 = (nt32 - 1u) % N32, qC = mt32 / P32, rC = mt32 % P32;
  const int64_t sK = (T32 - 1u) % N32;
  i128 best_o = -1, best_b = -1;
  // 32-bit residue arithmetic: N <= 4096 (the clamped path's limit), so P^2 < 2^24
  const uint32_t inv32 = invn;
  const uint32_t sR = (uint32_t)startR, sA = (uint32_t)a0, rR32 = (uint32_t)rR, rC32 = (uint32_t)rC;
  for (uint32_t sm = lane; sm < N32; sm += 32) {
    const int64_t cnt = q + (sm < (uint32_t)r ? 1 : 0);
    const int64_t Rs = qR + ((sm >= sR ? sm - sR : sm + N32 - sR) < rR32 ? 1 : 0);
    const uint32_t diff = sm >= sA ? sm - sA : sm + N32 - sA;
    const uint32_t dq = diff / d32;
    int64_t Cs = 0;
    if (dq * d32 == diff) Cs = qC + ((dq * inv32) % P32 < rC32 ? 1 : 0);
    const int64_t Ks = sm == (uint32_t)sK ? 1 : 0;
    const i128 o = (i128)2 * K * ((i128)tm * tn * cnt - (i128)tm * dw * Cs - (i128)dh * tn * Rs + (i128)dh * dw * Ks);
    const i128 b = (i128)K * bpe * ((i128)(tm + tn) * cnt - (i128)dw * Cs - (i128)dh * Rs);
    best_o = o > best_o ? o : best_o;
    best_b = b > best_b ? b : best_b;
  }
  int64_t mo = (int64_t)best_o, mb = (int64_t)best_b;  // < 2^63: bounded by the totals
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mo = max(mo, (int64_t)__shfl_xor_sync(0xffffffffu, mo, o));
    mb = max(mb, (int64_t)__shfl_xor_sync(0xffffffffu, mb, o));
  }
  if (lane != 0) return;
  PairDemand dd;
  dd.T = T;
  dd.tot[0] = (int64_t)tot_ops; dd.tot[1] = 0; dd.tot[2] = 0; dd.tot[3] = (int64_t)tot_bytes;
  dd.mx[0] = mo; dd.mx[1] = 0; dd.mx[2] = 0; dd.mx[3] = mb;
  emit_pair(out, p, dd, u.fp, s, 1, u.tdt);
}

// One pair, whole warp.  D: this warp's 2*(N_max+1) int64 scratch.
__device__ void clamped_pair(int fam, const ConfigView &v, int64_t c, const DevSpec &s, const FeatOut &out,
                             int64_t p, int64_t *D) {
  const int lane = threadIdx.x & 31;
  const UniformCfg u = config_of(fam, v, c);  // status, T, footprint, dtype (padded totals unused)
  if (u.status != 0 || (u.tdt >= 0 && !s.tensor_ok[u.tdt])) {
    if (lane == 0) emit_error(out, p, u.status != 0 ? u.status : SP_PAIR_E_DTYPE);
    return;
  }
  if (fam == SP_GEMM) {
    clamped_gemm_pair(v, c, u, s, out, p);
    return;
  }
  const int N = s.num_sms;
  for (int i = lane; i < 2 * (N + 1); i += 32) D[i] = 0;
  __syncwarp();
  ClampRuns cr;
  {  // fused MoE: expert-major, m-block, n-block
    const int64_t M = fld(v, 0, c), E = fld(v, 1, c), topk = fld(v, 2, c), H = fld(v, 3, c), Nn = fld(v, 4, c),
                  bm = fld(v, 5, c), bn = fld(v, 6, c);
    const int64_t bpe = bytes_per_elem((int)fld(v, 13, c));
    const int64_t nt = cdiv64(Nn, bn), wl = Nn - (nt - 1) * bn;
    const int64_t off = v.ragged_off ? __ldg(v.ragged_off + c) : -1;
    const int64_t mtk = M * topk, qq = mtk / E, rr = mtk - qq * E;
    int64_t base = 0;  // m-blocks of the experts before this chunk
    for (int64_t e0 = 0; e0 < E; e0 += 32) {
      const int64_t e = e0 + lane;
      const int64_t te = e < E ? (off >= 0 ? (int64_t)__ldg(v.ragged + off + e) : qq + (e < rr ? 1 : 0)) : 0;
      const int64_t mb = cdiv64(te, bm);
      int64_t incl = mb;  // inclusive warp scan of the m-block counts
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int64_t first = base + incl - mb;
      for (int64_t j = 0; j < mb; ++j) {
        const int64_t ma = min(bm, te - j * bm), t0 = (first + j) * nt;
        if (nt > 1) add_run(cr, D, N, t0, nt - 1, 2 * ma * bn * H, (ma + bn) * H * bpe);
        add_run(cr, D, N, t0 + nt - 1, 1, 2 * ma * wl * H, (ma + wl) * H * bpe);
      }
      base += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  // totals (128-bit) and the exact-range rule (R22)
  int bad = 0;
  int64_t tot[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    unsigned long long lo = (unsigned long long)cr.tot[k], hi = (unsigned long long)(cr.tot[k] >> 64);
    unsigned __int128 t = 0;
    for (int l = 0; l < 32; ++l) {
      const unsigned long long a = __shfl_sync(0xffffffffu, lo, l), b = __shfl_sync(0xffffffffu, hi, l);
      t += ((unsigned __int128)b << 64) | a;
    }
    bad |= t > kI64Max;
    tot[k] = (int64_t)t;
  }
  const int64_t cst[2] = {warp_sum64(cr.cst[0]), warp_sum64(cr.cst[1])};
  __syncwarp();
  // S_j = cst + prefix(D)[j]; lanes own contiguous chunks of the N SMs
  const int chunk = (N + 31) / 32, j0 = min(N, lane * chunk), j1 = min(N, j0 + chunk);
  int64_t mx[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int64_t *d = D + k * (N + 1);
    int64_t part = 0;
    for (int j = j0; j < j1; ++j) part += d[j];
    int64_t incl = part;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int64_t run = cst[k] + incl - part, best = INT64_MIN;
    for (int j = j0; j < j1; ++j) {
      run += d[j];
      best = max(best, run);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    mx[k] = best;
  }
  __syncwarp();
  if (lane != 0) return;
  if (bad) { emit_error(out, p, SP_PAIR_E_RANGE); return; }
  PairDemand d;
  d.T = u.T;
  d.tot[0] = tot[0]; d.tot[1] = 0; d.tot[2] = 0; d.tot[3] = tot[1];
  d.mx[0] = mx[0]; d.mx[1] = 0; d.mx[2] = 0; d.mx[3] = mx[1];
  emit_pair(out, p, d, u.fp, s, 1, u.tdt);
}

__global__ void featurize_clamped(int fam, ConfigView cfg, const DevSpec *__restrict__ specs, int g0, int n_specs,
                                  int64_t n_pairs, const int64_t *__restrict__ cfg_idx,
                                  const int32_t *__restrict__ spec_idx, int max_sms, FeatOut out) {
  extern __shared__ int64_t s_diff[];
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int64_t *D = s_diff + (size_t)warp * 2 * (max_sms + 1);
  for (int64_t p = (int64_t)blockIdx.x * nw + warp; p < n_pairs; p += (int64_t)gridDim.x * nw) {
    int64_t c;
    int g;
    if (cfg_idx) {
      c = __ldg(cfg_idx + p);
      g = __ldg(spec_idx + p);
      if (c < 0 || c >= cfg.n_configs || g < 0 || g >= n_specs) {
        if ((threadIdx.x & 31) == 0) emit_error(out, p, SP_PAIR_E_INDEX);
        continue;
      }
    } else {
      g = g0 + (int)(p / cfg.n_configs);
      c = p - (int64_t)(g - g0) * cfg.n_configs;
    }
    clamped_pair(fam, cfg, c, specs[g], out, p, D);
    __syncwarp();
  }
}

}  // namespace

int launch_featurize_uniform(int family, const ConfigView &cfg, const DevSpec *specs, int spec_begin,
                             int spec_end, int64_t n_pairs, const int64_t *cfg_idx,
                             const int32_t *spec_idx, const FeatOut &out, void *stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (cfg_idx == nullptr) {  // CROSS
    if (cfg.n_configs == 0 || spec_end <= spec_begin) return 0;
    dim3 grid((unsigned)((cfg.n_configs + kThreads - 1) / kThreads),
              (unsigned)((spec_end - spec_begin + kSpecTile - 1) / kSpecTile));
    if (family == SP_GEMM_SPLITK)
      featurize_splitk_cross<<<grid, kThreads, 0, st>>>(cfg, specs, spec_begin, spec_end, out);
    else
      featurize_uniform_cross<<<grid, kThreads, 0, st>>>(family, cfg, specs, spec_begin, spec_end, out);
  } else {
    if (n_pairs == 0) return 0;
    unsigned blocks = (unsigned)((n_pairs + kThreads - 1) / kThreads);
    if (family == SP_GEMM_SPLITK)
      featurize_splitk_list<<<blocks, kThreads, 0, st>>>(cfg, specs, spec_end, n_pairs, cfg_idx, spec_idx, out);
    else
      featurize_uniform_list<<<blocks, kThreads, 0, st>>>(family, cfg, specs, spec_end, n_pairs, cfg_idx,
                                                           spec_idx, out);
  }
  return (int)cudaGetLastError();
}

int launch_uniform_prepass(int family, const ConfigView &cfg, uint64_t *pre, int64_t ldc, void *stream) {
  if (cfg.n_configs == 0) return 0;
  uniform_prepass<<<(unsigned)((cfg.n_configs + kThreads - 1) / kThreads), kThreads, 0,
                    reinterpret_cast<cudaStream_t>(stream)>>>(family, cfg, pre, ldc);
  return (int)cudaGetLastError();
}

int launch_featurize_clamped(int family, const ConfigView &cfg, const DevSpec *specs, int spec_begin, int n_specs,
                             int64_t n_pairs, const int64_t *cfg_idx, const int32_t *spec_idx, int max_sms,
                             const FeatOut &out, int num_device_sms, void *stream) {
  if (n_pairs == 0) return 0;
  const size_t per_warp = (size_t)2 * (max_sms + 1) * sizeof(int64_t);
  const int warps = (int)std::max<size_t>(1, std::min<size_t>(8, (96 * 1024) / per_warp));
  const size_t smem = per_warp * warps;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(featurize_clamped, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  const int64_t blocks = std::min<int64_t>((n_pairs + warps - 1) / warps, (int64_t)num_device_sms * 16);
  featurize_clamped<<<(unsigned)blocks, 32 * warps, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
      family, cfg, specs, spec_begin, n_specs, n_pairs, cfg_idx, spec_idx, max_sms, out);
  return (int)cudaGetLastError();
}

}  // namespace sp
