// Feature stage for FlashInfer FA2 attention, prefill and decode (Table V
// P:413; non-uniform causal tasks P:262; readings R4, R10-R13).
//
// Tasks: kv-head h outermost, then request b, q-block i, kv-chunk c (R4).  A
// task's demands are affine in its kv units u = kv_eff/BKV:
//   Tensor = 4*BQ*hd*BKV*u, XU = BQ*(BKV+1)*u, bytes = bpe*hd*(BQ + 2*BKV*u),
// so per SM only two numbers matter: its task count n_j (closed form under
// cyclic dealing, R5) and its unit sum S_j.  All nkv kv-heads repeat the same
// task sequence of length L, so with A[r] = sum of u over head-0 tasks k with
// k mod N = r, the per-SM sums are the rotations S_j = sum_h A[(j - h*L) mod N]
// (exact: task t = h*L + k goes to SM t mod N).
//
// Layout: one warp per config.  Lanes take 32 consecutive head-0 tasks per
// step; with N >= 32 the 32 residues are distinct, so each lane updates its
// own shared-memory accumulator with one shared reduction (red.shared.add,
// one issue slot instead of load + add + store).  The task
// sequence does not depend on the spec, so in SP_PAIRS_CROSS mode a warp
// accumulates once per *distinct SM count* of the spec range (the 11 GPUs of
// Table VI have 7) and then emits every spec of its group; the distinct set
// is a template parameter so residues and offsets live in registers.  Configs
// with T <= min N (every SM holds at most one task: most decode batches) skip
// the accumulators: max_j S_j is the largest task's u.
// The kernel is bound by integer issue, not by HBM.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"

namespace sp {
namespace {

#ifndef SP_ATTN_MINB
#define SP_ATTN_MINB 4  // 32 warps/SM (64 regs): measured best of 3..6 on cfg2
#endif

constexpr int kWarps = 8;           // warps per block
constexpr int kSimWarps = 4;        // warps per block of the scheduler-simulation kernel
constexpr int kMaxDistinct = 8;     // distinct SM counts per group (api.cu plans accordingly)
constexpr int64_t kI32Max = 2147483647LL;
constexpr int64_t kU32Max = 4294967295LL;
constexpr unsigned __int128 kI64Max = 9223372036854775807ULL;
typedef unsigned __int128 u128;

// Field indices (include/synperf.h, SP_ATTENTION)
enum { BS, NH, NKV, HD, BQ, BKV, CHUNK, CAUSAL, WARPS, REGS, SMEM, DTYPE };

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
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
__device__ __forceinline__ uint32_t warp_max_u32(uint32_t v) { return __reduce_max_sync(0xffffffffu, v); }

// Cheap FastDiv setup: powers of two need no division.
__device__ __forceinline__ FastDiv make_fd(uint32_t d) {
  FastDiv f;
  f.d = d;
  f.s = d <= 1 ? 0 : 32 - __clz(d - 1);
  f.m = (d & (d - 1)) ? fastdiv_magic(d, f.s) : 1u;
  return f;
}

// Per-config scalars shared by all lanes.
struct AttnCfg {
  int status;
  int32_t bs, nh, nkv, hd, bq, bkv, chunk, causal, dt, g;  // input fields are int32
  const int32_t *req;
  Footprint fp;
};

// Divisors of a config's hot arithmetic (FastDiv: multiply-high + shift).
// make_fd costs a 64-bit division; the cross path gets them from attn_prepass
// (thread per config) instead of recomputing them warp-uniformly.
struct AttnDivs {
  FastDiv g, bkv, bq, chunk;
};
__device__ __forceinline__ AttnDivs make_divs(const AttnCfg &a) {
  AttnDivs d;
  d.g = make_fd((uint32_t)a.g);
  d.bkv = make_fd((uint32_t)a.bkv);
  d.bq = make_fd((uint32_t)a.bq);
  d.chunk = a.chunk > 0 ? make_fd((uint32_t)a.chunk) : FastDiv{1u, 1u, 0u};
  return d;
}

// PLANNER: accept kv_chunk = -1 (non-causal) for the split-KV planner (R24).
// The cross schedule kernel uses PLANNER = false and reports such configs as
// SP_PAIR_E_TILE; attn_planner_cross then rewrites their records (keeping the
// hot kernel's code -- and its register allocation -- free of the planner).
template <bool PLANNER = true>
__device__ __forceinline__ AttnCfg load_cfg(const ConfigView &v, int64_t c, int lane) {
  AttnCfg a{};
  const int32_t f = lane < 12 ? __ldg(v.fields + (int64_t)lane * v.ld + c) : 0;
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
  // kv_chunk -1: the split-KV planner chooses it per spec (R24; non-causal only)
  if (a.bq < 1 || a.bkv < 1 || a.chunk < (PLANNER ? -1 : 0) || (a.chunk == -1 && a.causal)) {
    a.status = SP_PAIR_E_TILE;
    return a;
  }
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
  a.fp.smem = smem > 0 ? smem : ((int64_t)a.bq + 2 * (int64_t)a.bkv) * a.hd * 2;
  a.fp.warps = warps;
  a.fp.regs = regs;
  return a;
}

// kv extent of q-block i of a request (R10-R11): q_last = floor((min((i+1)BQ, rows)-1)/g),
// kv_need = min(kvlen, kvlen - qlen + q_last + 1) if causal, else kvlen.
__device__ __forceinline__ uint32_t kv_need(uint64_t i, uint64_t bq, uint64_t rows, uint32_t qlen,
                                            uint32_t kvlen, bool causal, const FastDiv &fg) {
  if (!causal) return kvlen;
  const uint64_t e = min((i + 1) * bq, rows) - 1;
  const uint32_t q_last = fg.div((uint32_t)e);
  return min(kvlen, kvlen - qlen + q_last + 1);
}

__device__ __forceinline__ uint64_t sat_add(uint64_t a, uint64_t b) {
  const uint64_t lim = 1ull << 40;
  const uint64_t s = a + b;
  return s > lim ? lim : s;
}

// Split-KV planner (R24; FlashInfer's decode planner, F depends on S):
// with max_grid = N_SM * occ work items, no split if nkv * sum_b nqb_b already
// reaches it; otherwise the smallest chunk 16c (c >= 1) with
// nkv * sum_b nqb_b * ceil(kv_b / 16c) <= max_grid, and 0 (unsplit) if that
// chunk covers the longest request.  Warp-cooperative binary search (the item
// count is non-increasing in c).  Non-causal configs only.
constexpr int32_t kPlannerPage = 16;

__device__ int32_t plan_chunk(const AttnCfg &a, const DevSpec &sp, int lane) {
  const uint64_t max_grid = (uint64_t)sp.num_sms * (uint64_t)occupancy(a.fp, sp);
  uint64_t w0 = 0;
  uint32_t maxkv = 0;
  for (int64_t b = lane; b < a.bs; b += 32) {
    const uint64_t q = __ldg(a.req + 2 * b), kv = __ldg(a.req + 2 * b + 1);
    w0 += (q * a.g + a.bq - 1) / a.bq;
    maxkv = max(maxkv, (uint32_t)kv);
  }
  w0 = warp_sum_u64(w0) * (uint64_t)a.nkv;
  maxkv = warp_max_u32(maxkv);
  if (w0 >= max_grid) return 0;
  auto items = [&](uint32_t chunk) -> uint64_t {
    uint64_t n = 0;
    for (int64_t b = lane; b < a.bs; b += 32) {
      const uint64_t q = __ldg(a.req + 2 * b), kv = __ldg(a.req + 2 * b + 1);
      n += (q * a.g + a.bq - 1) / a.bq * ((kv + chunk - 1) / chunk);
    }
    return warp_sum_u64(n) * (uint64_t)a.nkv;
  };
  uint32_t lo = 1, hi = (maxkv + kPlannerPage - 1) / kPlannerPage;  // items(16*hi) = w0 < max_grid
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (items(mid * kPlannerPage) <= max_grid) hi = mid; else lo = mid + 1;
  }
  const uint32_t chunk = lo * kPlannerPage;
  return chunk >= maxkv ? 0 : (int32_t)chunk;
}

// Pre-pass: per-head task count L (lanes over requests; causal split-KV walks
// the request's q-blocks).  Saturates at 2^40 (anything above 2^31 is RANGE).
// 32-bit operands throughout: q*g < 2^31, BQ, BKV, chunk, kv < 2^31 (validated),
// so every "x + d - 1" below is < 2^32 (FastDiv::div takes any 32-bit n).
__device__ int64_t count_tasks(const AttnCfg &a, int lane, const AttnDivs &dv) {
  uint64_t part = 0;
  for (int64_t b = lane; b < a.bs; b += 32) {
    const uint32_t q = __ldg(a.req + 2 * b), kv = __ldg(a.req + 2 * b + 1);
    const uint32_t rows = q * (uint32_t)a.g, nqb = dv.bq.div(rows + (uint32_t)a.bq - 1u);
    if (a.chunk == 0) {
      part = sat_add(part, nqb);
    } else if (!a.causal) {
      part = sat_add(part, (uint64_t)nqb * dv.chunk.div(kv + (uint32_t)a.chunk - 1u));
    } else {
      for (uint32_t i = 0; i < nqb && part < (1ull << 40); ++i)
        part = sat_add(part, dv.chunk.div(kv_need(i, a.bq, rows, q, kv, true, dv.g) + (uint32_t)a.chunk - 1u));
    }
  }
  return (int64_t)min(warp_sum_u64(part), (uint64_t)(1ull << 40));
}

// Sparse path (T <= min N): every SM holds at most one task, so only the unit
// sum U and the largest unit umax are needed.  Lanes over requests.
__device__ void sparse_units(const AttnCfg &a, int lane, const AttnDivs &dv, uint64_t &U, uint32_t &umax) {
  uint64_t us = 0;
  uint32_t um = 0;
  for (int64_t b = lane; b < a.bs; b += 32) {
    const uint32_t q = __ldg(a.req + 2 * b), kv = __ldg(a.req + 2 * b + 1);
    const uint32_t rows = q * (uint32_t)a.g, nqb = dv.bq.div(rows + (uint32_t)a.bq - 1u);
    for (uint32_t i = 0; i < nqb; ++i) {
      const uint32_t need = kv_need(i, a.bq, rows, q, kv, a.causal, dv.g);
      if (a.chunk == 0) {
        const uint32_t u = dv.bkv.div(need + (uint32_t)a.bkv - 1u);
        us += u;
        um = max(um, u);
      } else {
        for (uint32_t c0 = 0; c0 < need; c0 += (uint32_t)a.chunk) {
          const uint32_t u = dv.bkv.div(min((uint32_t)a.chunk, need - c0) + (uint32_t)a.bkv - 1u);
          us += u;
          um = max(um, u);
          if (need - c0 <= (uint32_t)a.chunk) break;  // (c0 + chunk may wrap 32 bits)
        }
      }
    }
  }
  U = warp_sum_u64(us);
  umax = warp_max_u32(um);
}

struct DistinctMax {
  int64_t maxS, maxB;  // max_j S_j and max_j (BQ*n_j + 2*BKV*S_j)
};

// Request scratch (accumulate): per-request parameters of a chunk of 32
// requests, 7 arrays of 32 words.

__device__ __forceinline__ uint32_t lanemask_le() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
  return m;
}

// Causal + split-KV (rare): each q-block has its own chunk count.  Lanes take
// 32 q-blocks of one request, scan their chunk counts, then walk their own
// chunks (positions are not lane-consecutive: atomic adds).
template <int ND>
__device__ uint64_t accumulate_causal_split(const AttnCfg &a, uint32_t *acc, const int32_t (&off)[ND],
                                            const FastDiv *fdN, int lane, const FastDiv &fg, const FastDiv &fbkv) {
  uint32_t base = 0;
  uint64_t usum = 0;
  for (int64_t b = 0; b < a.bs; ++b) {
    const uint32_t qlen = __ldg(a.req + 2 * b), kvlen = __ldg(a.req + 2 * b + 1);
    const uint32_t rows = qlen * (uint32_t)a.g;
    const uint32_t nqb = (rows + (uint32_t)a.bq - 1u) / (uint32_t)a.bq;
    for (uint32_t i0 = 0; i0 < nqb; i0 += 32) {
      const uint32_t i = i0 + lane;
      uint32_t need = 0, n_ch = 0;
      if (i < nqb) {
        need = kv_need(i, a.bq, rows, qlen, kvlen, true, fg);
        n_ch = (uint32_t)((need + (uint64_t)a.chunk - 1) / a.chunk);
      }
      uint32_t incl = n_ch;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t start = base + incl - n_ch;
      for (uint32_t ch = 0; ch < n_ch; ++ch) {
        const uint32_t len = min((uint32_t)a.chunk, need - ch * (uint32_t)a.chunk);
        const uint32_t u = fbkv.div(len + (uint32_t)a.bkv - 1);
#pragma unroll
        for (int d = 0; d < ND; ++d) atomicAdd(acc + off[d] + fdN[d].mod(start + ch), u);
        usum += u;
      }
      base += total;
      __syncwarp();
    }
  }
  return usum;
}

// General path: per-SM accumulators in the warp's shared-memory region, one
// region per distinct SM count (N[d] words at off[d]).  The head-0 task stream
// is walked flat across request boundaries: requests are taken 32 at a time
// (lane = request: its task count, start and per-request constants go to the
// warp's scratch), then each step gives lane l the task k0 + l and finds its
// request from a boundary bitmask (one warp OR-reduction per step).
template <int ND, bool SMALL>
__device__ uint64_t accumulate(const AttnCfg &a, uint32_t *acc, int words, uint32_t *scr, const int32_t (&N)[ND],
                               const int32_t (&off)[ND], const FastDiv *fdN, int lane, const AttnDivs &dv) {
  for (int w = lane * 4; w < words; w += 128) *reinterpret_cast<uint4 *>(acc + w) = make_uint4(0, 0, 0, 0);
  __syncwarp();
  const FastDiv &fg = dv.g, &fbkv = dv.bkv;
  const bool split = a.chunk > 0;
  if (split && a.causal) {
    const uint64_t us = accumulate_causal_split<ND>(a, acc, off, fdN, lane, fg, fbkv);
    __syncwarp();
    return warp_sum_u64(us);
  }
  const FastDiv &fbq = dv.bq;
  // causal without split-KV and g | BQ: kv_need is affine in the q-block index, and
  // when BKV divides 32 BQ/g the units of q-blocks 32 apart differ by a constant
  const uint32_t a_per = (uint32_t)(a.bq / a.g);
  const bool lin = !split && a.causal && a.bq % a.g == 0 && (int64_t)a.bq * 33 < (1ll << 30) &&
                   (32u * a_per) % (uint32_t)a.bkv == 0;
  const uint32_t dlt = lin ? (32u * a_per) / (uint32_t)a.bkv : 0u;
  const FastDiv &fchunk = dv.chunk;
  const uint32_t acc_s = (uint32_t)__cvta_generic_to_shared(acc);  // shared-window byte address
  const uint32_t lm_le = lanemask_le();
  uint32_t *s_start = scr, *s_a1 = scr + 32, *s_a2 = scr + 64, *s_a3 = scr + 96, *s_uf = scr + 128,
           *s_ul = scr + 160;
  uint32_t base = 0;  // head-0 index of the chunk's first task (< 2^31, checked by the pre-pass)
  uint64_t usum = 0;
  for (int64_t b0 = 0; b0 < a.bs; b0 += 32) {
    // ---- lane = request b0 + lane: task count and per-request constants
    const bool has = b0 + lane < a.bs;
    uint32_t tasks = 0, a1 = 0, a2 = 0, a3 = 0, uf = 0, ul = 0;
    if (has) {
      const uint32_t q = __ldg(a.req + 2 * (b0 + lane)), kv = __ldg(a.req + 2 * (b0 + lane) + 1);
      const uint32_t rows = q * (uint32_t)a.g;  // < 2^31 (validated)
      const uint32_t nqb = fbq.div(rows + (uint32_t)a.bq - 1u);
      if (!split) {
        tasks = nqb;
        if (a.causal) {
          a1 = rows;
          a2 = q;
          a3 = kv;
        } else {
          uf = ul = fbkv.div(kv + (uint32_t)a.bkv - 1u);  // kv_need = kvlen for every q-block
        }
      } else {  // non-causal split-KV: chunks of one q-block share kv_need = kvlen
        const uint32_t n_ch = fchunk.div(kv + (uint32_t)a.chunk - 1u);
        tasks = nqb * n_ch;
        a1 = n_ch;
        if (nqb > 1) {  // chunk index = task mod n_ch (make_fd: an fp64 division)
          const FastDiv f = make_fd(n_ch);
          a2 = f.m;
          a3 = f.s;
        }  // one q-block (decode): the chunk index is the task index; a2 = 0 marks it
        uf = fbkv.div(min((uint32_t)a.chunk, kv) + (uint32_t)a.bkv - 1u);
        ul = fbkv.div(kv - (n_ch - 1u) * (uint32_t)a.chunk + (uint32_t)a.bkv - 1u);
      }
    }
    uint32_t incl = tasks;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const uint32_t start = incl - tasks, total = __shfl_sync(0xffffffffu, incl, 31);
    s_start[lane] = start;
    s_a1[lane] = a1;
    s_a2[lane] = a2;
    s_a3[lane] = a3;
    s_uf[lane] = uf;
    s_ul[lane] = ul;
    __syncwarp();
    const uint32_t nreq = (uint32_t)min((int64_t)32, a.bs - b0);
    uint32_t p[ND];  // byte address of this lane's accumulator for each distinct N
#pragma unroll
    for (int d = 0; d < ND; ++d) p[d] = acc_s + 4u * (uint32_t)(off[d] + (int32_t)fdN[d].mod(base + lane));
    uint32_t hi[ND];  // end of each region (byte address): residue wrap point
#pragma unroll
    for (int d = 0; d < ND; ++d) hi[d] = acc_s + 4u * (uint32_t)(off[d] + N[d]);
    // kv units of task kl of a request described by (a1, a2, a3, uf, ul)
    auto unit = [&](uint32_t kl, uint32_t r1, uint32_t r2, uint32_t r3, uint32_t ruf, uint32_t rul) -> uint32_t {
      if (!split) {
        if (!a.causal) return ruf;
        // q-block kl: q_last = floor((min((kl+1)BQ, rows)-1)/g), kv_need, kv_eff = ceil(need/BKV)*BKV
        const uint32_t e = (uint32_t)min((uint64_t)(kl + 1) * (uint64_t)a.bq, (uint64_t)r1) - 1u;
        const uint32_t need = min(r3, r3 - r2 + fg.div(e) + 1u);
        return fbkv.div(need + (uint32_t)a.bkv - 1u);
      }
      // chunk index kl mod n_ch (kl itself for one q-block): full chunks, then the last one
      const uint32_t ch = r2 ? FastDiv{r1, r2, r3}.mod(kl) : kl;
      return ch == r1 - 1u ? rul : ruf;
    };
    // one step: lane task base + k0 + lane gets u (0 for idle lanes).  The
    // residue pointers wrap lazily: each region has kAttnSlack words past N, so
    // a pointer may run up to 2 steps (index <= N + 31) before wrap() brings it
    // back below N (N >= 64 on this path): the wrap test is paid every other
    // step (ncu: it was 18% of the kernel's instructions when paid every step).
    auto add = [&](uint32_t k, uint32_t u, bool active) {
      usum += u;
      if (SMALL) {
#pragma unroll
        for (int d = 0; d < ND; ++d)
          if (active) atomicAdd(acc + off[d] + fdN[d].mod(base + k), u);
      } else {
#pragma unroll
        for (int d = 0; d < ND; ++d) {
          // one ATOMS.ADD instead of load + add + store: the kernel is issue bound
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(p[d]), "r"(u) : "memory");
          p[d] += 128u;
        }
      }
      // distinct addresses per step and no reads until the loop ends (the
      // __syncwarp after it orders them for the fold); the atomic path may diverge
      if (SMALL) __syncwarp();
    };
    // minus the region length in bytes, from N read back from shared memory: with N
    // itself ptxas rematerialised -4N from a uniform register (one more MOV per
    // region and wrap); this form compiles to compare + predicated add (-2% time)
    uint32_t nspan[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) nspan[d] = 0u - 4u * fdN[d].d;
    auto wrap = [&]() {
      if (!SMALL) {
        // compare + predicated add: 2 instructions per region (the C form compiled to 4)
#pragma unroll
        for (int d = 0; d < ND; ++d)
          asm("{\n.reg .pred w;\nsetp.ge.u32 w, %0, %1;\n@w add.u32 %0, %0, %2;\n}" : "+r"(p[d]) : "r"(hi[d]),
              "r"(nspan[d]));
      }
    };
    uint32_t bcur = 0;  // chunk-local request holding task k0
    uint32_t k0 = 0;
    while (k0 < total) {
      // steps wholly inside request bcur: its constants are warp-uniform
      const uint32_t st = s_start[bcur];
      const uint32_t nxt = bcur + 1 < nreq ? s_start[bcur + 1] : total;
      if (k0 + 32 <= nxt) {
        const uint32_t r1 = s_a1[bcur], r2 = s_a2[bcur], r3 = s_a3[bcur], ruf = s_uf[bcur], rul = s_ul[bcur];
        if (lin && r3 < (1u << 30)) {
          // causal, g | BQ: kv_need(kl) = min(kv, kv - q + (kl+1)*BQ/g) (R10-R11; exact for the
          // last q-block too, where the min takes kv), so u(kl) = min(v(kl), ceil(kv/BKV)) with
          // v(kl) = ceil((kv - q + (kl+1)*BQ/g) / BKV); BKV | 32*BQ/g makes v(kl + 32) = v(kl) + dlt
          // exactly: a lane's next unit is an add and a min.  kv < 2^30 and (kl+1)*BQ/g <= q + BQ/g
          // keep every operand below 2^31.
          const uint32_t ucap = fbkv.div31(r3 - 1u) + 1u;
          uint32_t v = fbkv.div31(r3 - r2 + (k0 + lane - st + 1u) * a_per - 1u) + 1u;  // argument >= kv - q + a_per - 1 >= 0
          for (; k0 + 64 <= nxt; k0 += 64) {
            add(k0 + lane, min(v, ucap), true);
            v += dlt;
            add(k0 + 32 + lane, min(v, ucap), true);
            v += dlt;
            wrap();
          }
          if (k0 + 32 <= nxt) {
            add(k0 + lane, min(v, ucap), true);
            wrap();
            k0 += 32;
          }
        } else {
          for (; k0 + 64 <= nxt; k0 += 64) {
            add(k0 + lane, unit(k0 + lane - st, r1, r2, r3, ruf, rul), true);
            add(k0 + 32 + lane, unit(k0 + 32 + lane - st, r1, r2, r3, ruf, rul), true);
            wrap();
          }
          if (k0 + 32 <= nxt) {
            add(k0 + lane, unit(k0 + lane - st, r1, r2, r3, ruf, rul), true);
            wrap();
            k0 += 32;
          }
        }
        if (k0 >= total) break;
        if (k0 == nxt) { ++bcur; continue; }
      }
      // a step crossing request boundaries: each lane finds its request from
      // the bitmask of request starts inside (k0, k0 + 32)
      const uint32_t k = k0 + lane;
      const bool active = k < total;
      const uint32_t bit = (has && start > k0 && start < k0 + 32) ? (1u << (start - k0)) : 0u;
      const uint32_t M = __reduce_or_sync(0xffffffffu, bit);
      const uint32_t bl = min(bcur + __popc(M & lm_le), nreq - 1);
      const uint32_t u = unit(k - s_start[bl], s_a1[bl], s_a2[bl], s_a3[bl], s_uf[bl], s_ul[bl]);
      add(k, active ? u : 0u, active);
      wrap();
      bcur += __popc(M) + (__any_sync(0xffffffffu, has && start == k0 + 32) ? 1u : 0u);
      k0 += 32;
    }
    base += total;
    __syncwarp();
  }
  if (!SMALL) {  // fold the lazy-wrap overflow A[N, N+32) back onto A[0, 32)
#pragma unroll
    for (int d = 0; d < ND; ++d) acc[off[d] + lane] += acc[off[d] + N[d] + lane];
    __syncwarp();
  }
  return warp_sum_u64(usum);
}

// Fold the nkv rotations of one distinct N and take the per-quantity maxima.
// SM j holds qn + (j < rn) tasks; max_j (BQ n_j + 2 BKV S_j) is taken over the
// two task-count classes separately.  S_j fits 32 bits when nkv * U < 2^32.
//
// Fast form (N <= kFoldDupMax): A is first duplicated into A[N, 2N), so the
// rotated index j - h*L mod N becomes the plain offset j + N - (h*L mod N);
// each lane keeps the sums of its R = ceil(N/32) residues in registers and a
// head costs R shared loads + R adds.  Reads reach index 2N + 31 (the caller
// guarantees that much readable space; lanes past N are discarded).  32-bit
// sums only, and few instantiations: the kernel is instruction-cache bound
// once its code grows (ncu: stalled_no_instructions).
#ifndef SP_FOLD_DUP_MAX
#define SP_FOLD_DUP_MAX 192
#endif
constexpr int kFoldDupMax = SP_FOLD_DUP_MAX;

template <typename SumT, int R>
__device__ __forceinline__ void fold_rows(uint32_t *A, int32_t N, uint32_t Lm, int32_t nkv, uint32_t rn, int lane,
                                          SumT &m_lo, SumT &m_hi) {
  SumT S[R];
  if (nkv == 1) {  // one head: no rotation, S_j = A[j]
#pragma unroll
    for (int i = 0; i < R; ++i) S[i] = (uint32_t)(lane + 32 * i) < (uint32_t)N ? A[lane + 32 * i] : 0u;
  } else {
    // the duplicate overwrites memory other lanes read in the previous region's
    // fold (regions fold last-first): order those reads first (the REDUX maxima in
    // between synchronize the lanes but do not order shared memory)
    __syncwarp();
#pragma unroll
    for (int i = 0; i < R; ++i)
      if (lane + 32 * i < N) A[N + lane + 32 * i] = A[lane + 32 * i];
    __syncwarp();
#pragma unroll
    for (int i = 0; i < R; ++i) S[i] = 0;
    const uint32_t *b0 = A + N + lane;
    uint32_t o = 0;  // h * L mod N
#pragma unroll 1  // code size: the kernel is instruction-cache sensitive
    for (int32_t h = 0; h < nkv; ++h) {
      const uint32_t *b = b0 - o;
#pragma unroll
      for (int i = 0; i < R; ++i) S[i] += b[32 * i];
      asm("{\n.reg .pred w;\nadd.u32 %0, %0, %1;\nsetp.ge.u32 w, %0, %2;\n@w sub.u32 %0, %0, %2;\n}"
          : "+r"(o)
          : "r"(Lm), "r"((uint32_t)N));
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const uint32_t sj = (uint32_t)(lane + 32 * i);
    if (sj < (uint32_t)N) {
      if (sj < rn) m_lo = max(m_lo, S[i]);
      else m_hi = max(m_hi, S[i]);
    }
  }
}

// Per distinct N: the maxima of S_j over the two task-count classes, SMs
// j < rn (qn + 1 tasks) and j >= rn (qn tasks), with T = qn N + rn.  The
// record's max_j S_j and max_j (BQ n_j + 2 BKV S_j) follow from (lo, hi) by
// finish_max, in the (thread-per-config) emit kernel.
struct DistinctLoHi {
  int64_t lo, hi;
};

template <typename SumT>
__device__ DistinctLoHi fold(const AttnCfg &a, uint32_t *A, int32_t N, const FastDiv &fdN, uint32_t L, uint32_t T,
                             int lane) {
  const uint32_t Lm = fdN.mod(L);
  const uint32_t rn = T - fdN.div(T) * (uint32_t)N;
  SumT m_lo = 0, m_hi = 0;
  if (sizeof(SumT) == 4 && N <= kFoldDupMax) {
    switch ((N + 31) >> 5) {
      case 1: fold_rows<SumT, 1>(A, N, Lm, a.nkv, rn, lane, m_lo, m_hi); break;
      case 2: fold_rows<SumT, 2>(A, N, Lm, a.nkv, rn, lane, m_lo, m_hi); break;
      case 3: fold_rows<SumT, 3>(A, N, Lm, a.nkv, rn, lane, m_lo, m_hi); break;
      case 4: fold_rows<SumT, 4>(A, N, Lm, a.nkv, rn, lane, m_lo, m_hi); break;
      case 5: fold_rows<SumT, 5>(A, N, Lm, a.nkv, rn, lane, m_lo, m_hi); break;
      default: fold_rows<SumT, 6>(A, N, Lm, a.nkv, rn, lane, m_lo, m_hi); break;
    }
  } else {
    for (int32_t s = lane; s < N; s += 32) {
      SumT S = 0;
      int32_t o = 0;
      for (int32_t h = 0; h < a.nkv; ++h) {
        int32_t idx = s - o;
        idx += idx < 0 ? N : 0;
        S += A[idx];
        o += (int32_t)Lm;
        o -= o >= N ? N : 0;
      }
      if ((uint32_t)s < rn) m_lo = max(m_lo, S);
      else m_hi = max(m_hi, S);
    }
  }
  if (sizeof(SumT) == 4)  // one REDUX each instead of a 5-step 64-bit shuffle tree
    return DistinctLoHi{(int64_t)__reduce_max_sync(0xffffffffu, (uint32_t)m_lo),
                        (int64_t)__reduce_max_sync(0xffffffffu, (uint32_t)m_hi)};
  return DistinctLoHi{warp_max64((int64_t)m_lo), warp_max64((int64_t)m_hi)};
}

// max_j S_j and max_j (BQ n_j + 2 BKV S_j) of a distinct N from the class maxima
// (lo over the rn SMs with qn + 1 tasks, hi over the others; T = qn N + rn).
// Sparse configs (T <= N, at most one task per SM) pass (umax, umax): for T < N
// the hi term 2 BKV umax (qn = 0) never exceeds the lo term BQ + 2 BKV umax, and
// for T = N (rn = 0, every SM one task) the hi term is the answer.
__device__ __forceinline__ DistinctMax finish_max(int64_t lo, int64_t hi, int64_t T, const FastDiv &fN, int64_t bq,
                                                  int64_t bkv) {
  const int32_t N = (int32_t)fN.d;
  const int64_t qn = fN.div((uint32_t)T), rn = T - qn * N;  // T < 2^31 (range rule)
  int64_t mB = 0;
  if (rn > 0) mB = bq * (qn + 1) + 2 * bkv * lo;
  if (rn < N) mB = max(mB, bq * qn + 2 * bkv * hi);
  return DistinctMax{max(lo, hi), mB};
}

// a*b with a "> INT64_MAX" flag, without 128-bit overflow (operands < 2^96).
__device__ __forceinline__ u128 mul_le_i64(u128 a, u128 b, bool &bad) {
  if (a == 0 || b == 0) return 0;
  if (a > kI64Max || b > kI64Max) { bad = true; return 0; }
  return a * b;
}

// One (config, spec) record from the accumulated per-distinct maxima.
// Config-level part of a pair's record: T and the GPU totals (exact, 128-bit,
// with the exact-range rule R22); identical for every spec of the config.
struct AttnTotals {
  int status;     // config status
  int range_bad;  // a total >= 2^63 (reported after the spec's dtype check)
  int64_t T;
  int64_t tot[4];
};

__device__ __forceinline__ AttnTotals attn_totals(const AttnCfg &a, int cfg_status, int64_t L, uint64_t U) {
  AttnTotals t{};
  t.status = cfg_status;
  if (cfg_status) return t;
  t.T = L * a.nkv;
  const u128 Ua = (u128)U * (u128)a.nkv;  // < 2^63 (U < 2^32, nkv < 2^31)
  bool bad = false;
  const u128 totT = mul_le_i64((u128)4 * (u128)a.bq * (u128)a.hd * (u128)a.bkv, Ua, bad);
  const u128 totX = mul_le_i64((u128)a.bq * ((u128)a.bkv + 1), Ua, bad);
  const u128 totB = mul_le_i64((u128)2 * (u128)a.hd, (u128)a.bq * (u128)t.T + (u128)2 * (u128)a.bkv * Ua, bad);
  t.range_bad = bad || totT > kI64Max || totX > kI64Max || totB > kI64Max;
  t.tot[0] = (int64_t)totT;
  t.tot[1] = 0;
  t.tot[2] = (int64_t)totX;
  t.tot[3] = (int64_t)totB;
  return t;
}

// One pair: the spec-dependent checks in the oracle's order, the busiest-SM
// demands from the distinct-N maxima, and the record.
__device__ __forceinline__ void attn_emit_pair(const FeatOut &out, int64_t p, const AttnCfg &a, const AttnTotals &t,
                                               const DistinctMax &m, const DevSpec &s) {
  if (t.status) { emit_error(out, p, t.status); return; }
  const int tdt = (int)a.dt;
  if (!s.tensor_ok[tdt]) { emit_error(out, p, SP_PAIR_E_DTYPE); return; }
  if (t.range_bad) { emit_error(out, p, SP_PAIR_E_RANGE); return; }
  PairDemand d;
  d.T = t.T;
#pragma unroll
  for (int q = 0; q < 4; ++q) d.tot[q] = t.tot[q];
  d.mx[0] = (int64_t)4 * a.bq * a.hd * a.bkv * m.maxS;  // <= totT (maxS <= U*nkv)
  d.mx[1] = 0;
  d.mx[2] = (int64_t)a.bq * ((int64_t)a.bkv + 1) * m.maxS;
  d.mx[3] = (int64_t)2 * a.hd * m.maxB;
  emit_pair(out, p, d, a.fp, s, 5, tdt);
}

__device__ __forceinline__ void attn_emit(const FeatOut &out, int64_t p, const AttnCfg &a, int cfg_status,
                                          int64_t L, uint64_t U, const DistinctMax &m, const DevSpec &s) {
  attn_emit_pair(out, p, a, attn_totals(a, cfg_status, L, U), m, s);
}

// Whole per-config pipeline for one distinct set; per-distinct maxima go to
// mS[d * ms], mB[d * ms] (written by lane 0).
// Lpre >= 0: the task count L from attn_prepass (else counted here).
template <int ND, bool SMALL>
__device__ int attn_config(const AttnCfg &a, const AttnDivs &dv, int64_t Lpre, uint32_t *acc, int words,
                           uint32_t *scr, const int32_t (&N)[ND], const int32_t (&off)[ND], const FastDiv *fdN,
                           int32_t minN, int lane, int64_t &L, uint64_t &U, int64_t *mS, int64_t *mB, int64_t ms) {
  L = Lpre >= 0 ? Lpre : count_tasks(a, lane, dv);
  if (L > kI32Max || L * a.nkv > kI32Max) return SP_PAIR_E_RANGE;
  const int64_t T = L * a.nkv;
  if (T <= minN) {
    uint32_t umax;
    sparse_units(a, lane, dv, U, umax);
    if (U > (uint64_t)kU32Max) return SP_PAIR_E_RANGE;
    if (lane == 0)  // every SM holds at most one task: (lo, hi) = (umax, umax), see sparse_lohi
      for (int d = 0; d < ND; ++d) {
        mS[d * ms] = (int64_t)umax;
        mB[d * ms] = (int64_t)umax;
      }
    __syncwarp();
    return 0;
  }
  U = accumulate<ND, SMALL>(a, acc, words, scr, N, off, fdN, lane, dv);
  if (U > (uint64_t)kU32Max) return SP_PAIR_E_RANGE;
  const bool s32 = U * (uint64_t)a.nkv < (1ull << 32);
  // last region first: fold() duplicates region d into [off_d + N_d, off_d + 2 N_d),
  // over regions already folded and the (dead) request scratch that follows them
#pragma unroll 1
  for (int d = ND - 1; d >= 0; --d) {
    const DistinctLoHi m = s32 ? fold<uint32_t>(a, acc + off[d], N[d], fdN[d], (uint32_t)L, (uint32_t)T, lane)
                               : fold<uint64_t>(a, acc + off[d], N[d], fdN[d], (uint32_t)L, (uint32_t)T, lane);
    if (lane == 0) {  // (lo, hi): finish_max makes the record's maxima
      mS[d * ms] = m.lo;
      mB[d * ms] = m.hi;
    }
  }
  __syncwarp();
  return 0;
}

// Fields the record needs, read by the lane that owns config c (no validation:
// only used for configs whose stashed status is 0).
__device__ __forceinline__ AttnCfg load_cfg_lane(const ConfigView &v, int64_t c) {
  AttnCfg a{};
  a.nkv = __ldg(v.fields + (int64_t)NKV * v.ld + c);
  a.hd = __ldg(v.fields + (int64_t)HD * v.ld + c);
  a.bq = __ldg(v.fields + (int64_t)BQ * v.ld + c);
  a.bkv = __ldg(v.fields + (int64_t)BKV * v.ld + c);
  a.dt = __ldg(v.fields + (int64_t)DTYPE * v.ld + c);
  const int64_t smem = __ldg(v.fields + (int64_t)SMEM * v.ld + c);
  a.fp.smem = smem > 0 ? smem : ((int64_t)a.bq + 2 * (int64_t)a.bkv) * a.hd * 2;
  a.fp.warps = __ldg(v.fields + (int64_t)WARPS * v.ld + c);
  a.fp.regs = __ldg(v.fields + (int64_t)REGS * v.ld + c);
  return a;
}

// Per-warp shared-memory region: [stash of 32 configs | request scratch | accumulators].
// fold()'s duplicate of the last region (N <= kFoldDupMax, reads to 2N + 31) must fit in the request scratch
static_assert(kAttnScratchWords >= kFoldDupMax + 32, "fold duplicate overruns the warp region");

// ---- cross-mode pre-pass (thread per config).  Everything about a config that
// does not need its task stream is scalar work: validation (in the oracle's
// order, as load_cfg), g, the task count L (count_tasks), the range rule on L,
// and the FastDiv constants of g, BKV, BQ and the kv chunk (a 64-bit division
// each).  A warp per config did it warp-uniformly, 32x the instructions.
// Configs whose whole record follows from it are finished here: invalid
// configs, and sparse ones (T <= the smallest SM count of the range: every SM
// holds at most one task, so max_j S_j = the largest task's u for every
// distinct N).  The rest are flagged for attn_schedule_cross, which reads L
// and the divisors from the record.  Causal + split-KV configs (a chunk count
// per q-block) leave L to the warp.
enum : uint32_t { kPreWarp = 1u, kPreWarpCounts = 2u };

// Returns the config's cost for attn_order (its task count, clamped at 2^26), -1 if the
// warps have nothing to do for it.
__device__ __forceinline__ int attn_prepass_config(const ConfigView &v, const AttnResults &res, int32_t min_n,
                                                   int32_t n_slots, int64_t c) {
  if (c >= v.n_configs) return -1;
  int32_t f[12];
#pragma unroll
  for (int k = 0; k < 12; ++k) f[k] = __ldg(v.fields + (int64_t)k * v.ld + c);
  const int32_t bs = f[BS], nh = f[NH], nkv = f[NKV], hd = f[HD], bq = f[BQ], bkv = f[BKV], chunk = f[CHUNK],
                causal = f[CAUSAL], dt = f[DTYPE];
  const int64_t off = v.ragged_off ? __ldg(v.ragged_off + c) : -1;
  int st = 0;
  int32_t g = 0;
  // validation, in load_cfg's (the oracle's) order
  if (off < 0 || bs < 1 || nh < 1 || nkv < 1 || hd < 1) st = SP_PAIR_E_DIM;
  else if (bq < 1 || bkv < 1 || chunk < 0) st = SP_PAIR_E_TILE;  // kv_chunk -1: attn_planner_cross
  else if (f[WARPS] < 1 || f[REGS] < 1 || f[SMEM] < 0) st = SP_PAIR_E_RES;
  else if (dt != SP_BF16 && dt != SP_FP16) st = SP_PAIR_E_DTYPE;
  else if (nh % nkv != 0) st = SP_PAIR_E_HEADS;
  const int32_t *req = st ? nullptr : v.ragged + off;
  uint32_t flags = 0;
  int64_t L = 0;
  uint64_t U = 0;
  AttnDivs dv{};
  if (!st) {
    g = nh / nkv;
    dv.g = make_fd((uint32_t)g);
    dv.bkv = make_fd((uint32_t)bkv);
    dv.bq = make_fd((uint32_t)bq);
    dv.chunk = chunk > 0 ? make_fd((uint32_t)chunk) : FastDiv{1u, 1u, 0u};
    const bool csplit = chunk > 0 && causal;  // a chunk count per q-block: the warp counts L
    // one pass over the requests: validation (the first failing request decides),
    // the task count (count_tasks, saturating at 2^40) and, while the running
    // count can still be sparse (T <= min_n), the units (sparse_units)
    uint64_t part = 0;
    uint32_t um = 0;
    bool sparse = !csplit;
    for (int32_t b = 0; b < bs; ++b) {
      const int64_t q = __ldg(req + 2 * b), kv = __ldg(req + 2 * b + 1);
      if (q < 1 || kv < 1) st = SP_PAIR_E_DIM;
      else if (causal && kv < q) st = SP_PAIR_E_CAUSAL;
      else if (q * g > kI32Max) st = SP_PAIR_E_RANGE;
      if (st) break;
      if (csplit) continue;
      const uint32_t rows = (uint32_t)q * (uint32_t)g, nqb = dv.bq.div(rows + (uint32_t)bq - 1u);
      part = sat_add(part, chunk == 0 ? (uint64_t)nqb
                                      : (uint64_t)nqb * dv.chunk.div((uint32_t)kv + (uint32_t)chunk - 1u));
      sparse = sparse && part * (uint64_t)nkv <= (uint64_t)min_n;
      if (!sparse) continue;
      // units of one q-block of kv extent `need`: unsplit, one task of ceil(need/BKV);
      // split, n - 1 full chunks of ceil(chunk/BKV) and a last one (closed form)
      auto units = [&](uint32_t need, uint64_t &su, uint32_t &mu) {
        if (chunk == 0) {
          su = mu = dv.bkv.div(need + (uint32_t)bkv - 1u);
        } else {
          const uint32_t n = dv.chunk.div(need + (uint32_t)chunk - 1u);
          const uint32_t ul = dv.bkv.div(need - (n - 1u) * (uint32_t)chunk + (uint32_t)bkv - 1u);
          const uint32_t uf = n > 1 ? dv.bkv.div((uint32_t)chunk + (uint32_t)bkv - 1u) : 0u;
          su = (uint64_t)(n - 1u) * uf + ul;
          mu = max(uf, ul);
        }
      };
      uint64_t su;
      uint32_t mu;
      if (!causal) {  // every q-block has kv_need = kvlen
        units((uint32_t)kv, su, mu);
        U += (uint64_t)nqb * su;
        um = max(um, mu);
      } else {  // causal, unsplit (csplit is the warp's): q-block i has ceil(kv_need(i)/BKV) units
        // <= min_n tasks in all.  32-bit forms (kv_need >= 1, so ceil(n/BKV) = (n-1)/BKV + 1
        // with n - 1 < 2^31; (i+1) BQ < rows + BQ < 2^32); the last q-block needs the whole kv
        // (q_last = q - 1), so it holds the request's largest unit.
        const uint32_t qu = (uint32_t)q, kvu = (uint32_t)kv;
        uint64_t usum = 0;
        if (bq % g == 0 && bq < (1 << 30)) {
          // kv_need(i) = kv - max(t_i, 0), t_i = q - (i+1) BQ/g (R10-R11, as the schedule kernel)
          const int32_t a_per = bq / g;
          int32_t t = (int32_t)qu - a_per;
          for (uint32_t i = 0; i < nqb; ++i, t -= a_per) usum += dv.bkv.div31(kvu - 1u - (uint32_t)max(t, 0)) + 1u;
        } else {
          for (uint32_t i = 0, e1 = (uint32_t)bq; i < nqb; ++i, e1 += (uint32_t)bq) {
            const uint32_t q_last = dv.g.div31(min(e1, rows) - 1u);
            usum += dv.bkv.div31(min(kvu, kvu - qu + q_last + 1u) - 1u) + 1u;
          }
        }
        U += usum;
        um = max(um, dv.bkv.div31(kvu - 1u) + 1u);
      }
    }
    if (!st) {
      if (csplit) {
        flags = kPreWarp | kPreWarpCounts;
      } else {
        L = (int64_t)part;
        if (L > kI32Max || L * nkv > kI32Max) {
          st = SP_PAIR_E_RANGE;
          L = 0;
        } else if (!sparse) {
          flags = kPreWarp;
        } else if (U > (uint64_t)kU32Max) {
          st = SP_PAIR_E_RANGE;
          L = 0;
        } else {  // sparse: every SM holds at most one task
          for (int32_t d = 0; d < n_slots; ++d) {
            res.mS[(int64_t)d * res.ld + c] = (int64_t)um;  // (lo, hi) = (umax, umax): see finish_max
            res.mB[(int64_t)d * res.ld + c] = (int64_t)um;
          }
        }
      }
    }
    if (st || flags) U = 0;  // res.U is final for finished (sparse) configs only
  }
  res.st[c] = st;
  res.L[c] = L;
  res.U[c] = U;
  uint32_t *pr = res.pre + c;
  const int64_t ld = res.ld;
  pr[0] = flags;
  if (flags) {
    pr[1 * ld] = (uint32_t)g;
    pr[2 * ld] = dv.g.m;
    pr[3 * ld] = dv.g.s;
    pr[4 * ld] = dv.bkv.m;
    pr[5 * ld] = dv.bkv.s;
    pr[6 * ld] = dv.bq.m;
    pr[7 * ld] = dv.bq.s;
    pr[8 * ld] = dv.chunk.m;
    pr[9 * ld] = dv.chunk.s;
  }
  // cost estimate for attn_order: the task count, clamped (a chunk's sum stays below 2^31);
  // causal split-KV configs (L counted by the warp) count as the largest
  return !flags ? -1 : (flags & kPreWarpCounts) ? (1 << 26) : (int)min(L * (int64_t)nkv, (int64_t)1 << 26);
}

__global__ void __launch_bounds__(256) attn_prepass(ConfigView v, AttnResults res, int32_t min_n, int32_t n_slots) {
  __shared__ int s_hist[kAttnCostBuckets];
  if (threadIdx.x < kAttnCostBuckets) s_hist[threadIdx.x] = 0;
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int t = attn_prepass_config(v, res, min_n, n_slots, c);
  // a chunk of 32 configs (this warp's) costs the sum of its configs' tasks: class floor(log2 sum)
  const uint32_t sum = __reduce_add_sync(0xffffffffu, (uint32_t)max(t, 0));
  const bool any = __any_sync(0xffffffffu, t >= 0);
  const int cb = any ? 31 - __clz((int)max(sum, 1u)) : -1;
  if ((threadIdx.x & 31) == 0 && c < v.n_configs) {
    res.chunk_b[c >> 5] = (int8_t)cb;
    if (cb >= 0) atomicAdd(s_hist + cb, 1);
  }
  __syncthreads();
  if (threadIdx.x < kAttnCostBuckets && s_hist[threadIdx.x]) atomicAdd(res.hist + threadIdx.x, s_hist[threadIdx.x]);
}

// The chunks of 32 configs with warp work, heaviest cost class first (res.order;
// see kAttnCostBuckets).  Thread per chunk: its class (attn_prepass), a
// block-local slot by a shared atomic, a per-(block, class) range from the
// global cursors.
__global__ void __launch_bounds__(256) attn_order(AttnResults res, int64_t n_chunks) {
  __shared__ int s_cnt[kAttnCostBuckets], s_base[kAttnCostBuckets];
  if (threadIdx.x < kAttnCostBuckets) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int b = k < n_chunks ? (int)res.chunk_b[k] : -1;
  const int slot = b >= 0 ? atomicAdd(&s_cnt[b], 1) : 0;
  __syncthreads();
  if (threadIdx.x < kAttnCostBuckets) {
    const int bb = threadIdx.x;
    int start = 0;  // chunks of the heavier classes
    for (int x = kAttnCostBuckets - 1; x > bb; --x) start += res.hist[x];
    s_base[bb] = s_cnt[bb] ? start + atomicAdd(res.hist + kAttnCostBuckets + bb, s_cnt[bb]) : 0;
  }
  __syncthreads();
  if (b >= 0) res.order[s_base[b] + slot] = (int32_t)k;
}

// A flagged config for the warp: its fields (lanes 0..11, one load each) and the
// pre-pass record (lanes 0..9), broadcast by shuffles.  Valid by construction.
__device__ __forceinline__ AttnCfg load_cfg_pre(const ConfigView &v, const AttnResults &res, int64_t c, int lane,
                                                AttnDivs &dv, uint32_t &flags) {
  AttnCfg a{};
  const int32_t f = lane < 12 ? __ldg(v.fields + (int64_t)lane * v.ld + c) : 0;
  const uint32_t r = lane < kAttnPreWords ? __ldg(res.pre + (int64_t)lane * res.ld + c) : 0u;
  a.bs = __shfl_sync(0xffffffffu, f, BS);
  a.nh = __shfl_sync(0xffffffffu, f, NH);
  a.nkv = __shfl_sync(0xffffffffu, f, NKV);
  a.hd = __shfl_sync(0xffffffffu, f, HD);
  a.bq = __shfl_sync(0xffffffffu, f, BQ);
  a.bkv = __shfl_sync(0xffffffffu, f, BKV);
  a.chunk = __shfl_sync(0xffffffffu, f, CHUNK);
  a.causal = __shfl_sync(0xffffffffu, f, CAUSAL);
  a.dt = __shfl_sync(0xffffffffu, f, DTYPE);
  flags = __shfl_sync(0xffffffffu, r, 0);
  a.g = (int32_t)__shfl_sync(0xffffffffu, r, 1);
  dv.g = FastDiv{(uint32_t)a.g, __shfl_sync(0xffffffffu, r, 2), __shfl_sync(0xffffffffu, r, 3)};
  dv.bkv = FastDiv{(uint32_t)a.bkv, __shfl_sync(0xffffffffu, r, 4), __shfl_sync(0xffffffffu, r, 5)};
  dv.bq = FastDiv{(uint32_t)a.bq, __shfl_sync(0xffffffffu, r, 6), __shfl_sync(0xffffffffu, r, 7)};
  dv.chunk = FastDiv{a.chunk > 0 ? (uint32_t)a.chunk : 1u, __shfl_sync(0xffffffffu, r, 8),
                     __shfl_sync(0xffffffffu, r, 9)};
  a.req = v.ragged + __ldg(v.ragged_off + c);
  return a;
}

// CROSS mode.  Warps take chunks of 32 consecutive configs from a per-group
// Schedule kernel (cross mode): warps pull chunks of 32 configs; per config
// the head-0 task stream is accumulated once per distinct SM count of the
// launch group and folded into per-distinct maxima, written to the context's
// result scratch (res.mS/mB[slot][c], res.st/L/U[c]).  The records are written
// by attn_emit_cross: keeping the emit code (128-bit range checks, fp64
// cycle conversions) out of this kernel keeps its hot code inside the
// instruction cache (ncu: stalled_no_instructions was its top stall).
template <int ND, bool SMALL>
__global__ void __launch_bounds__(kWarps * 32, SP_ATTN_MINB) attn_schedule_cross(ConfigView cfg, AttnPlan plan,
                                                                             AttnResults res) {
  extern __shared__ uint32_t smem[];
  __shared__ FastDiv s_fd[kMaxDistinct];
  const AttnGroup grp = plan.groups[blockIdx.y];
  int32_t N[ND], off[ND];
  int32_t minN = INT32_MAX, words = 0;
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    N[d] = __ldg(plan.distinct_n + grp.distinct_first + d);
    off[d] = __ldg(plan.distinct_off + grp.distinct_first + d);
    minN = min(minN, N[d]);
    words = max(words, off[d] + N[d] + kAttnSlack);
  }
  words = (words + 3) & ~3;
  if (threadIdx.x < ND) s_fd[threadIdx.x] = make_fd((uint32_t)N[threadIdx.x]);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // warp region: [accumulators: words_per_warp - kAttnScratchWords][request scratch]
  uint32_t *acc = smem + (size_t)warp * plan.words_per_warp;
  uint32_t *scr = acc + (plan.words_per_warp - kAttnScratchWords);
  int *counter = plan.counters + blockIdx.y;
  int64_t *mS = res.mS + (int64_t)grp.distinct_first * res.ld, *mB = res.mB + (int64_t)grp.distinct_first * res.ld;
  // chunks of 32 configs with work for the warps, heaviest cost class first (attn_order)
  const int64_t F = __reduce_add_sync(0xffffffffu, lane < kAttnCostBuckets ? (uint32_t)__ldg(res.hist + lane) : 0u);
  const int64_t C = cfg.n_configs;
  for (;;) {
    int64_t item = 0;
    if (lane == 0) item = atomicAdd(counter, 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= F) break;
    const int64_t c0 = (int64_t)__ldg(res.order + item) * 32;
    // configs the pre-pass left to the warps (invalid and sparse ones are done)
    const bool mine = c0 + lane < C && (__ldg(res.pre + c0 + lane) & kPreWarp);
    uint32_t todo = __ballot_sync(0xffffffffu, mine);
    while (todo) {
      const int j = __ffs(todo) - 1;
      todo &= todo - 1;
      const int64_t c = c0 + j;
      AttnDivs dv;
      uint32_t flags;
      const AttnCfg a = load_cfg_pre(cfg, res, c, lane, dv, flags);
      int64_t L = 0;
      uint64_t U = 0;
      const int64_t Lpre = (flags & kPreWarpCounts) ? -1 : __ldg(res.L + c);
      const int st = attn_config<ND, SMALL>(a, dv, Lpre, acc, words, scr, N, off, s_fd, minN, lane, L, U, mS + c,
                                            mB + c, res.ld);
      // the per-config fields do not depend on the group: group 0 writes them
      if (lane == 0 && blockIdx.y == 0) {
        res.st[c] = st;
        res.L[c] = L;
        res.U[c] = U;
      }
    }
  }
}

// Emit kernel (cross mode): thread per config, specs of the range in turn;
// consecutive threads write consecutive records of one spec (full sectors).
constexpr int kEmitSpecTile = 16;

// Record writer of the cross path: thread per config, grid y over tiles of 16
// specs staged in shared memory (with their distinct-N slots).  The config-level
// totals are computed once per config; each spec then costs its dtype check, the
// busiest-SM demands and the record store (pair p = j * C + c: a warp's stores
// to every SoA row are 32 consecutive elements).
#ifndef SP_EMIT_MINB
#define SP_EMIT_MINB 3  // 80 registers, 3 blocks/SM: measured best of 1, 3, 4 on cfg2 (128 registers left it at 23% warps)
#endif
__global__ void __launch_bounds__(256, SP_EMIT_MINB) attn_emit_cross(ConfigView cfg, const DevSpec *__restrict__ specs, int g0,
                                                       int n_specs, const int32_t *__restrict__ spec_slot,
                                                       AttnResults res, FeatOut out) {
  __shared__ DevSpec s_spec[kEmitSpecTile];
  __shared__ int32_t s_slot[kEmitSpecTile];
  __shared__ FastDiv s_fn[kEmitSpecTile];
  const int j0 = blockIdx.y * kEmitSpecTile, j1 = min(n_specs, j0 + kEmitSpecTile);
  {
    const int n_words = (j1 - j0) * (int)(sizeof(DevSpec) / 16);
    const int4 *src = reinterpret_cast<const int4 *>(specs + g0 + j0);
    int4 *dst = reinterpret_cast<int4 *>(s_spec);
    for (int i = threadIdx.x; i < n_words; i += blockDim.x) dst[i] = __ldg(src + i);
    if (threadIdx.x < j1 - j0) {
      s_slot[threadIdx.x] = __ldg(spec_slot + j0 + threadIdx.x);
      s_fn[threadIdx.x] = make_fd((uint32_t)__ldg(&specs[g0 + j0 + threadIdx.x].num_sms));
    }
  }
  __syncthreads();
  const int64_t C = cfg.n_configs;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const int st = __ldg(res.st + c);
  const AttnCfg al = st ? AttnCfg{} : load_cfg_lane(cfg, c);
  const AttnTotals tt = attn_totals(al, st, st ? 0 : __ldg(res.L + c), st ? 0 : __ldg(res.U + c));
  for (int j = j0; j < j1; ++j) {
    const int64_t slot = s_slot[j - j0];
    DistinctMax m{0, 0};
    if (!st)
      m = finish_max(__ldg(res.mS + slot * res.ld + c), __ldg(res.mB + slot * res.ld + c), tt.T, s_fn[j - j0],
                     al.bq, al.bkv);
    attn_emit_pair(out, (int64_t)j * C + c, al, tt, m, s_spec[j - j0]);
  }
}

// One (config, spec) pair through the per-pair cyclic path (LIST mode and
// planner configs): accumulate + fold for the pair's own SM count; the
// planner's chunk (R24) replaces kv_chunk = -1.  Lane 0 writes record p.
__device__ void attn_one_pair(const ConfigView &cfg, int64_t c, const DevSpec &sp, int64_t p, uint32_t *acc,
                              uint32_t *scr, FastDiv *fd, int64_t *sm, int lane, const FeatOut &out) {
  const int32_t N[1] = {sp.num_sms}, off[1] = {0};
  if (lane == 0) *fd = make_fd((uint32_t)N[0]);
  __syncwarp();
  AttnCfg a = load_cfg(cfg, c, lane);
  int st = a.status;
  int64_t L = 0;
  uint64_t U = 0;
  const int words = (N[0] + kAttnSlack + 3) & ~3;
  if (st == 0) {
    if (a.chunk == -1) a.chunk = plan_chunk(a, sp, lane);
    const AttnDivs dv = make_divs(a);
    if (N[0] >= kAttnLazyMinN)
      st = attn_config<1, false>(a, dv, -1, acc, words, scr, N, off, fd, N[0], lane, L, U, sm, sm + 1, 1);
    else
      st = attn_config<1, true>(a, dv, -1, acc, words, scr, N, off, fd, N[0], lane, L, U, sm, sm + 1, 1);
  }
  if (lane == 0)
    attn_emit(out, p, a, st, L, U, st ? DistinctMax{0, 0} : finish_max(sm[0], sm[1], L * a.nkv, *fd, a.bq, a.bkv),
              sp);
  __syncwarp();
}

__global__ void __launch_bounds__(kWarps * 32, 2) featurize_attention_list(ConfigView cfg,
                                                                           const DevSpec *__restrict__ specs,
                                                                           int n_specs, int words_per_warp,
                                                                           int64_t n_pairs,
                                                                           const int64_t *__restrict__ cfg_idx,
                                                                           const int32_t *__restrict__ spec_idx,
                                                                           FeatOut out) {
  extern __shared__ uint32_t smem[];
  __shared__ FastDiv s_fd[kWarps];
  __shared__ int64_t s_m[kWarps][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t *region = smem + (size_t)warp * words_per_warp;
  uint32_t *acc = region, *scr = acc + (words_per_warp - kAttnScratchWords);
  for (int64_t p = (int64_t)blockIdx.x * kWarps + warp; p < n_pairs; p += (int64_t)gridDim.x * kWarps) {
    const int64_t c = __ldg(cfg_idx + p);
    const int32_t g = __ldg(spec_idx + p);
    if (c < 0 || c >= cfg.n_configs || g < 0 || g >= n_specs) {
      if (lane == 0) emit_error(out, p, SP_PAIR_E_INDEX);
      continue;
    }
    attn_one_pair(cfg, c, specs[g], p, acc, scr, s_fd + warp, s_m[warp], lane, out);
  }
}

// CROSS mode, planner configs (kv_chunk = -1): the cross kernels wrote them
// as SP_PAIR_E_TILE (their chunk depends on the spec); this pass, launched
// after attn_emit_cross on the same stream, rewrites their records.  A warp
// takes 32 configs, skips the others with one ballot, and runs each planner
// config through every spec of the range on the per-pair path.
__global__ void __launch_bounds__(kWarps * 32, 2) attn_planner_cross(ConfigView cfg, const DevSpec *__restrict__ specs,
                                                                     int g0, int n_specs, int words_per_warp,
                                                                     FeatOut out) {
  extern __shared__ uint32_t smem[];
  __shared__ FastDiv s_fd[kWarps];
  __shared__ int64_t s_m[kWarps][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t *acc = smem + (size_t)warp * words_per_warp;
  uint32_t *scr = acc + (words_per_warp - kAttnScratchWords);
  const int64_t C = cfg.n_configs;
  for (int64_t c0 = ((int64_t)blockIdx.x * kWarps + warp) * 32; c0 < C; c0 += (int64_t)gridDim.x * kWarps * 32) {
    const int64_t cl = c0 + lane;
    const bool plan = cl < C && __ldg(cfg.fields + (int64_t)CHUNK * cfg.ld + cl) == -1;
    unsigned m = __ballot_sync(0xffffffffu, plan);
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      for (int k = 0; k < n_specs; ++k)
        attn_one_pair(cfg, c0 + j, specs[g0 + k], (int64_t)k * C + c0 + j, acc, scr, s_fd + warp, s_m[warp], lane,
                      out);
    }
  }
}

// ---------------------------------------------------------------------------
// Non-cyclic schedulers: SP_SCHED_GREEDY (hardware RR
// with retirement: the first N*occ tasks dealt cyclically, then each task to
// the SM with the least busy time) and SP_SCHED_MINHEAP
// (persistent kernel: W = min(N*occ, T) workers pinned round-robin to SMs,
// each task to the least-loaded worker).  Ties: lowest index.
//
// A task's busy time max(Tensor/Th_T, XU/Th_X) is u * max(4 BQ hd BKV / Th_T,
// BQ (BKV+1) / Th_X): both pipes scale with its kv units u, so the greedy
// order is decided by u-sums alone -- exact integers, no spec throughput.
// The decisions are sequential, so one warp walks one pair's full task list
// (all kv-heads, R4 order) and keeps the per-target loads in shared memory
// with a two-level min structure: per 32-entry group, its least (load, index);
// a task costs one scan of the group minima, one update and one group rescan,
// each a warp reduction.  This is the modelling path for persistent kernels
// (FlashInfer FA3); it is ~100x slower per pair than the cyclic path.
struct SimRegion {
  uint64_t *load;   // [W]
  uint32_t *count;  // [W]
  uint64_t *gmin;   // [G] least load of each 32-entry group
  uint32_t *gidx;   // [G] its index
};

// Warp-wide least (load, idx): least load, then lowest index among equals.
__device__ __forceinline__ void warp_argmin(uint64_t &ld, uint32_t &ix) {
  const uint32_t hi = __reduce_min_sync(0xffffffffu, (uint32_t)(ld >> 32));
  const uint32_t lo = __reduce_min_sync(0xffffffffu, (uint32_t)(ld >> 32) == hi ? (uint32_t)ld : 0xffffffffu);
  const bool win = (uint32_t)(ld >> 32) == hi && (uint32_t)ld == lo;
  ix = __reduce_min_sync(0xffffffffu, win ? ix : 0xffffffffu);
  ld = ((uint64_t)hi << 32) | lo;
}

__device__ __forceinline__ void group_rescan(const SimRegion &r, uint32_t W, uint32_t g, int lane) {
  const uint32_t i = g * 32 + lane;
  uint64_t ld = i < W ? r.load[i] : ~0ull;
  uint32_t ix = i < W ? i : 0xffffffffu;
  warp_argmin(ld, ix);
  if (lane == 0) {
    r.gmin[g] = ld;
    r.gidx[g] = ix;
  }
  __syncwarp();
}

template <int MODE>  // 1 GREEDY, 2 MINHEAP
__device__ void attn_sim_pair(const AttnCfg &a, const SimRegion &r, uint32_t N, uint32_t occ, int lane, int64_t &L,
                              uint64_t &U, DistinctMax &m, int &st) {
  const FastDiv fg = make_fd((uint32_t)a.g);
  L = count_tasks(a, lane, make_divs(a));
  if (L > kI32Max || L * a.nkv > kI32Max) { st = SP_PAIR_E_RANGE; return; }
  const uint32_t T = (uint32_t)(L * a.nkv);
  const uint64_t slots = (uint64_t)N * occ;
  const uint32_t W = MODE == 1 ? N : (uint32_t)(slots < T ? slots : T);
  const uint32_t R = MODE == 1 ? (uint32_t)(slots < T ? slots : T) : W;  // tasks placed without a search
  const uint32_t G = (W + 31) / 32;
  for (uint32_t i = lane; i < W; i += 32) {
    r.load[i] = 0;
    r.count[i] = 0;
  }
  __syncwarp();
  uint32_t t = 0, tgt = 0;  // task index; its cyclic target while t < R (tgt = t mod N, or t)
  uint64_t usum = 0;
  auto place = [&](uint32_t u) {
    if (t < R) {
      if (lane == 0) {
        r.load[tgt] += u;
        r.count[tgt] += 1;
      }
      ++tgt;
      if (MODE == 1 && tgt == N) tgt = 0;
      if (++t == R && R < T) {  // all resident slots taken: build the group minima
        __syncwarp();
        for (uint32_t g = 0; g < G; ++g) group_rescan(r, W, g, lane);
      }
      return;
    }
    uint64_t ld = ~0ull;
    uint32_t ix = 0xffffffffu;
    for (uint32_t g = lane; g < G; g += 32) {
      const uint64_t v = r.gmin[g];
      const uint32_t vi = r.gidx[g];
      if (v < ld || (v == ld && vi < ix)) { ld = v; ix = vi; }
    }
    warp_argmin(ld, ix);
    if (lane == 0) {
      r.load[ix] += u;
      r.count[ix] += 1;
    }
    __syncwarp();
    group_rescan(r, W, ix / 32, lane);
    ++t;
  };
  // the task stream (R4): kv-head outermost, then request, q-block, kv-chunk
  for (int32_t h = 0; h < a.nkv; ++h) {
    for (int64_t b = 0; b < a.bs; ++b) {
      const uint32_t q = __ldg(a.req + 2 * b), kv = __ldg(a.req + 2 * b + 1);
      const uint64_t rows = (uint64_t)q * a.g, nqb = (rows + a.bq - 1) / a.bq;
      for (uint64_t i = 0; i < nqb; ++i) {
        const uint32_t need = kv_need(i, a.bq, rows, q, kv, a.causal, fg);
        if (a.chunk == 0) {
          const uint32_t u = (uint32_t)((need + a.bkv - 1) / a.bkv);
          if (h == 0) usum += u;
          place(u);
        } else {
          for (uint64_t c0 = 0; c0 < need; c0 += a.chunk) {
            const uint32_t u = (uint32_t)((min((uint64_t)a.chunk, need - c0) + a.bkv - 1) / a.bkv);
            if (h == 0) usum += u;
            place(u);
          }
        }
      }
    }
  }
  __syncwarp();
  U = usum;
  if (U > (uint64_t)kU32Max) { st = SP_PAIR_E_RANGE; return; }
  // per-SM task count n_j and unit sum S_j (MINHEAP: sum of the SM's workers)
  int64_t mS = 0, mB = 0;
  for (uint32_t j = lane; j < N; j += 32) {
    uint64_t S = 0, n = 0;
    for (uint32_t w = j; w < W; w += N) {
      S += r.load[w];
      n += r.count[w];
    }
    mS = max(mS, (int64_t)S);
    mB = max(mB, (int64_t)a.bq * (int64_t)n + 2 * (int64_t)a.bkv * (int64_t)S);
  }
  m.maxS = warp_max64(mS);
  m.maxB = warp_max64(mB);
  st = 0;
}

template <int MODE>
__global__ void __launch_bounds__(kSimWarps * 32) attn_sched_sim(ConfigView cfg, const DevSpec *__restrict__ specs,
                                                               int g0, int n_specs, int64_t n_pairs,
                                                               const int64_t *__restrict__ cfg_idx,
                                                               const int32_t *__restrict__ spec_idx,
                                                               int64_t words_per_warp, FeatOut out) {
  extern __shared__ uint64_t sim_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  uint64_t *base = sim_smem + (size_t)warp * words_per_warp;
  const int64_t C = cfg.n_configs;
  for (int64_t p = (int64_t)blockIdx.x * nw + warp; p < n_pairs; p += (int64_t)gridDim.x * nw) {
    int64_t c;
    int32_t g;
    if (cfg_idx) {
      c = __ldg(cfg_idx + p);
      g = __ldg(spec_idx + p);
      if (c < 0 || c >= C || g < 0 || g >= n_specs) {
        if (lane == 0) emit_error(out, p, SP_PAIR_E_INDEX);
        continue;
      }
    } else {
      c = p % C;
      g = g0 + (int32_t)(p / C);
    }
    const DevSpec &sp = specs[g];
    AttnCfg a = load_cfg(cfg, c, lane);
    int st = a.status;
    int64_t L = 0;
    uint64_t U = 0;
    DistinctMax m{0, 0};
    if (st == 0 && a.chunk == -1) a.chunk = plan_chunk(a, sp, lane);  // R24
    if (st == 0) {
      const uint32_t N = (uint32_t)sp.num_sms;
      const uint32_t occ = (uint32_t)occupancy(a.fp, sp);
      const uint64_t W = MODE == 1 ? N : (uint64_t)N * occ;  // upper bound of the targets
      SimRegion r;
      r.load = base;
      r.count = reinterpret_cast<uint32_t *>(base + W);
      r.gmin = base + W + (W + 1) / 2;
      r.gidx = reinterpret_cast<uint32_t *>(r.gmin + (W + 31) / 32);
      attn_sim_pair<MODE>(a, r, N, occ, lane, L, U, m, st);
    }
    if (lane == 0) attn_emit(out, p, a, st, L, U, m, sp);
    __syncwarp();
  }
}

// 64-bit words of shared memory one warp needs for W targets.
__host__ __device__ constexpr int64_t sim_words(int64_t W) { return W + (W + 1) / 2 + 2 * ((W + 31) / 32) + 2; }

template <int ND, bool SMALL>
int launch_cross(const ConfigView &cfg, const AttnPlan &plan, const AttnResults &res, int num_device_sms,
                 cudaStream_t st, int group_y0, int n_groups, const LaunchHook &hook) {
  const size_t smem = (size_t)kWarps * plan.words_per_warp * 4;
  cudaError_t e = cudaFuncSetAttribute(attn_schedule_cross<ND, SMALL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return (int)e;
  // chunks of 32 configs are handed out dynamically: launch about as many
  // warps as can be resident, never more than there are chunks
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, attn_schedule_cross<ND, SMALL>, kWarps * 32, smem);
  if (e != cudaSuccess) return (int)e;
  const int64_t chunks = (cfg.n_configs + 31) / 32;
  int64_t want = (chunks + kWarps - 1) / kWarps;
  int64_t cap = (int64_t)num_device_sms * (per_sm > 0 ? per_sm : 1);
  AttnPlan sub = plan;
  sub.groups = plan.groups + group_y0;
  sub.counters = plan.counters + group_y0;
  dim3 grid((unsigned)(want < cap ? want : cap), (unsigned)n_groups);
  hook.on_begin("attn_schedule_cross", st);
  attn_schedule_cross<ND, SMALL><<<grid, kWarps * 32, smem, st>>>(cfg, sub, res);
  hook.on_end(st);
  return (int)cudaGetLastError();
}

template <bool SMALL>
int launch_nd(int nd, const ConfigView &cfg, const AttnPlan &plan, const AttnResults &res, int sms,
              cudaStream_t st, int y0, int ny, const LaunchHook &hook) {
  switch (nd) {
    case 1: return launch_cross<1, SMALL>(cfg, plan, res, sms, st, y0, ny, hook);
    case 2: return launch_cross<2, SMALL>(cfg, plan, res, sms, st, y0, ny, hook);
    case 3: return launch_cross<3, SMALL>(cfg, plan, res, sms, st, y0, ny, hook);
    case 4: return launch_cross<4, SMALL>(cfg, plan, res, sms, st, y0, ny, hook);
    case 5: return launch_cross<5, SMALL>(cfg, plan, res, sms, st, y0, ny, hook);
    case 6: return launch_cross<6, SMALL>(cfg, plan, res, sms, st, y0, ny, hook);
    case 7: return launch_cross<7, SMALL>(cfg, plan, res, sms, st, y0, ny, hook);
    default: return launch_cross<8, SMALL>(cfg, plan, res, sms, st, y0, ny, hook);
  }
}

// ------------------------------------------------------------------ clamped edge tiles (attention)

// SPEC's clamped reading applied to FA2 tasks (NEXT-4): a task
// computes only its in-range query rows qr = min(BQ, rows - i BQ) over its
// exact kv length len (no BKV padding): Tensor 4 qr len hd, XU qr len + qr
// ceil(len/BKV), bytes (qr hd + 2 len hd) bpe.  Demands are no longer affine
// in one unit count, so the head-rotation identity of the cross kernel does not
// apply: a warp per pair walks every task (all kv-heads, in task order, lanes
// over 32 q-blocks with a scan of their chunk counts for the task index) and
// adds its demands to three per-SM arrays in shared memory (64-bit atomics:
// exact in any order), then takes the totals and the per-quantity maxima.
// O(T/32) per pair: a modelling variant.
__device__ void attn_clamped_pair(const ConfigView &cfg, int64_t c, const DevSpec &sp, int64_t p,
                                  unsigned long long *S, int lane, const FeatOut &out) {
  AttnCfg a = load_cfg(cfg, c, lane);
  if (a.status) {
    if (lane == 0) emit_error(out, p, a.status);
    return;
  }
  if (a.chunk == -1) a.chunk = plan_chunk(a, sp, lane);
  const FastDiv fg = make_fd((uint32_t)a.g);
  const int64_t L = count_tasks(a, lane, make_divs(a));
  if (L > kI32Max || L * a.nkv > kI32Max) {
    if (lane == 0) emit_error(out, p, SP_PAIR_E_RANGE);
    return;
  }
  const int N = sp.num_sms;
  const FastDiv fN = make_fd((uint32_t)N);
  for (int i = lane; i < 3 * N; i += 32) S[i] = 0ull;
  __syncwarp();
  u128 tot[3] = {0, 0, 0};
  uint64_t U = 0;
  const uint64_t hd = (uint64_t)a.hd, bq = (uint64_t)a.bq, bkv = (uint64_t)a.bkv, bpe = 2;  // bf16/fp16 (validated)
  uint32_t base = 0;  // index of the next task (< 2^31)
  for (int32_t h = 0; h < a.nkv; ++h) {
    for (int64_t b = 0; b < a.bs; ++b) {
      const uint32_t q = __ldg(a.req + 2 * b), kv = __ldg(a.req + 2 * b + 1);
      const uint64_t rows = (uint64_t)q * a.g, nqb = (rows + bq - 1) / bq;
      for (uint64_t i0 = 0; i0 < nqb; i0 += 32) {
        const uint64_t i = i0 + lane;
        const bool act = i < nqb;
        const uint32_t need = act ? kv_need(i, bq, rows, q, kv, a.causal != 0, fg) : 0u;
        const uint32_t nch = !act ? 0u : (a.chunk > 0 ? (need + (uint32_t)a.chunk - 1u) / (uint32_t)a.chunk : 1u);
        uint32_t incl = nch;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const uint32_t start = base + incl - nch;
        base += __shfl_sync(0xffffffffu, incl, 31);
        const uint64_t qr = act ? min(bq, rows - i * bq) : 0;
        for (uint32_t cc = 0; cc < nch; ++cc) {
          const uint64_t len = a.chunk > 0 ? min((uint64_t)a.chunk, (uint64_t)need - (uint64_t)cc * a.chunk) : need;
          const uint64_t units = (len + bkv - 1) / bkv;
          const uint64_t w[3] = {4 * qr * len * hd, qr * len + qr * units, (qr * hd + 2 * len * hd) * bpe};
          const uint32_t j = fN.mod(start + cc);
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            atomicAdd(S + k * N + j, (unsigned long long)w[k]);
            tot[k] += w[k];
          }
          if (h == 0) U += units;
        }
      }
    }
  }
  __syncwarp();
  U = warp_sum_u64(U);
  int bad = 0;
  int64_t T64[3], mx[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const unsigned long long lo = (unsigned long long)tot[k], hi = (unsigned long long)(tot[k] >> 64);
    u128 t = 0;
    for (int l = 0; l < 32; ++l)
      t += ((u128)__shfl_sync(0xffffffffu, hi, l) << 64) | __shfl_sync(0xffffffffu, lo, l);
    bad |= t > kI64Max;
    T64[k] = (int64_t)t;
    unsigned long long m = 0;
    for (int jj = lane; jj < N; jj += 32) m = max(m, S[k * N + jj]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    mx[k] = (int64_t)m;
  }
  __syncwarp();
  if (lane != 0) return;
  if (U > (uint64_t)kU32Max) { emit_error(out, p, SP_PAIR_E_RANGE); return; }  // validation order: before dtype
  if (!sp.tensor_ok[a.dt]) { emit_error(out, p, SP_PAIR_E_DTYPE); return; }
  if (bad) { emit_error(out, p, SP_PAIR_E_RANGE); return; }
  PairDemand d;
  d.T = L * a.nkv;
  d.tot[0] = T64[0]; d.tot[1] = 0; d.tot[2] = T64[1]; d.tot[3] = T64[2];
  d.mx[0] = mx[0]; d.mx[1] = 0; d.mx[2] = mx[1]; d.mx[3] = mx[2];
  emit_pair(out, p, d, a.fp, sp, 5, a.dt);
}

__global__ void attn_clamped_kernel(ConfigView cfg, const DevSpec *__restrict__ specs, int g0, int n_specs,
                                    int64_t n_pairs, const int64_t *__restrict__ cfg_idx,
                                    const int32_t *__restrict__ spec_idx, int max_sms, FeatOut out) {
  extern __shared__ unsigned long long s_acc[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  unsigned long long *S = s_acc + (size_t)warp * 3 * max_sms;
  for (int64_t p = (int64_t)blockIdx.x * nw + warp; p < n_pairs; p += (int64_t)gridDim.x * nw) {
    int64_t c;
    int g;
    if (cfg_idx) {
      c = __ldg(cfg_idx + p);
      g = __ldg(spec_idx + p);
      if (c < 0 || c >= cfg.n_configs || g < 0 || g >= n_specs) {
        if (lane == 0) emit_error(out, p, SP_PAIR_E_INDEX);
        continue;
      }
    } else {
      g = g0 + (int)(p / cfg.n_configs);
      c = p - (int64_t)(g - g0) * cfg.n_configs;
    }
    attn_clamped_pair(cfg, c, specs[g], p, S, lane, out);
    __syncwarp();
  }
}

}  // namespace

int launch_attention_sim(int mode, const ConfigView &cfg, const DevSpec *specs, int spec_begin, int spec_end,
                         int n_specs, int64_t n_pairs, const int64_t *cfg_idx, const int32_t *spec_idx,
                         int64_t max_targets, const FeatOut &out, int num_device_sms, void *stream,
                         const LaunchHook &hook) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (n_pairs == 0) return 0;
  const int64_t words = sim_words(max_targets);
  const int64_t budget = 227 * 1024;
  const int nw = (int)std::min<int64_t>(kSimWarps, budget / (words * 8));
  if (nw < 1) return (int)cudaErrorInvalidValue;  // the caller checks attention_sim_smem_bytes first
  const size_t smem = (size_t)nw * words * 8;
  void (*kern)(ConfigView, const DevSpec *, int, int, int64_t, const int64_t *, const int32_t *, int64_t, FeatOut) =
      mode == SP_SCHED_GREEDY ? attn_sched_sim<1> : attn_sched_sim<2>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  int64_t want = (n_pairs + nw - 1) / nw;
  int64_t cap = (int64_t)num_device_sms * 16;
  hook.on_begin(mode == SP_SCHED_GREEDY ? "attn_sched_greedy" : "attn_sched_minheap", st);
  kern<<<(unsigned)(want < cap ? want : cap), nw * 32, smem, st>>>(
      cfg, specs, spec_begin, cfg_idx ? n_specs : spec_end - spec_begin, n_pairs, cfg_idx, spec_idx, words, out);
  hook.on_end(st);
  return (int)cudaGetLastError();
}

// shared memory one warp of the simulation kernel needs (<= 227 KB or unsupported)
int64_t attention_sim_smem_bytes(int64_t max_targets) { return sim_words(max_targets) * 8; }

// Per-config record of the fused attention path (layout in sp_internal.h): what
// attn_emit_cross computes once per config before its spec loop -- status, T
// and the exact GPU totals (attn_totals) -- for the fused kernel's producers,
// which finish each pair from it, its spec and the slot's (lo, hi).
__global__ void __launch_bounds__(256) attn_fuse_prep(ConfigView cfg, AttnResults res, uint64_t *__restrict__ pre,
                                                      int64_t ldc) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cfg.n_configs) return;
  const int st = __ldg(res.st + c);
  const bool planner = __ldg(cfg.fields + (int64_t)CHUNK * cfg.ld + c) == -1;
  const AttnCfg al = st ? AttnCfg{} : load_cfg_lane(cfg, c);
  const AttnTotals tt = attn_totals(al, st, st ? 0 : __ldg(res.L + c), st ? 0 : __ldg(res.U + c));
  pre[c] = (uint64_t)(uint32_t)tt.status | (uint64_t)(tt.range_bad ? 1u : 0u) << 8 | (uint64_t)(planner ? 1u : 0u) << 9 |
           (uint64_t)(uint32_t)(st ? 0 : al.dt + 1) << 16 | (uint64_t)(uint32_t)tt.T << 32;
  pre[1 * ldc + c] = (uint64_t)tt.tot[0];
  pre[2 * ldc + c] = (uint64_t)tt.tot[2];
  pre[3 * ldc + c] = (uint64_t)tt.tot[3];
  pre[4 * ldc + c] = (uint64_t)(uint32_t)al.bq | (uint64_t)(uint32_t)al.bkv << 32;
  pre[5 * ldc + c] = (uint64_t)(uint32_t)min(al.fp.smem, (int64_t)0xffffffffLL) | (uint64_t)(uint32_t)al.fp.warps << 32;
  pre[6 * ldc + c] = (uint64_t)(uint32_t)al.fp.regs | (uint64_t)(uint32_t)al.hd << 32;
}

int launch_attn_fuse_prep(const ConfigView &cfg, const AttnResults &res, uint64_t *pre, int64_t ldc, void *stream) {
  if (cfg.n_configs == 0) return 0;
  attn_fuse_prep<<<(unsigned)((cfg.n_configs + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      cfg, res, pre, ldc);
  return (int)cudaGetLastError();
}

int launch_featurize_attention(const ConfigView &cfg, const DevSpec *specs, int spec_begin, int spec_end,
                               int n_specs, const AttnPlan &plan, const AttnResults &res, int64_t n_pairs,
                               const int64_t *cfg_idx, const int32_t *spec_idx, int32_t max_sms,
                               const FeatOut &out, int num_device_sms, void *stream, const LaunchHook &hook,
                               bool emit) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (cfg_idx == nullptr) {
    if (cfg.n_configs == 0 || plan.n_groups == 0) return 0;
    // one launch per run of groups with the same (distinct count, small-N) shape
    // work counters, then the cost-bucket counts and cursors (contiguous: api.cu attn_cross)
    cudaError_t me = cudaMemsetAsync(plan.counters, 0, (size_t)(plan.n_groups + 2 * kAttnCostBuckets) * sizeof(int), st);
    if (me != cudaSuccess) return (int)me;
    hook.on_begin("attn_prepass", st);
    attn_prepass<<<(unsigned)((cfg.n_configs + 255) / 256), 256, 0, st>>>(cfg, res, plan.min_n, plan.n_slots);
    hook.on_end(st);
    me = cudaGetLastError();
    if (me != cudaSuccess) return (int)me;
    hook.on_begin("attn_order", st);
    const int64_t n_chunks = (cfg.n_configs + 31) / 32;
    attn_order<<<(unsigned)((n_chunks + 255) / 256), 256, 0, st>>>(res, n_chunks);
    hook.on_end(st);
    me = cudaGetLastError();
    if (me != cudaSuccess) return (int)me;
    for (int y = 0; y < plan.n_groups;) {
      const int nd = plan.host_nd[y];
      const bool small = plan.host_small[y];
      int y1 = y + 1;
      while (y1 < plan.n_groups && plan.host_nd[y1] == nd && plan.host_small[y1] == small) ++y1;
      int e = small ? launch_nd<true>(nd, cfg, plan, res, num_device_sms, st, y, y1 - y, hook)
                    : launch_nd<false>(nd, cfg, plan, res, num_device_sms, st, y, y1 - y, hook);
      if (e) return e;
      y = y1;
    }
    cudaError_t le;
    if (emit) {
      const dim3 blocks((unsigned)((cfg.n_configs + 255) / 256),
                        (unsigned)((spec_end - spec_begin + kEmitSpecTile - 1) / kEmitSpecTile));
      hook.on_begin("attn_emit_cross", st);
      attn_emit_cross<<<blocks, 256, 0, st>>>(cfg, specs, spec_begin, spec_end - spec_begin, plan.spec_slot, res,
                                              out);
      hook.on_end(st);
      le = cudaGetLastError();
      if (le != cudaSuccess) return (int)le;
    }
    // planner configs (kv_chunk = -1): per pair, after the cross kernels skipped them
    const int pw = ((max_sms + kAttnSlack + 3) & ~3) + kAttnScratchWords;
    const size_t psmem = (size_t)kWarps * pw * 4;
    le = cudaFuncSetAttribute(attn_planner_cross, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem);
    if (le != cudaSuccess) return (int)le;
    const int64_t pwant = (cfg.n_configs + 32 * kWarps - 1) / (32 * kWarps);
    const int64_t pcap = (int64_t)num_device_sms * 4;
    hook.on_begin("attn_planner_cross", st);
    attn_planner_cross<<<(unsigned)(pwant < pcap ? pwant : pcap), kWarps * 32, psmem, st>>>(
        cfg, specs, spec_begin, spec_end - spec_begin, pw, out);
    hook.on_end(st);
    return (int)cudaGetLastError();
  }
  if (n_pairs == 0) return 0;
  const int words = ((max_sms + kAttnSlack + 3) & ~3) + kAttnScratchWords;  // accumulators + request scratch
  const size_t smem = (size_t)kWarps * words * 4;
  cudaError_t e = cudaFuncSetAttribute(featurize_attention_list, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return (int)e;
  int64_t want = (n_pairs + kWarps - 1) / kWarps;
  int64_t cap = (int64_t)num_device_sms * 8;
  hook.on_begin("featurize_attention_list", st);
  featurize_attention_list<<<(unsigned)(want < cap ? want : cap), kWarps * 32, smem, st>>>(
      cfg, specs, n_specs, words, n_pairs, cfg_idx, spec_idx, out);
  hook.on_end(st);
  return (int)cudaGetLastError();
}

int launch_attention_clamped(const ConfigView &cfg, const DevSpec *specs, int spec_begin, int n_specs,
                             int64_t n_pairs, const int64_t *cfg_idx, const int32_t *spec_idx, int max_sms,
                             const FeatOut &out, int num_device_sms, void *stream) {
  if (n_pairs == 0) return 0;
  const size_t per_warp = (size_t)3 * max_sms * sizeof(unsigned long long);
  const int warps = (int)std::max<size_t>(1, std::min<size_t>(8, (200 * 1024) / per_warp));
  const size_t smem = per_warp * warps;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(attn_clamped_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  const int64_t blocks = std::min<int64_t>((n_pairs + warps - 1) / warps, (int64_t)num_device_sms * 16);
  attn_clamped_kernel<<<(unsigned)blocks, 32 * warps, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
      cfg, specs, spec_begin, n_specs, n_pairs, cfg_idx, spec_idx, max_sms, out);
  return (int)cudaGetLastError();
}

}  // namespace sp
