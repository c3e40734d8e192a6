// End-to-end serving composition (PAPER §V-D):
// the Workload Generator expanded on the GPU, and the sequential-sum composer.
//
// Plan (sp_e2e_plan_create / _update): the host validates the model and the
// request traces, computes per-trace prefix offsets (O(#requests)) and uploads
// them with the requests in one copy.  Two kernels then write every config
// batch the composition needs, in the layouts include/synperf.h documents:
//   e2e_expand  one warp per step: the step's attention config (E2, E5) and
//               its ragged (qlen, kvlen) list, compacted in batch order with a
//               ballot (active requests = output_len > k);
//   e2e_tables  one thread per token-count slot: the GEMM (E4), RMSNorm and
//               SiLU&Mul (E6) configs of that M.
// Per-layer kernels are identical within a step (one config, multiplicity L),
// and every decode step with the same batch size shares its GEMM / norm /
// activation configs (slot = M-1), so only attention is per step.
//
// Compose (sp_e2e_compose): one block per (trace, spec) walks the trace's
// steps, gathers the predicted latencies of the step's invocations, adds the
// interpolated collectives (E7) and writes the per-step sum (fp32) and the
// per-trace totals and breakdown (fp64 block reduction, E8).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <new>
#include <string>
#include <vector>

#include "ctx.h"
#include "sp_internal.h"
#include "synperf.h"

using namespace sp;

namespace {

constexpr int kMaxCommPoints = 64;
constexpr int64_t kI32Max = 2147483647LL;

// ---------------------------------------------------------------- kernels

struct ExpandArgs {
  int32_t n_traces, max_batch;
  int64_t n_steps, n_slots, n_gemm;
  const int64_t *req_off;         // [R+1]
  const int32_t *in_len, *out_len;
  const int64_t *step_off;        // [R+1] first step of each trace
  const int64_t *rag_off;         // [R+1] first ragged int32 of each trace
  const int32_t *tokens;          // [R] prefill token count of each trace
  int32_t *attn_fields;           // [12][n_steps]
  int64_t *attn_roff;             // [n_steps]
  int32_t *attn_ragged;           // [n_ragged]
  int32_t *gemm_fields;           // [11][n_gemm]
  int32_t *rms_fields;            // [6][n_slots]
  int32_t *silu_fields;           // [6][n_slots]
  int32_t nh, nkv, hd, hidden, inter, vocab, qkv_n;
};

constexpr int kStepsPerWarp = 32;  // = lanes: lane j stores step j of the warp's chunk

// E2 + E5: each warp expands kStepsPerWarp consecutive steps (one binary search
// for the first step's trace, then a walk across trace boundaries).  Lanes hold
// the current trace's first 64 requests in registers; larger batches read the
// rest through L1.
__global__ void __launch_bounds__(256) e2e_expand_kernel(ExpandArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s_first = warp * kStepsPerWarp; s_first < a.n_steps; s_first += nwarps * kStepsPerWarp) {
    const int64_t s_last = min(a.n_steps, s_first + kStepsPerWarp);
    // trace of the first step: last r with step_off[r] <= s_first
    int lo = 0, hi = a.n_traces - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (__ldg(a.step_off + mid) <= s_first) lo = mid; else hi = mid - 1;
    }
    int r = lo;
    int64_t t_begin = __ldg(a.step_off + r), t_end = __ldg(a.step_off + r + 1);
    int64_t b0 = __ldg(a.req_off + r), nb = __ldg(a.req_off + r + 1) - b0;
    int32_t in0 = 0, out0 = 0, in1 = 0, out1 = 0;  // requests lane, lane + 32
    auto load_trace = [&]() {
      in0 = lane < nb ? __ldg(a.in_len + b0 + lane) : 0;
      out0 = lane < nb ? __ldg(a.out_len + b0 + lane) : 0;
      in1 = lane + 32 < nb ? __ldg(a.in_len + b0 + lane + 32) : 0;
      out1 = lane + 32 < nb ? __ldg(a.out_len + b0 + lane + 32) : 0;
    };
    load_trace();
    int32_t my_bs = 0;
    bool my_pf = false;
    int64_t my_roff = 0;
    // entries of the trace's decode steps before step k: sum_b min(out_b - 1, k - 1), which
    // grows by the decode batch of step k-1 (min(o-1, k) - min(o-1, k-1) = [o > k]); summed
    // over the requests only at the warp's first step when that step is mid-trace
    int64_t run_before = -1;
    for (int64_t s = s_first; s < s_last; ++s) {
      while (s >= t_end) {  // next trace (steps of a trace are contiguous; empty traces cannot occur)
        run_before = -1;
        ++r;
        t_begin = t_end;
        t_end = __ldg(a.step_off + r + 1);
        b0 = __ldg(a.req_off + r);
        nb = __ldg(a.req_off + r + 1) - b0;
        load_trace();
      }
      const int32_t k = (int32_t)(s - t_begin);
      int64_t roff = __ldg(a.rag_off + r);
      int32_t bs;
      if (k == 0) {  // prefill: every request, qlen = kvlen = input_len, batch order
        for (int64_t b = lane; b < nb; b += 32) {
          const int32_t q = b < 32 ? in0 : (b < 64 ? in1 : __ldg(a.in_len + b0 + b));
          *reinterpret_cast<int2 *>(a.attn_ragged + roff + 2 * b) = make_int2(q, q);
        }
        bs = (int32_t)nb;
        run_before = 0;  // step 1: no decode entries before it
      } else {
        // entries before this step: nb (prefill) + sum_b min(out_b - 1, k - 1) (decode steps 1..k-1)
        int64_t before = run_before;
        if (before < 0) {
          before = 0;
          for (int64_t b = lane; b < nb; b += 32) {
            const int32_t o = b < 32 ? out0 : (b < 64 ? out1 : __ldg(a.out_len + b0 + b));
            before += min(o - 1, k - 1);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) before += __shfl_xor_sync(0xffffffffu, before, o);
        }
        roff += 2 * (nb + before);
        int32_t pos = 0;
        for (int64_t b = 0; b < nb; b += 32) {
          const int64_t bi = b + lane;
          const bool in = bi < nb;
          const int32_t o = !in ? 0 : (bi < 32 ? out0 : (bi < 64 ? out1 : __ldg(a.out_len + b0 + bi)));
          const bool act = in && o > k;
          const unsigned m = __ballot_sync(0xffffffffu, act);
          if (act) {
            const int32_t q = bi < 32 ? in0 : (bi < 64 ? in1 : __ldg(a.in_len + b0 + bi));
            const int32_t p = pos + __popc(m & ((1u << lane) - 1u));
            *reinterpret_cast<int2 *>(a.attn_ragged + roff + 2 * p) = make_int2(1, q + k);
          }
          pos += __popc(m);
        }
        bs = pos;
        run_before = before + pos;
      }
      if (lane == (int)(s - s_first)) {  // lane j keeps step s_first + j's fields for one coalesced store
        my_bs = bs;
        my_pf = k == 0;
        my_roff = roff;
      }
    }
    // the fields and ragged offsets of the warp's steps: row f, columns s_first..s_last-1
    const int64_t s = s_first + lane;
    if (s < s_last) {
      const int32_t bs = my_bs;
      const bool pf = my_pf;
      int32_t v[SP_NFIELDS_ATTENTION] = {
          bs,                                                   // BS
          a.nh,                                                 // NH
          a.nkv,                                                // NKV
          a.hd,                                                 // HD
          pf ? 128 : 16,                                        // BQ
          64,                                                   // BKV
          pf ? 0 : ((int64_t)bs * a.nkv < 128 ? 1024 : 0),      // KV_CHUNK
          pf ? 1 : 0,                                           // CAUSAL
          4,                                                    // WARPS
          pf ? 168 : 64,                                        // REGS
          0,                                                    // SMEM (default footprint)
          SP_BF16};                                             // DTYPE
#pragma unroll
      for (int f = 0; f < SP_NFIELDS_ATTENTION; ++f) a.attn_fields[(int64_t)f * a.n_steps + s] = v[f];
      a.attn_roff[s] = my_roff;
    }
  }
}

__device__ __forceinline__ void put_gemm(const ExpandArgs &a, int64_t col, int32_t M, int32_t N, int32_t K) {
  // E4: tile by token count
  int32_t tm, tn, stages;
  if (M <= 64) { tm = 64; tn = 128; stages = 4; }
  else if (M <= 256) { tm = 128; tn = 128; stages = 4; }
  else { tm = 128; tn = 256; stages = 3; }
  const int32_t area = tm * tn;
  const int32_t warps = area <= 8192 ? 4 : 8;
  const int32_t regs = area <= 8192 ? 128 : (area <= 16384 ? 168 : 232);
  const int32_t v[SP_NFIELDS_GEMM] = {M, N, K, tm, tn, 64, stages, warps, regs, 0, SP_BF16};
#pragma unroll
  for (int f = 0; f < SP_NFIELDS_GEMM; ++f) a.gemm_fields[(int64_t)f * a.n_gemm + col] = v[f];
}

__device__ __forceinline__ void put_row(int32_t *fields, int64_t ld, int64_t col, int32_t seq, int32_t dim) {
  const int32_t warps = max(1, min(32, (dim + 255) / 256));  // E6
  const int32_t v[SP_NFIELDS_RMSNORM] = {seq, dim, warps, 32, 0, SP_BF16};
#pragma unroll
  for (int f = 0; f < SP_NFIELDS_RMSNORM; ++f) fields[(int64_t)f * ld + col] = v[f];
}

// E3/E4/E6: thread per token-count slot.
__global__ void __launch_bounds__(256) e2e_tables_kernel(ExpandArgs a) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < a.n_slots;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t M = j < a.max_batch ? (int32_t)(j + 1) : __ldg(a.tokens + (j - a.max_batch));
    put_gemm(a, 0 * a.n_slots + j, M, a.qkv_n, a.hidden);             // QKV
    put_gemm(a, 1 * a.n_slots + j, M, a.hidden, a.nh * a.hd);         // O proj
    put_gemm(a, 2 * a.n_slots + j, M, 2 * a.inter, a.hidden);         // GateUp
    put_gemm(a, 3 * a.n_slots + j, M, a.hidden, a.inter);             // Down
    if (j < a.max_batch) put_gemm(a, 4 * a.n_slots + j, M, a.vocab, a.hidden);  // LM head (rows = seqs)
    put_row(a.rms_fields, a.n_slots, j, M, a.hidden);
    put_row(a.silu_fields, a.n_slots, j, M, a.inter);
  }
}

struct ComposeArgs {
  int32_t n_traces, max_batch, n_layers, tp, pp, hidden;
  int64_t n_steps, n_slots, n_gemm;
  int32_t spec_begin;
  const int64_t *req_off, *step_off;
  const int32_t *tokens;
  const int32_t *attn_bs;  // attention field row BS [n_steps]
  const float *lat_gemm, *lat_attn, *lat_rms, *lat_silu;
  const double *comm;      // [P] ln(bytes), then [n_specs][P] allreduce, [n_specs][P] sendrecv
  int32_t comm_points, comm_specs;
  float *step_us;
  double *trace_us, *trace_cat;
};

// E7: linear in ln(bytes) between calibration points, flat outside.
__device__ __forceinline__ double interp(const double *lx, const double *ly, int P, double x) {
  if (x <= lx[0]) return ly[0];
  if (x >= lx[P - 1]) return ly[P - 1];
  int i = 0;
  while (i + 2 < P && lx[i + 1] <= x) ++i;
  const double t = (x - lx[i]) / (lx[i + 1] - lx[i]);
  return ly[i] + t * (ly[i + 1] - ly[i]);
}

constexpr int kComposeThreads = 256;

__global__ void __launch_bounds__(kComposeThreads) e2e_compose_kernel(ComposeArgs a) {
  const int r = blockIdx.x;
  const int gi = blockIdx.y;
  const int g = a.spec_begin + gi;
  const int64_t s0 = a.step_off[r], ns = a.step_off[r + 1] - s0;
  const int32_t nreq = (int32_t)(a.req_off[r + 1] - a.req_off[r]);
  const float *lg = a.lat_gemm + (int64_t)gi * a.n_gemm;
  const float *lr = a.lat_rms + (int64_t)gi * a.n_slots;
  const float *lsi = a.lat_silu + (int64_t)gi * a.n_slots;
  const float *la = a.lat_attn + (int64_t)gi * a.n_steps;
  const double L = (double)a.n_layers;
  const bool comm = a.comm != nullptr && (a.tp > 1 || a.pp > 1);
  const int P = a.comm_points;
  const double *lx = a.comm;
  const double *ar = comm ? a.comm + P + (int64_t)g * P : nullptr;
  const double *sr = comm ? a.comm + P + (int64_t)a.comm_specs * P + (int64_t)g * P : nullptr;
  double acc[SP_E2E_NCAT] = {0, 0, 0, 0, 0};
  for (int64_t k = threadIdx.x; k < ns; k += kComposeThreads) {
    const int64_t s = s0 + k;
    const int32_t seqs = k == 0 ? nreq : __ldg(a.attn_bs + s);
    const int64_t slot = k == 0 ? (int64_t)a.max_batch + r : (int64_t)seqs - 1;
    const double qkv = lg[0 * a.n_slots + slot], o = lg[1 * a.n_slots + slot];
    const double gu = lg[2 * a.n_slots + slot], dn = lg[3 * a.n_slots + slot];
    const double lm = lg[4 * a.n_slots + (seqs - 1)];
    const double rms = lr[slot], silu = lsi[slot], attn = la[s];
    double cm = 0.0;
    if (comm) {
      const int64_t M = slot < a.max_batch ? slot + 1 : (int64_t)__ldg(a.tokens + (slot - a.max_batch));
      const double x = log((double)M * (double)a.hidden * 2.0);  // E7: M*hidden*bf16
      if (a.tp > 1) cm += 2.0 * L * interp(lx, ar, P, x);
      if (a.pp > 1) cm += (double)(a.pp - 1) * interp(lx, sr, P, x);
    }
    const double cg = L * (qkv + o + gu + dn) + lm;
    const double ca = L * attn;
    const double cr = (2.0 * L + 1.0) * rms;
    const double cs = L * silu;
    const double step = cg + ca + cr + cs + cm;
    if (a.step_us) a.step_us[(int64_t)gi * a.n_steps + s] = (float)step;
    acc[0] += cg;
    acc[1] += ca;
    acc[2] += cr;
    acc[3] += cs;
    acc[4] += cm;
  }
  // block reduction: warp shuffles, then the 8 warp partials
  __shared__ double part[kComposeThreads / 32][SP_E2E_NCAT];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < SP_E2E_NCAT; ++c) {
    double v = acc[c];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) part[w][c] = v;
  }
  __syncthreads();
  if (threadIdx.x < SP_E2E_NCAT) {
    double v = 0.0;
    for (int i = 0; i < kComposeThreads / 32; ++i) v += part[i][threadIdx.x];
    if (a.trace_cat) a.trace_cat[((int64_t)gi * a.n_traces + r) * SP_E2E_NCAT + threadIdx.x] = v;
    part[0][threadIdx.x] = v;  // safe: every read of part[0][c] by thread c happened above
  }
  __syncthreads();
  if (threadIdx.x == 0 && a.trace_us) {
    double t = 0.0;
    for (int c = 0; c < SP_E2E_NCAT; ++c) t += part[0][c];
    a.trace_us[(int64_t)gi * a.n_traces + r] = t;
  }
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

// ---------------------------------------------------------------- handles

struct sp_comm_model {
  sp_ctx *ctx = nullptr;
  int32_t n_specs = 0, n_points = 0;
  DevBuf dev;  // [P] ln(bytes), [n_specs][P] allreduce, [n_specs][P] sendrecv (fp64)
};

struct sp_e2e_plan {
  sp_ctx *ctx = nullptr;
  sp_serving_model m{};
  sp_e2e_info info{};
  void *dev = nullptr;
  size_t dev_cap = 0;
  void *host = nullptr;  // pinned staging of the uploads
  size_t host_cap = 0;
  cudaEvent_t staged = nullptr;  // the last upload has read `host`
  // views into dev
  int64_t *req_off = nullptr, *step_off = nullptr, *rag_off = nullptr;
  int32_t *in_len = nullptr, *out_len = nullptr, *tokens = nullptr;
  int32_t *attn_fields = nullptr, *attn_ragged = nullptr, *gemm_fields = nullptr;
  int32_t *rms_fields = nullptr, *silu_fields = nullptr;
  int64_t *attn_roff = nullptr;
  ExpandArgs args{};
  ~sp_e2e_plan() {
    if (dev) cudaFree(dev);
    if (host) cudaFreeHost(host);
    if (staged) cudaEventDestroy(staged);
  }
};

static sp_status check_model(sp_ctx *ctx, const sp_serving_model *m) {
  if (!m) return fail(ctx, SP_E_ARG, "e2e: model is NULL");
  if (m->n_layers < 1 || m->hidden < 1 || m->n_heads < 1 || m->n_kv_heads < 1 || m->head_dim < 1 ||
      m->intermediate < 1 || m->vocab < 1 || m->tp < 1 || m->pp < 1)
    return fail(ctx, SP_E_ARG, "e2e: model dimensions and tp/pp must be >= 1");
  if (m->n_heads % m->tp || m->n_kv_heads % m->tp || m->intermediate % m->tp || m->vocab % m->tp)
    return fail(ctx, SP_E_ARG, "e2e: heads, kv heads, intermediate and vocab must be divisible by tp");
  if (m->n_layers % m->pp) return fail(ctx, SP_E_ARG, "e2e: n_layers must be divisible by pp");
  if ((m->n_heads / m->tp) % (m->n_kv_heads / m->tp))
    return fail(ctx, SP_E_ARG, "e2e: heads per rank must be divisible by kv heads per rank");
  if (m->dtype != SP_BF16) return fail(ctx, SP_E_ARG, "e2e: only SP_BF16 serving models are supported (E9)");
  const int64_t qkv = (int64_t)(m->n_heads + 2 * m->n_kv_heads) / m->tp * m->head_dim;
  if (qkv > kI32Max || 2LL * m->intermediate > kI32Max || (int64_t)m->n_heads * m->head_dim > kI32Max)
    return fail(ctx, SP_E_ARG, "e2e: a GEMM dimension exceeds int32");
  return SP_OK;
}

static sp_status plan_launch(sp_e2e_plan *p, void *stream);

static sp_status plan_fill(sp_e2e_plan *p, int32_t R, const int64_t *req_off, const int32_t *in_len,
                           const int32_t *out_len, void *stream) {
  sp_ctx *ctx = p->ctx;
  if (R < 1 || !req_off || !in_len || !out_len) return fail(ctx, SP_E_ARG, "e2e plan: need >= 1 trace and host arrays");
  if (req_off[0] != 0) return fail(ctx, SP_E_ARG, "e2e plan: req_off[0] must be 0");
  const sp_serving_model &m = p->m;
  // host: validation and per-trace prefixes, O(#requests)
  std::vector<int64_t> step_off(R + 1), rag_off(R + 1);
  std::vector<int32_t> tokens(R);
  int32_t bmax = 0;
  step_off[0] = rag_off[0] = 0;
  for (int32_t r = 0; r < R; ++r) {
    const int64_t a = req_off[r], b = req_off[r + 1];
    if (b <= a) return fail(ctx, SP_E_DATA, "e2e plan: trace " + std::to_string(r) + " has no requests");
    if (b - a > kI32Max) return fail(ctx, SP_E_DATA, "e2e plan: batch too large");
    int64_t tok = 0, smax = 0, sout = 0;
    for (int64_t i = a; i < b; ++i) {
      if (in_len[i] < 1 || out_len[i] < 1)
        return fail(ctx, SP_E_DATA, "e2e plan: input_len and output_len must be >= 1");
      if ((int64_t)in_len[i] + out_len[i] - 1 > kI32Max)
        return fail(ctx, SP_E_DATA, "e2e plan: kvlen exceeds int32");
      tok += in_len[i];
      smax = std::max<int64_t>(smax, out_len[i]);
      sout += out_len[i];
    }
    if (tok > kI32Max) return fail(ctx, SP_E_DATA, "e2e plan: prefill token count exceeds int32");
    if (tok * (m.n_heads / m.n_kv_heads) > kI32Max)
      return fail(ctx, SP_E_DATA, "e2e plan: packed query rows exceed int32");
    tokens[r] = (int32_t)tok;
    bmax = std::max<int32_t>(bmax, (int32_t)(b - a));
    step_off[r + 1] = step_off[r] + smax;
    rag_off[r + 1] = rag_off[r] + 2 * sout;
  }
  const int64_t nreq = req_off[R];
  sp_e2e_info inf{};
  inf.n_traces = R;
  inf.max_batch = bmax;
  inf.n_requests = nreq;
  inf.n_steps = step_off[R];
  inf.n_ragged = rag_off[R];
  inf.n_slots = (int64_t)bmax + R;
  inf.n_configs[SP_GEMM] = 4 * inf.n_slots + bmax;
  inf.n_configs[SP_ATTENTION] = inf.n_steps;
  inf.n_configs[SP_RMSNORM] = inf.n_slots;
  inf.n_configs[SP_SILU_MUL] = inf.n_slots;
  inf.n_configs[SP_FUSED_MOE] = 0;

  // device layout (256-byte aligned sub-buffers)
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += align256(bytes); return o; };
  const size_t o_req = take(8 * (R + 1)), o_step = take(8 * (R + 1)), o_rag = take(8 * (R + 1));
  const size_t o_in = take(4 * nreq), o_out = take(4 * nreq), o_tok = take(4 * R);
  const size_t upload = off;  // everything above comes from the host in one copy
  const size_t o_af = take(4 * (size_t)SP_NFIELDS_ATTENTION * inf.n_steps);
  const size_t o_ar = take(8 * (size_t)inf.n_steps);
  const size_t o_ag = take(4 * (size_t)inf.n_ragged);
  const size_t o_gf = take(4 * (size_t)SP_NFIELDS_GEMM * inf.n_configs[SP_GEMM]);
  const size_t o_rf = take(4 * (size_t)SP_NFIELDS_RMSNORM * inf.n_slots);
  const size_t o_sf = take(4 * (size_t)SP_NFIELDS_SILU_MUL * inf.n_slots);
  const size_t total = off;

  cudaSetDevice(ctx->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (!p->staged && (e = cudaEventCreateWithFlags(&p->staged, cudaEventDisableTiming)) != cudaSuccess)
    return cuda_fail(ctx, e, "e2e plan: event");
  if (total > p->dev_cap) {
    if (p->dev) {
      cudaStreamSynchronize(st);  // earlier work on this stream may still read the old plan
      cudaFree(p->dev);
    }
    p->dev = nullptr;
    p->dev_cap = 0;
    if ((e = cudaMalloc(&p->dev, total)) != cudaSuccess) { p->dev = nullptr; return cuda_fail(ctx, e, "e2e plan: device buffers"); }
    p->dev_cap = total;
  }
  if (upload > p->host_cap) {
    cudaEventSynchronize(p->staged);
    if (p->host) cudaFreeHost(p->host);
    p->host = nullptr;
    p->host_cap = 0;
    if ((e = cudaMallocHost(&p->host, upload)) != cudaSuccess) { p->host = nullptr; return cuda_fail(ctx, e, "e2e plan: pinned staging"); }
    p->host_cap = upload;
  } else {
    cudaEventSynchronize(p->staged);  // the previous upload has finished reading the staging buffer
  }
  char *h = static_cast<char *>(p->host);
  memcpy(h + o_req, req_off, 8 * (R + 1));
  memcpy(h + o_step, step_off.data(), 8 * (R + 1));
  memcpy(h + o_rag, rag_off.data(), 8 * (R + 1));
  memcpy(h + o_in, in_len, 4 * nreq);
  memcpy(h + o_out, out_len, 4 * nreq);
  memcpy(h + o_tok, tokens.data(), 4 * R);
  if ((e = cudaMemcpyAsync(p->dev, h, upload, cudaMemcpyHostToDevice, st)) != cudaSuccess)
    return cuda_fail(ctx, e, "e2e plan: upload");
  cudaEventRecord(p->staged, st);

  char *d = static_cast<char *>(p->dev);
  p->req_off = (int64_t *)(d + o_req);
  p->step_off = (int64_t *)(d + o_step);
  p->rag_off = (int64_t *)(d + o_rag);
  p->in_len = (int32_t *)(d + o_in);
  p->out_len = (int32_t *)(d + o_out);
  p->tokens = (int32_t *)(d + o_tok);
  p->attn_fields = (int32_t *)(d + o_af);
  p->attn_roff = (int64_t *)(d + o_ar);
  p->attn_ragged = (int32_t *)(d + o_ag);
  p->gemm_fields = (int32_t *)(d + o_gf);
  p->rms_fields = (int32_t *)(d + o_rf);
  p->silu_fields = (int32_t *)(d + o_sf);
  p->info = inf;

  ExpandArgs a{};
  a.n_traces = R;
  a.max_batch = bmax;
  a.n_steps = inf.n_steps;
  a.n_slots = inf.n_slots;
  a.n_gemm = inf.n_configs[SP_GEMM];
  a.req_off = p->req_off;
  a.in_len = p->in_len;
  a.out_len = p->out_len;
  a.step_off = p->step_off;
  a.rag_off = p->rag_off;
  a.tokens = p->tokens;
  a.attn_fields = p->attn_fields;
  a.attn_roff = p->attn_roff;
  a.attn_ragged = p->attn_ragged;
  a.gemm_fields = p->gemm_fields;
  a.rms_fields = p->rms_fields;
  a.silu_fields = p->silu_fields;
  a.nh = m.n_heads / m.tp;
  a.nkv = m.n_kv_heads / m.tp;
  a.hd = m.head_dim;
  a.hidden = m.hidden;
  a.inter = m.intermediate / m.tp;
  a.vocab = m.vocab / m.tp;
  a.qkv_n = (m.n_heads + 2 * m.n_kv_heads) / m.tp * m.head_dim;
  p->args = a;
  return plan_launch(p, stream);
}

static sp_status plan_launch(sp_e2e_plan *p, void *stream) {
  sp_ctx *ctx = p->ctx;
  const sp_e2e_info &inf = p->info;
  const ExpandArgs &a = p->args;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  cudaSetDevice(ctx->device);
  const LaunchHook hk = ctx->hook();
  const int64_t warps_needed = (inf.n_steps + kStepsPerWarp - 1) / kStepsPerWarp;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((warps_needed + 7) / 8, (int64_t)ctx->num_sms * 16));
  hk.on_begin("e2e_expand", stream);
  e2e_expand_kernel<<<blocks, 256, 0, st>>>(a);
  hk.on_end(stream);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(ctx, e, "e2e plan: expand launch");
  const int tblocks = (int)std::max<int64_t>(1, std::min<int64_t>((inf.n_slots + 255) / 256, 1024));
  hk.on_begin("e2e_tables", stream);
  e2e_tables_kernel<<<tblocks, 256, 0, st>>>(a);
  hk.on_end(stream);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(ctx, e, "e2e plan: tables launch");
  return SP_OK;
}

extern "C" sp_status sp_e2e_plan_create(sp_ctx *ctx, const sp_serving_model *model, int32_t n_traces,
                                        const int64_t *req_off, const int32_t *input_len,
                                        const int32_t *output_len, void *stream, sp_e2e_plan **out) {
  if (!ctx) return fail(nullptr, SP_E_ARG, "sp_e2e_plan_create: ctx is NULL");
  if (!out) return fail(ctx, SP_E_ARG, "sp_e2e_plan_create: out is NULL");
  *out = nullptr;
  sp_status s = check_model(ctx, model);
  if (s != SP_OK) return s;
  ctx->err.clear();
  sp_e2e_plan *p = new (std::nothrow) sp_e2e_plan;
  if (!p) return fail(ctx, SP_E_INTERNAL, "sp_e2e_plan_create: out of host memory");
  p->ctx = ctx;
  p->m = *model;
  s = plan_fill(p, n_traces, req_off, input_len, output_len, stream);
  if (s != SP_OK) {
    cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream));
    delete p;
    return s;
  }
  *out = p;
  return SP_OK;
}

extern "C" sp_status sp_e2e_plan_update(sp_e2e_plan *plan, int32_t n_traces, const int64_t *req_off,
                                        const int32_t *input_len, const int32_t *output_len, void *stream) {
  if (!plan) return fail(nullptr, SP_E_ARG, "sp_e2e_plan_update: plan is NULL");
  plan->ctx->err.clear();
  return plan_fill(plan, n_traces, req_off, input_len, output_len, stream);
}

extern "C" sp_status sp_e2e_plan_expand(sp_e2e_plan *plan, void *stream) {
  if (!plan) return fail(nullptr, SP_E_ARG, "sp_e2e_plan_expand: plan is NULL");
  plan->ctx->err.clear();
  return plan_launch(plan, stream);
}

extern "C" void sp_free_e2e_plan(sp_e2e_plan *plan) { delete plan; }

extern "C" sp_status sp_e2e_plan_info(const sp_e2e_plan *plan, sp_e2e_info *out) {
  if (!plan || !out) return fail(plan ? plan->ctx : nullptr, SP_E_ARG, "sp_e2e_plan_info: NULL argument");
  *out = plan->info;
  return SP_OK;
}

extern "C" sp_status sp_e2e_plan_batch(const sp_e2e_plan *plan, int32_t family, sp_config_batch *out) {
  if (!plan || !out) return fail(plan ? plan->ctx : nullptr, SP_E_ARG, "sp_e2e_plan_batch: NULL argument");
  sp_config_batch b{};
  b.family = family;
  switch (family) {
    case SP_ATTENTION:
      b.n_fields = SP_NFIELDS_ATTENTION;
      b.fields = plan->attn_fields;
      b.ragged = plan->attn_ragged;
      b.ragged_off = plan->attn_roff;
      b.n_ragged = plan->info.n_ragged;
      break;
    case SP_GEMM: b.n_fields = SP_NFIELDS_GEMM; b.fields = plan->gemm_fields; break;
    case SP_RMSNORM: b.n_fields = SP_NFIELDS_RMSNORM; b.fields = plan->rms_fields; break;
    case SP_SILU_MUL: b.n_fields = SP_NFIELDS_SILU_MUL; b.fields = plan->silu_fields; break;
    default: return fail(plan->ctx, SP_E_ARG, "sp_e2e_plan_batch: the serving template has no such family");
  }
  b.n_configs = plan->info.n_configs[family];
  b.field_ld = b.n_configs;
  *out = b;
  return SP_OK;
}

extern "C" sp_status sp_load_comm_model(sp_ctx *ctx, const sp_comm_desc *d, sp_comm_model **out) {
  if (!ctx) return fail(nullptr, SP_E_ARG, "sp_load_comm_model: ctx is NULL");
  if (!d || !out) return fail(ctx, SP_E_ARG, "sp_load_comm_model: NULL argument");
  *out = nullptr;
  if (d->n_specs < 1 || d->n_points < 1 || d->n_points > kMaxCommPoints || !d->bytes || !d->allreduce_us ||
      !d->sendrecv_us)
    return fail(ctx, SP_E_ARG, "sp_load_comm_model: need n_specs >= 1, 1 <= n_points <= 64 and three tables");
  const int P = d->n_points;
  for (int i = 0; i < P; ++i) {
    if (!(d->bytes[i] > 0) || !std::isfinite(d->bytes[i]) || (i > 0 && !(d->bytes[i] > d->bytes[i - 1])))
      return fail(ctx, SP_E_DATA, "sp_load_comm_model: bytes must be finite, > 0 and strictly increasing");
  }
  for (const double *t : {d->allreduce_us, d->sendrecv_us})
    for (int64_t g = 0; g < d->n_specs; ++g)
      for (int i = 0; i < P; ++i) {
        const double v = t[g * P + i];
        if (!std::isfinite(v) || v < 0 || (i > 0 && v < t[g * P + i - 1]))
          return fail(ctx, SP_E_DATA, "sp_load_comm_model: latencies must be finite, >= 0 and non-decreasing (S:546)");
      }
  std::vector<double> img((size_t)P * (1 + 2 * (size_t)d->n_specs));
  for (int i = 0; i < P; ++i) img[i] = std::log(d->bytes[i]);
  memcpy(img.data() + P, d->allreduce_us, sizeof(double) * P * (size_t)d->n_specs);
  memcpy(img.data() + P + (size_t)P * d->n_specs, d->sendrecv_us, sizeof(double) * P * (size_t)d->n_specs);
  sp_comm_model *c = new (std::nothrow) sp_comm_model;
  if (!c) return fail(ctx, SP_E_INTERNAL, "sp_load_comm_model: out of host memory");
  cudaSetDevice(ctx->device);
  cudaError_t e = c->dev.alloc_copy(img.data(), img.size() * sizeof(double));
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(ctx, e, "sp_load_comm_model: upload");
  }
  c->ctx = ctx;
  c->n_specs = d->n_specs;
  c->n_points = P;
  *out = c;
  return SP_OK;
}

extern "C" void sp_free_comm_model(sp_comm_model *comm) { delete comm; }

extern "C" sp_status sp_e2e_compose(sp_ctx *ctx, const sp_e2e_plan *plan, int32_t spec_begin, int32_t spec_end,
                                    const sp_comm_model *comm, const sp_e2e_latencies *lat, float *step_us,
                                    double *trace_us, double *trace_cat, void *stream) {
  if (!ctx) return fail(nullptr, SP_E_ARG, "sp_e2e_compose: ctx is NULL");
  if (!plan || !lat) return fail(ctx, SP_E_ARG, "sp_e2e_compose: NULL argument");
  if (spec_begin < 0 || spec_end < spec_begin) return fail(ctx, SP_E_ARG, "sp_e2e_compose: bad spec range");
  if (!lat->gemm || !lat->attention || !lat->rmsnorm || !lat->silu_mul)
    return fail(ctx, SP_E_ARG, "sp_e2e_compose: every family's latencies are needed");
  const sp_serving_model &m = plan->m;
  const bool need_comm = m.tp > 1 || m.pp > 1;
  if (need_comm && (!comm || comm->n_specs < spec_end))
    return fail(ctx, SP_E_ARG, "sp_e2e_compose: tp/pp > 1 needs a comm model covering the spec range");
  const int G = spec_end - spec_begin;
  if (G == 0) return SP_OK;
  if (G > 65535) return fail(ctx, SP_E_UNSUPPORTED, "sp_e2e_compose: at most 65535 specs per call");
  ctx->err.clear();
  cudaSetDevice(ctx->device);
  ComposeArgs a{};
  a.n_traces = plan->info.n_traces;
  a.max_batch = plan->info.max_batch;
  a.n_layers = m.n_layers;
  a.tp = m.tp;
  a.pp = m.pp;
  a.hidden = m.hidden;
  a.n_steps = plan->info.n_steps;
  a.n_slots = plan->info.n_slots;
  a.n_gemm = plan->info.n_configs[SP_GEMM];
  a.spec_begin = spec_begin;
  a.req_off = plan->req_off;
  a.step_off = plan->step_off;
  a.tokens = plan->tokens;
  a.attn_bs = plan->attn_fields;  // field row 0 = BS
  a.lat_gemm = lat->gemm;
  a.lat_attn = lat->attention;
  a.lat_rms = lat->rmsnorm;
  a.lat_silu = lat->silu_mul;
  a.comm = need_comm ? (const double *)comm->dev.p : nullptr;
  a.comm_points = need_comm ? comm->n_points : 0;
  a.comm_specs = need_comm ? comm->n_specs : 0;
  a.step_us = step_us;
  a.trace_us = trace_us;
  a.trace_cat = trace_cat;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const LaunchHook hk = ctx->hook();
  hk.on_begin("e2e_compose", stream);
  e2e_compose_kernel<<<dim3(a.n_traces, G), kComposeThreads, 0, st>>>(a);
  hk.on_end(stream);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "sp_e2e_compose: launch");
  return SP_OK;
}
