// sp_predict_host: the host-buffer end-to-end call (SPEC S:407 predict_latency,
// batched over a CROSS range of specs).  HOST configs in, HOST fp32 latencies
// out, spec-major [g - spec_begin][c].  Everything between is the device path:
// the configs go up in slices over three streams -- the H2D of slice i + 1 and
// the D2H of slice i - 1 overlap the kernels of slice i (sp_featurize_predict:
// the fused kernel for the uniform families, featurize + predict otherwise).
//
//  * Config slices (the default): slice weights, e.g. (1, 2, 3, 2) for
//    attention, whose kernels outlast the copies (a short first copy-in and
//    last copy-out), and 8 equal slices for the copy-bound uniform families.
//    Each slice copies only its own range of the ragged data (attention
//    (qlen, kvlen) pairs, MoE histograms), planned from the host offsets at
//    the slice boundaries.  The plan is exact when the ragged data is laid out
//    config by config (as any sequential builder does); a device guard checks
//    every config of the slice (ragged_guard_kernel) and, where the plan
//    missed its data, zeroes its length field in the device copy (so it costs
//    one cheap SP_PAIR_E_DIM pair instead of reading stale data) and raises a
//    flag, and the call is then redone with one whole copy of the ragged data.
//  * Spec slices (a wide spec axis, G >= 64 and >= 4 slices, e.g. config 5):
//    the configs go up once, then spec ranges are predicted while the previous
//    range's latencies -- a contiguous run of the spec-major output -- go down.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "ctx.h"

using namespace sp;

namespace {

// Device check of one config slice's ragged copy plan [lo, hi) (see above).
__global__ void ragged_guard_kernel(int32_t *len_row, const int64_t *roff, int64_t c0, int64_t c1, int64_t lo,
                                    int64_t hi, int mult, int32_t *flag) {
  const int64_t c = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= c1) return;
  const int64_t off = roff[c];
  if (off < 0) return;
  const int64_t end = off + (int64_t)mult * len_row[c];
  if (off < lo || end > hi) {
    len_row[c] = 0;
    atomicOr(flag, 1);
  }
}

// (field row holding a config's ragged length, elements per unit of it)
void ragged_rule(int fam, int &row, int &mult) {
  if (fam == SP_ATTENTION) { row = 0; mult = 2; }  // batch size; (qlen, kvlen) per request
  else { row = 1; mult = 1; }                      // fused MoE: E; one count per expert
}

// Per-slice ragged ranges from the host offsets at the slice boundaries (the
// first / last config with data within 64 of each boundary).  Empty if no
// cheap plan exists (then the ragged data is copied whole).
std::vector<std::pair<int64_t, int64_t>> ragged_plan(const sp_config_batch &h, const std::vector<int64_t> &b) {
  std::vector<std::pair<int64_t, int64_t>> out;
  if (!h.ragged_off || b.size() < 3) return out;
  int row, mult;
  ragged_rule(h.family, row, mult);
  int64_t prev = 0;
  for (size_t i = 0; i + 1 < b.size(); ++i) {
    const int64_t a = b[i], e = b[i + 1];
    int64_t ia = -1, ib = -1;
    for (int64_t k = a; k < std::min(e, a + 64); ++k)
      if (h.ragged_off[k] >= 0) { ia = k; break; }
    for (int64_t k = e - 1; k >= std::max(a, e - 64); --k)
      if (h.ragged_off[k] >= 0) { ib = k; break; }
    if (ia < 0 || ib < 0) return {};  // long runs without ragged data (balanced MoE): copy whole
    const int64_t lo = h.ragged_off[ia], hi = h.ragged_off[ib] + (int64_t)mult * h.fields[(int64_t)row * h.field_ld + ib];
    if (lo < prev || hi < lo || hi > h.n_ragged) return {};
    out.emplace_back(lo, hi);
    prev = hi;
  }
  return out;
}

cudaEvent_t host_event(sp_ctx *ctx, size_t i) {
  while (ctx->h_events.size() <= i) {
    cudaEvent_t e = nullptr;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    ctx->h_events.push_back(e);
  }
  return ctx->h_events[i];
}

#define HCHECK(x, what)                                  \
  do {                                                   \
    cudaError_t e_ = (x);                                \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, what); \
  } while (0)

sp_status run(sp_ctx *ctx, const sp_config_batch *h, const sp_specs *specs, int32_t g0, int32_t g1,
              const sp_model *model, float *host_latency, const float *weights, int32_t n_slices, cudaStream_t comp,
              bool plan, bool *plan_missed) {
  const int64_t C = h->n_configs, G = g1 - g0, nf = h->n_fields;
  const int fam = h->family;
  const bool rag = h->ragged_off != nullptr && h->n_ragged > 0;
  if (!ctx->h_h2d) HCHECK(cudaStreamCreateWithFlags(&ctx->h_h2d, cudaStreamNonBlocking), "sp_predict_host: stream");
  if (!ctx->h_d2h) HCHECK(cudaStreamCreateWithFlags(&ctx->h_d2h, cudaStreamNonBlocking), "sp_predict_host: stream");
  cudaStream_t s_h2d = ctx->h_h2d, s_d2h = ctx->h_d2h;
  size_t ev = 0;
  auto next_event = [&]() { return host_event(ctx, ev++); };

  // staging buffers: configs [nf][C], offsets, ragged data, guard flag
  HCHECK(ctx->h_fields.need((size_t)std::max<int64_t>(nf * C, 1) * 4), "sp_predict_host: staging");
  if (h->ragged_off) HCHECK(ctx->h_roff.need((size_t)std::max<int64_t>(C, 1) * 8), "sp_predict_host: staging");
  if (h->ragged) HCHECK(ctx->h_ragged.need((size_t)std::max<int64_t>(h->n_ragged, 1) * 4), "sp_predict_host: staging");
  HCHECK(ctx->h_flag.need(16), "sp_predict_host: staging");
  int32_t *d_fields = (int32_t *)ctx->h_fields.p, *d_ragged = (int32_t *)ctx->h_ragged.p;
  int64_t *d_roff = (int64_t *)ctx->h_roff.p;
  int32_t *d_flag = (int32_t *)ctx->h_flag.p;

  // the copies must not overwrite staging a previous call on `comp` still reads
  cudaEvent_t e0 = next_event();
  if (!e0) return fail(ctx, SP_E_INTERNAL, "sp_predict_host: event");
  HCHECK(cudaEventRecord(e0, comp), "sp_predict_host: event");
  HCHECK(cudaStreamWaitEvent(s_h2d, e0, 0), "sp_predict_host: event");
  HCHECK(cudaStreamWaitEvent(s_d2h, e0, 0), "sp_predict_host: event");

  const int64_t rec = 11 * 8 + 12 * 4 + 1;  // record bytes per pair
  auto features = [&](int64_t n, sp_features &f) -> sp_status {
    const int64_t ld = (std::max<int64_t>(n, 1) + 31) & ~(int64_t)31;
    HCHECK(ctx->h_feats.need((size_t)(ld * rec)), "sp_predict_host: feature scratch");
    char *b = (char *)ctx->h_feats.p;
    f.family = fam;
    f.n_pairs = n;
    f.ld = ld;
    f.ints = (int64_t *)b;
    f.flts = (float *)(b + ld * 88);
    f.status = (uint8_t *)(b + ld * 136);
    return SP_OK;
  };

  if (G >= 64 && G >= 4 * std::max(n_slices, 1)) {
    // ---- spec slices: configs up once, then spec ranges [ga, gb)
    const int64_t k = std::max<int64_t>(n_slices, 8);
    std::vector<int64_t> b;
    for (int64_t i = 0; i <= k; ++i) b.push_back(g0 + G * i / k);
    int64_t gmax = 0;
    for (int64_t i = 0; i < k; ++i) gmax = std::max(gmax, b[i + 1] - b[i]);
    HCHECK(cudaMemcpy2DAsync(d_fields, (size_t)C * 4, h->fields, (size_t)h->field_ld * 4, (size_t)C * 4, (size_t)nf,
                             cudaMemcpyHostToDevice, s_h2d),
           "sp_predict_host: H2D");
    if (h->ragged_off)
      HCHECK(cudaMemcpyAsync(d_roff, h->ragged_off, (size_t)C * 8, cudaMemcpyHostToDevice, s_h2d), "sp_predict_host: H2D");
    if (rag)
      HCHECK(cudaMemcpyAsync(d_ragged, h->ragged, (size_t)h->n_ragged * 4, cudaMemcpyHostToDevice, s_h2d),
             "sp_predict_host: H2D");
    cudaEvent_t eu = next_event();
    HCHECK(cudaEventRecord(eu, s_h2d), "sp_predict_host: event");
    HCHECK(cudaStreamWaitEvent(comp, eu, 0), "sp_predict_host: event");
    for (int i = 0; i < 2; ++i) HCHECK(ctx->h_lat[i].need((size_t)std::max<int64_t>(gmax * C, 1) * 4), "sp_predict_host: staging");
    sp_config_batch d = *h;
    d.fields = d_fields;
    d.field_ld = C;
    d.ragged = h->ragged ? d_ragged : nullptr;
    d.ragged_off = h->ragged_off ? d_roff : nullptr;
    std::vector<cudaEvent_t> done;
    for (int64_t i = 0; i < k; ++i) {
      const int64_t ga = b[i], gb = b[i + 1];
      if (gb == ga) { done.push_back(nullptr); continue; }
      float *lat = (float *)ctx->h_lat[i % 2].p;
      if (i >= 2 && done[i - 2]) HCHECK(cudaStreamWaitEvent(comp, done[i - 2], 0), "sp_predict_host: event");
      sp_features f;
      sp_status st = features((gb - ga) * C, f);
      if (st != SP_OK) return st;
      sp_pairing pr{SP_PAIRS_CROSS, (int32_t)ga, (int32_t)gb, 0, 0, nullptr, nullptr};
      st = sp_featurize_predict(ctx, &d, specs, &pr, model, &f, lat, nullptr, comp);
      if (st != SP_OK) return st;
      cudaEvent_t ek = next_event(), ed = next_event();
      HCHECK(cudaEventRecord(ek, comp), "sp_predict_host: event");
      HCHECK(cudaStreamWaitEvent(s_d2h, ek, 0), "sp_predict_host: event");
      HCHECK(cudaMemcpyAsync(host_latency + (ga - g0) * C, lat, (size_t)((gb - ga) * C) * 4, cudaMemcpyDeviceToHost,
                             s_d2h),
             "sp_predict_host: D2H");
      HCHECK(cudaEventRecord(ed, s_d2h), "sp_predict_host: event");
      done.push_back(ed);
    }
  } else {
    // ---- config slices
    std::vector<int64_t> b{0};
    // measured on cfg2 after the round-2 kernel work: (1,2,3,2) 5.15 ms, (1,3,3,1) 5.27, (1,2,2,1)
    // 5.20, (1,2,3,3,1) 5.22 per step -- the later slices' copy-in hides under the longer kernels
    static const float kAttnWeights[4] = {1.f, 2.f, 3.f, 2.f};
    if (!weights && n_slices == 0 && fam == SP_ATTENTION) {  // kernels outlast the copies: short ends
      weights = kAttnWeights;
      n_slices = 4;
    }
    if (weights && n_slices > 0) {
      double tot = 0, cum = 0;
      for (int i = 0; i < n_slices; ++i) tot += std::max(0.0f, weights[i]);
      for (int i = 0; i < n_slices; ++i) {
        cum += std::max(0.0f, weights[i]);
        const int64_t x = (int64_t)((double)C * (tot > 0 ? cum / tot : 1.0));
        if (x > b.back() && x <= C) b.push_back(x);
      }
      if (b.back() != C) b.push_back(C);
    } else {
      // default 8 equal slices (copy-bound uniform families: measured 3.13e9 vs 2.99e9 pairs/s with 4 on cfg3)
      const int64_t k = std::max<int64_t>(1, std::min<int64_t>(n_slices > 0 ? n_slices : 8, C));
      for (int64_t i = 1; i <= k; ++i) b.push_back(C * i / k);
    }
    const int64_t ns = (int64_t)b.size() - 1;
    int64_t cmax = 0;
    for (int64_t i = 0; i < ns; ++i) cmax = std::max(cmax, b[i + 1] - b[i]);
    for (int i = 0; i < 2; ++i) HCHECK(ctx->h_lat[i].need((size_t)std::max<int64_t>(G * cmax, 1) * 4), "sp_predict_host: staging");
    std::vector<std::pair<int64_t, int64_t>> ranges;
    if (rag && plan) ranges = ragged_plan(*h, b);
    if (rag && ranges.empty())  // one whole copy ahead of the first slice
      HCHECK(cudaMemcpyAsync(d_ragged, h->ragged, (size_t)h->n_ragged * 4, cudaMemcpyHostToDevice, s_h2d),
             "sp_predict_host: H2D");
    if (!ranges.empty()) HCHECK(cudaMemsetAsync(d_flag, 0, 4, s_h2d), "sp_predict_host: flag");
    int row = 0, mult = 1;
    ragged_rule(fam, row, mult);
    std::vector<cudaEvent_t> done;
    for (int64_t i = 0; i < ns; ++i) {
      const int64_t c0 = b[i], c1 = b[i + 1], nc = c1 - c0;
      HCHECK(cudaMemcpy2DAsync(d_fields + c0, (size_t)C * 4, h->fields + c0, (size_t)h->field_ld * 4, (size_t)nc * 4,
                               (size_t)nf, cudaMemcpyHostToDevice, s_h2d),
             "sp_predict_host: H2D");
      if (h->ragged_off)
        HCHECK(cudaMemcpyAsync(d_roff + c0, h->ragged_off + c0, (size_t)nc * 8, cudaMemcpyHostToDevice, s_h2d),
               "sp_predict_host: H2D");
      if (!ranges.empty()) {
        const int64_t lo = ranges[i].first, hi = ranges[i].second;
        if (hi > lo)
          HCHECK(cudaMemcpyAsync(d_ragged + lo, h->ragged + lo, (size_t)(hi - lo) * 4, cudaMemcpyHostToDevice, s_h2d),
                 "sp_predict_host: H2D");
        const unsigned blocks = (unsigned)((nc + 255) / 256);
        if (blocks) {  // on the copy stream: off the kernels' critical path
          const LaunchHook hk = ctx->hook();
          hk.on_begin("ragged_guard", s_h2d);
          ragged_guard_kernel<<<blocks, 256, 0, s_h2d>>>(d_fields + (int64_t)row * C, d_roff, c0, c1, lo, hi, mult,
                                                         d_flag);
          hk.on_end(s_h2d);
          HCHECK(cudaGetLastError(), "sp_predict_host: guard launch");
        }
      }
      cudaEvent_t eu = next_event();
      HCHECK(cudaEventRecord(eu, s_h2d), "sp_predict_host: event");
      HCHECK(cudaStreamWaitEvent(comp, eu, 0), "sp_predict_host: event");
      if (i >= 2) HCHECK(cudaStreamWaitEvent(comp, done[i - 2], 0), "sp_predict_host: event");
      sp_config_batch d = *h;
      d.fields = d_fields + c0;
      d.field_ld = C;
      d.n_configs = nc;
      d.ragged = h->ragged ? d_ragged : nullptr;
      d.ragged_off = h->ragged_off ? d_roff + c0 : nullptr;
      sp_features f;
      sp_status st = features(G * nc, f);
      if (st != SP_OK) return st;
      float *lat = (float *)ctx->h_lat[i % 2].p;
      sp_pairing pr{SP_PAIRS_CROSS, g0, g1, 0, 0, nullptr, nullptr};
      st = sp_featurize_predict(ctx, &d, specs, &pr, model, &f, lat, nullptr, comp);
      if (st != SP_OK) return st;
      cudaEvent_t ek = next_event(), ed = next_event();
      HCHECK(cudaEventRecord(ek, comp), "sp_predict_host: event");
      HCHECK(cudaStreamWaitEvent(s_d2h, ek, 0), "sp_predict_host: event");
      // rows g of the spec-major output: host [g][c0, c1) <- device [g][0, nc)
      HCHECK(cudaMemcpy2DAsync(host_latency + c0, (size_t)C * 4, lat, (size_t)nc * 4, (size_t)nc * 4, (size_t)G,
                               cudaMemcpyDeviceToHost, s_d2h),
             "sp_predict_host: D2H");
      HCHECK(cudaEventRecord(ed, s_d2h), "sp_predict_host: event");
      done.push_back(ed);
    }
    if (!ranges.empty()) {
      int32_t missed = 0;
      HCHECK(cudaMemcpyAsync(&missed, d_flag, 4, cudaMemcpyDeviceToHost, s_h2d), "sp_predict_host: flag");
      HCHECK(cudaStreamSynchronize(s_h2d), "sp_predict_host: flag");
      *plan_missed = missed != 0;
    }
  }
  HCHECK(cudaStreamSynchronize(s_d2h), "sp_predict_host: D2H");
  // later work on `comp` (the next call's staging) stays ordered after these copies
  cudaEvent_t el = next_event();
  HCHECK(cudaEventRecord(el, s_d2h), "sp_predict_host: event");
  HCHECK(cudaStreamWaitEvent(comp, el, 0), "sp_predict_host: event");
  return SP_OK;
}

}  // namespace

extern "C" sp_status sp_predict_host(sp_ctx *ctx, const sp_config_batch *host_cfg, const sp_specs *specs,
                                     int32_t spec_begin, int32_t spec_end, const sp_model *model, float *host_latency,
                                     const float *slice_weights, int32_t n_slices, void *stream) {
  if (!ctx) return fail(nullptr, SP_E_ARG, "sp_predict_host: ctx is NULL");
  if (!host_cfg || !specs || !model) return fail(ctx, SP_E_ARG, "sp_predict_host: NULL argument");
  const int32_t G = sp_specs_count(specs);
  if (spec_begin < 0 || spec_end > G || spec_begin > spec_end)
    return fail(ctx, SP_E_ARG, "sp_predict_host: spec range out of bounds");
  const sp_config_batch &h = *host_cfg;
  if (h.n_configs < 0 || h.field_ld < h.n_configs || h.n_fields <= 0)
    return fail(ctx, SP_E_ARG, "sp_predict_host: bad n_configs / field_ld / n_fields");
  if (n_slices < 0 || (slice_weights && n_slices == 0)) return fail(ctx, SP_E_ARG, "sp_predict_host: bad slices");
  const int64_t n = (int64_t)(spec_end - spec_begin) * h.n_configs;
  if (n == 0) return SP_OK;
  if (!host_latency || !h.fields) return fail(ctx, SP_E_ARG, "sp_predict_host: NULL buffer");
  if (h.n_ragged < 0 || (h.n_ragged > 0 && (!h.ragged || !h.ragged_off)))
    return fail(ctx, SP_E_ARG, "sp_predict_host: ragged data needs ragged and ragged_off");
  if (h.family != SP_ATTENTION && h.family != SP_FUSED_MOE && h.ragged_off)
    return fail(ctx, SP_E_ARG, "sp_predict_host: the family has no ragged data");
  ctx->err.clear();
  cudaSetDevice(ctx->device);
  cudaStream_t comp = reinterpret_cast<cudaStream_t>(stream);
  bool missed = false;
  sp_status st = run(ctx, &h, specs, spec_begin, spec_end, model, host_latency, slice_weights, n_slices, comp, true,
                     &missed);
  if (st == SP_OK && missed)  // the boundary plan missed some ragged data: redo with one whole copy
    st = run(ctx, &h, specs, spec_begin, spec_end, model, host_latency, slice_weights, n_slices, comp, false, &missed);
  return st;
}
