// Host side of the C-ABI (include/synperf.h): argument validation, spec
// staging (step a1), model layout, per-range attention plans and kernel
// dispatch.  No exception crosses the ABI; every entry point returns an
// sp_status and records a message for sp_last_error().
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "ctx.h"
#include "sp_internal.h"
#include "synperf.h"

using namespace sp;

namespace sp {
thread_local std::string g_noctx_err;
}  // namespace sp

namespace {

int nfields_of(int fam) {
  switch (fam) {
    case SP_GEMM: return SP_NFIELDS_GEMM;
    case SP_ATTENTION: return SP_NFIELDS_ATTENTION;
    case SP_FUSED_MOE: return SP_NFIELDS_FUSED_MOE;
    case SP_RMSNORM: return SP_NFIELDS_RMSNORM;
    case SP_SILU_MUL: return SP_NFIELDS_SILU_MUL;
    case SP_SCALED_MM: return SP_NFIELDS_SCALED_MM;
    case SP_GEMM_SPLITK: return SP_NFIELDS_GEMM_SPLITK;
    default: return -1;
  }
}

int pipes_count(int fam) {
  int p = family_pipes(fam), n = 0;
  for (int k = 0; k < 3; ++k) n += (p >> k) & 1;
  return n;
}

constexpr int kAttnMaxSms = 4096;
constexpr int kAttnWordBudget = 2048;
constexpr int kAttnMaxDistinct = 8;  // featurize_attention.cu kMaxDistinct

// Device copy of one attention spec-group plan (see featurize_attention.cu).
struct AttnPlanDev {
  DevBuf groups, group_specs, spec_dist, distinct_n, distinct_off, spec_slot;
  std::vector<int32_t> nd;   // host copies for the launcher
  std::vector<uint8_t> small;
  AttnPlan view{};
};

}  // namespace

struct sp_specs {
  sp_ctx *ctx = nullptr;
  std::vector<sp_gpu_spec> host;
  DevBuf dev;  // DevSpec[n]
  int32_t n = 0;
  int32_t max_sms = 0;
  std::mutex mu;
  std::map<std::pair<int, int>, std::unique_ptr<AttnPlanDev>> plans;
};

struct sp_model {
  int family = 0, n_in = 0, precision = 0;
  DevBuf fp32;   // fp32 path buffers (one allocation)
  MlpFp32 m32{};
  DevBuf bf16w;  // bf16 path: packed weights
  DevBuf bf16v;  // bf16 path: fp32 vectors
  MlpBf16 m16{};
};

// ------------------------------------------------------------------ context

extern "C" const char *sp_version(void) { return "synperf-b200 0.1 (sm_100a)"; }

extern "C" sp_status sp_create(int device, sp_ctx **out) {
  if (!out) return fail(nullptr, SP_E_ARG, "sp_create: out is NULL");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "sp_create: cudaGetDeviceCount");
  if (device < 0 || device >= n) return fail(nullptr, SP_E_ARG, "sp_create: bad device index");
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "sp_create: cudaGetDeviceProperties");
  if (prop.major != 10 || prop.minor != 0)
    return fail(nullptr, SP_E_UNSUPPORTED,
                "sp_create: libsynperf is built for sm_100a (B200); device is sm_" +
                    std::to_string(prop.major) + std::to_string(prop.minor));
  sp_ctx *c = new (std::nothrow) sp_ctx;
  if (!c) return fail(nullptr, SP_E_INTERNAL, "sp_create: out of host memory");
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  cudaSetDevice(device);
  e = cudaMalloc(&c->counters, kAttnCounterInts * sizeof(int));
  if (e != cudaSuccess) {
    c->counters = nullptr;
    delete c;
    return cuda_fail(nullptr, e, "sp_create: scratch allocation");
  }
  *out = c;
  return SP_OK;
}

extern "C" void sp_destroy(sp_ctx *ctx) { delete ctx; }

extern "C" const char *sp_last_error(const sp_ctx *ctx) {
  return ctx ? ctx->err.c_str() : g_noctx_err.c_str();
}

extern "C" int32_t sp_device_sms(const sp_ctx *ctx) { return ctx ? ctx->num_sms : 0; }

// ------------------------------------------------------------ a1 spec staging

extern "C" sp_status sp_load_gpu_specs(sp_ctx *ctx, const sp_gpu_spec *host_specs, int32_t n,
                                       uint32_t flags, sp_specs **out) {
  if (!ctx || !out || (!host_specs && n > 0) || n < 0)
    return fail(ctx, SP_E_ARG, "sp_load_gpu_specs: NULL argument or negative count");
  *out = nullptr;
  ctx->err.clear();
  cudaSetDevice(ctx->device);
  std::vector<DevSpec> dev(n);
  std::string warn;
  int32_t max_sms = 0;
  for (int32_t i = 0; i < n; ++i) {
    const sp_gpu_spec &s = host_specs[i];
    const std::string who = "spec " + std::to_string(i) + " (" + std::string(s.name, strnlen(s.name, 32)) + ")";
    // positivity invariants
    if (s.num_sms < 1) return fail(ctx, SP_E_DATA, who + ": invalid SM count");
    if (!(s.sm_clock_mhz > 0) || !std::isfinite(s.sm_clock_mhz))
      return fail(ctx, SP_E_DATA, who + ": non-positive SM clock");
    if (!(s.bw_global_gbps > 0) || !std::isfinite(s.bw_global_gbps) || !(s.bw_l2_gbps > 0) ||
        !std::isfinite(s.bw_l2_gbps))
      return fail(ctx, SP_E_DATA, who + ": non-positive memory bandwidth");
    if (s.th_fma < 1 || s.th_xu < 1 || s.smem_bw_bytes_per_clk < 1)
      return fail(ctx, SP_E_DATA, who + ": non-positive pipe throughput");
    if (s.th_tensor_bf16 < 0 || s.th_tensor_fp16 < 0 || s.th_tensor_fp8 < 0)
      return fail(ctx, SP_E_DATA, who + ": negative tensor throughput");
    if (s.smem_per_sm_bytes < 0 || s.regfile_per_sm_bytes < 4 || s.max_warps_per_sm < 1 ||
        s.max_ctas_per_sm < 1)
      return fail(ctx, SP_E_DATA, who + ": invalid occupancy limits");
    // Table II ranges: warnings unless SP_STRICT
    std::string out_of_range;
    const double cc = s.cc_major + s.cc_minor / 10.0;
    if (cc < 8.0 || cc > 12.0) out_of_range += " compute capability";
    if (s.num_sms < 78 || s.num_sms > 188) out_of_range += " SMs";
    if (s.sm_clock_mhz < 1410 || s.sm_clock_mhz > 2520) out_of_range += " clock";
    if (s.th_tensor_bf16 < 512 || s.th_tensor_bf16 > 4096) out_of_range += " tensor";
    if (s.th_fma < 64 || s.th_fma > 128) out_of_range += " FMA";
    if (s.th_xu != 16) out_of_range += " XU";
    if (s.bw_global_gbps < 696 || s.bw_global_gbps > 4916) out_of_range += " global-BW";
    if (s.bw_l2_gbps < 2430 || s.bw_l2_gbps > 10400) out_of_range += " L2-BW";
    if (s.smem_bw_bytes_per_clk != 128) out_of_range += " smem-BW";
    if (s.smem_per_sm_bytes < 100 * 1024 || s.smem_per_sm_bytes > 228 * 1024) out_of_range += " smem";
    if (s.regfile_per_sm_bytes != 256 * 1024) out_of_range += " RF";
    if (!out_of_range.empty()) {
      if (flags & SP_STRICT) return fail(ctx, SP_E_DATA, who + ": outside Table II ranges:" + out_of_range);
      if (warn.empty()) warn = "warning: " + who + " outside Table II ranges:" + out_of_range;
    }
    // derived constants in fp64 (Eq.4-5; C_mem = B/BW; R8)
    DevSpec d{};
    const double N = s.num_sms, f = s.sm_clock_mhz;
    d.num_sms = s.num_sms;
    d.smem_per_sm = s.smem_per_sm_bytes;
    d.regs_per_sm = s.regfile_per_sm_bytes / 4;
    d.max_warps = s.max_warps_per_sm;
    d.max_ctas = s.max_ctas_per_sm;
    const int32_t th_t[3] = {s.th_tensor_bf16, s.th_tensor_fp16, s.th_tensor_fp8};
    for (int k = 0; k < 3; ++k) {
      d.tensor_ok[k] = th_t[k] > 0;
      d.cg_tensor[k] = th_t[k] > 0 ? 1.0 / (N * th_t[k]) : 0.0;
      d.cs_tensor[k] = th_t[k] > 0 ? 1.0 / th_t[k] : 0.0;
    }
    d.cg_fma = 1.0 / (N * s.th_fma);
    d.cs_fma = 1.0 / s.th_fma;
    d.cg_xu = 1.0 / (N * s.th_xu);
    d.cs_xu = 1.0 / s.th_xu;
    d.glob_g = f / (s.bw_global_gbps * 1e3);
    d.l2_g = f / (s.bw_l2_gbps * 1e3);
    d.glob_s = f / (s.bw_global_gbps * 1e3 / N);
    d.l2_s = f / (s.bw_l2_gbps * 1e3 / N);
    d.smem_s = 1.0 / s.smem_bw_bytes_per_clk;
    d.inv_f = 1.0 / f;
    dev[i] = d;
    max_sms = std::max(max_sms, s.num_sms);
  }
  sp_specs *h = new (std::nothrow) sp_specs;
  if (!h) return fail(ctx, SP_E_INTERNAL, "sp_load_gpu_specs: out of host memory");
  h->ctx = ctx;
  h->host.assign(host_specs, host_specs + n);
  h->n = n;
  h->max_sms = max_sms;
  cudaError_t e = h->dev.alloc_copy(dev.data(), dev.size() * sizeof(DevSpec));
  if (e != cudaSuccess) {
    delete h;
    return cuda_fail(ctx, e, "sp_load_gpu_specs: upload");
  }
  *out = h;
  ctx->err = warn;
  return SP_OK;
}

extern "C" void sp_free_specs(sp_specs *specs) { delete specs; }
extern "C" int32_t sp_specs_count(const sp_specs *specs) { return specs ? specs->n : 0; }

// Attention plan for specs [b, e): distinct SM counts grouped so a warp's
// accumulators fit its shared-memory budget.  Built once per range, cached.
static sp_status attn_plan(sp_ctx *ctx, sp_specs *sp, int b, int e, const AttnPlan **out) {
  std::lock_guard<std::mutex> lock(sp->mu);
  auto key = std::make_pair(b, e);
  auto it = sp->plans.find(key);
  if (it != sp->plans.end()) { *out = &it->second->view; return SP_OK; }
  std::vector<int32_t> Ns;
  for (int g = b; g < e; ++g) Ns.push_back(sp->host[g].num_sms);
  std::sort(Ns.begin(), Ns.end());
  Ns.erase(std::unique(Ns.begin(), Ns.end()), Ns.end());
  if (!Ns.empty() && Ns.back() > kAttnMaxSms)
    return fail(ctx, SP_E_UNSUPPORTED, "attention featurization supports at most 4096 SMs per spec");
  const int budget = std::max(kAttnWordBudget, Ns.empty() ? 0 : ((Ns.back() + kAttnSlack + 3) & ~3));
  std::vector<AttnGroup> groups;
  std::vector<int32_t> gspecs, sdist, dn, doff;
  size_t i = 0;
  int words_max = 0;
  while (i < Ns.size()) {
    AttnGroup gr{};
    gr.distinct_first = (int32_t)dn.size();
    int words = 0;
    while (i < Ns.size() && gr.n_distinct < kAttnMaxDistinct && words + Ns[i] + kAttnSlack <= budget) {
      dn.push_back(Ns[i]);
      doff.push_back(words);
      words += Ns[i] + kAttnSlack;  // + the lazy-wrap overflow of the region
      ++gr.n_distinct;
      ++i;
    }
    words_max = std::max(words_max, (words + 3) & ~3);
    gr.spec_first = (int32_t)gspecs.size();
    for (int g = b; g < e; ++g) {
      const int32_t n = sp->host[g].num_sms;
      for (int d = 0; d < gr.n_distinct; ++d) {
        if (dn[gr.distinct_first + d] == n) {
          gspecs.push_back(g);
          sdist.push_back(gr.distinct_first + d);
          ++gr.n_specs;
        }
      }
    }
    groups.push_back(gr);
  }
  std::vector<int32_t> slot(e - b, -1);  // per spec of the range: its distinct slot
  for (int g = b; g < e; ++g)
    for (size_t d = 0; d < dn.size(); ++d)
      if (dn[d] == sp->host[g].num_sms) slot[g - b] = (int32_t)d;
  std::unique_ptr<AttnPlanDev> pd(new (std::nothrow) AttnPlanDev);
  if (!pd) return fail(ctx, SP_E_INTERNAL, "attention plan: out of host memory");
  cudaError_t err;
  if ((err = pd->groups.alloc_copy(groups.data(), groups.size() * sizeof(AttnGroup))) != cudaSuccess ||
      (err = pd->group_specs.alloc_copy(gspecs.data(), gspecs.size() * 4)) != cudaSuccess ||
      (err = pd->spec_dist.alloc_copy(sdist.data(), sdist.size() * 4)) != cudaSuccess ||
      (err = pd->distinct_n.alloc_copy(dn.data(), dn.size() * 4)) != cudaSuccess ||
      (err = pd->distinct_off.alloc_copy(doff.data(), doff.size() * 4)) != cudaSuccess ||
      (err = pd->spec_slot.alloc_copy(slot.data(), slot.size() * 4)) != cudaSuccess)
    return cuda_fail(ctx, err, "attention plan upload");
  pd->view.groups = (const AttnGroup *)pd->groups.p;
  pd->view.group_specs = (const int32_t *)pd->group_specs.p;
  pd->view.spec_dist = (const int32_t *)pd->spec_dist.p;
  pd->view.distinct_n = (const int32_t *)pd->distinct_n.p;
  pd->view.distinct_off = (const int32_t *)pd->distinct_off.p;
  pd->view.spec_slot = (const int32_t *)pd->spec_slot.p;
  pd->view.n_slots = (int32_t)dn.size();
  pd->view.min_n = dn.empty() ? 0 : dn.front();  // Ns ascending
  pd->view.n_groups = (int32_t)groups.size();
  pd->view.words_per_warp = words_max + kAttnScratchWords;  // accumulators + request scratch
  for (const AttnGroup &gr : groups) {
    pd->nd.push_back(gr.n_distinct);
    pd->small.push_back(dn[gr.distinct_first] < kAttnLazyMinN);  // Ns ascending: first is the smallest
  }
  pd->view.host_nd = pd->nd.data();
  pd->view.host_small = pd->small.data();
  *out = &pd->view;
  sp->plans.emplace(key, std::move(pd));
  return SP_OK;
}

// Context scratch, grow-only (include/synperf.h Conventions; sp_prepare).
static sp_status grow_buf(sp_ctx *ctx, void *&p, size_t &bytes, size_t need, const char *what) {
  if (need <= bytes) return SP_OK;
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
  cudaError_t me = cudaMalloc(&p, need);
  if (me != cudaSuccess) {
    p = nullptr;
    return cuda_fail(ctx, me, what);
  }
  bytes = need;
  return SP_OK;
}
// attention per-config results of the schedule kernel: st (4 B), L, U, and maxS/maxB per slot (8 B each)
static sp_status grow_attn_res(sp_ctx *ctx, int64_t C, int n_slots) {
  const int64_t ld = (C + 31) & ~(int64_t)31;
  return grow_buf(ctx, ctx->attn_res, ctx->attn_res_bytes,
                  (size_t)ld * (4 + 8 + 8 + 16 * (size_t)n_slots + 4 * (size_t)kAttnPreWords + 4),
                  "attention result scratch");
}
static sp_status grow_pre(sp_ctx *ctx, int64_t C) {
  const int64_t ldc = (C + 31) & ~(int64_t)31;
  return grow_buf(ctx, ctx->pre, ctx->pre_bytes, (size_t)ldc * kPreFields * sizeof(uint64_t),
                  "fused pre-pass scratch");
}

extern "C" sp_status sp_prepare(sp_ctx *ctx, int32_t family, int64_t n_configs, const sp_specs *specs_c,
                                int32_t spec_begin, int32_t spec_end) {
  if (!ctx) return fail(nullptr, SP_E_ARG, "sp_prepare: ctx is NULL");
  if (!specs_c || nfields_of(family) < 0 || n_configs < 0) return fail(ctx, SP_E_ARG, "sp_prepare: bad argument");
  sp_specs *specs = const_cast<sp_specs *>(specs_c);
  if (spec_begin < 0 || spec_end > specs->n || spec_begin > spec_end)
    return fail(ctx, SP_E_ARG, "sp_prepare: spec range out of bounds");
  ctx->err.clear();
  cudaSetDevice(ctx->device);
  if (family == SP_ATTENTION) {
    const AttnPlan *plan = nullptr;
    sp_status st = attn_plan(ctx, specs, spec_begin, spec_end, &plan);
    if (st != SP_OK) return st;
    st = grow_attn_res(ctx, n_configs, plan->n_slots);
    if (st != SP_OK) return st;
    return grow_pre(ctx, n_configs);  // the fused path's per-config record
  }
  if (family != SP_GEMM_SPLITK) return grow_pre(ctx, n_configs);
  return SP_OK;
}

// --------------------------------------------------------------- featurize

// Attention, CROSS: plan + scratch, then the pre-pass, schedule, (emit) and planner
// kernels.  emit = false for the fused path (the fused kernel writes the records).
static sp_status attn_cross(sp_ctx *ctx, sp_specs *specs, const sp_pairing *pairs, const ConfigView &cv,
                            const FeatOut &fo, int64_t n_pairs, void *stream, bool emit, AttnPlan &run,
                            AttnResults &res) {
  const AttnPlan *plan = nullptr;
  sp_status st = attn_plan(ctx, specs, pairs->spec_begin, pairs->spec_end, &plan);
  if (st != SP_OK) return st;
  if (plan->n_groups > kAttnMaxGroups)
    return fail(ctx, SP_E_UNSUPPORTED, "attention featurization: too many distinct SM-count groups");
  run = *plan;
  run.counters = ctx->counters;
  // per-config results of the schedule kernel: st (4 B), L, U, (lo, hi) per slot (8 B each), pre-pass record
  const int64_t C = cv.n_configs, ld = (C + 31) & ~(int64_t)31;
  st = grow_attn_res(ctx, C, run.n_slots);
  if (st != SP_OK) return st;
  char *base = (char *)ctx->attn_res;
  res.ld = ld;
  res.L = (int64_t *)base;
  res.U = (uint64_t *)(base + 8 * ld);
  res.mS = (int64_t *)(base + 16 * ld);
  res.mB = res.mS + (size_t)run.n_slots * ld;
  res.st = (int32_t *)(res.mB + (size_t)run.n_slots * ld);
  res.pre = (uint32_t *)(res.st + ld);
  res.order = (int32_t *)(res.pre + (size_t)kAttnPreWords * ld);
  res.chunk_b = (int8_t *)(res.order + ld / 32);
  res.hist = ctx->counters + run.n_groups;
  const int e = launch_featurize_attention(cv, (const DevSpec *)specs->dev.p, pairs->spec_begin, pairs->spec_end,
                                           specs->n, run, res, n_pairs, nullptr, nullptr, specs->max_sms, fo,
                                           ctx->num_sms, stream, ctx->hook(), emit);
  if (e) return cuda_fail(ctx, e, "sp_featurize: attention launch");
  return SP_OK;
}

extern "C" sp_status sp_featurize(sp_ctx *ctx, const sp_config_batch *cfg, const sp_specs *specs_c,
                                  const sp_pairing *pairs, const sp_features *out, void *stream) {
  return sp_featurize_sched(ctx, cfg, specs_c, pairs, SP_SCHED_RR, out, stream);
}

extern "C" sp_status sp_featurize_sched(sp_ctx *ctx, const sp_config_batch *cfg, const sp_specs *specs_c,
                                        const sp_pairing *pairs, int32_t scheduler, const sp_features *out,
                                        void *stream) {
  return sp_featurize_ex(ctx, cfg, specs_c, pairs, scheduler, 0u, out, stream);
}

extern "C" sp_status sp_featurize_ex(sp_ctx *ctx, const sp_config_batch *cfg, const sp_specs *specs_c,
                                     const sp_pairing *pairs, int32_t scheduler, uint32_t flags,
                                     const sp_features *out, void *stream) {
  if (!ctx) return fail(nullptr, SP_E_ARG, "sp_featurize: ctx is NULL");
  if (scheduler != SP_SCHED_RR && scheduler != SP_SCHED_GREEDY && scheduler != SP_SCHED_MINHEAP)
    return fail(ctx, SP_E_ARG, "sp_featurize_sched: unknown scheduler");
  if (flags & ~SP_FEAT_CLAMPED) return fail(ctx, SP_E_ARG, "sp_featurize_ex: unknown flag");
  if (!cfg || !specs_c || !pairs || !out) return fail(ctx, SP_E_ARG, "sp_featurize: NULL argument");
  sp_specs *specs = const_cast<sp_specs *>(specs_c);
  const int fam = cfg->family;
  if (nfields_of(fam) < 0) return fail(ctx, SP_E_ARG, "sp_featurize: unknown family");
  if (cfg->n_fields != nfields_of(fam))
    return fail(ctx, SP_E_ARG, "sp_featurize: n_fields does not match the family's field count");
  if (cfg->n_configs < 0 || cfg->field_ld < cfg->n_configs)
    return fail(ctx, SP_E_ARG, "sp_featurize: bad n_configs / field_ld");
  if (cfg->n_configs > 0 && !cfg->fields) return fail(ctx, SP_E_ARG, "sp_featurize: fields is NULL");
  if (fam == SP_ATTENTION && cfg->n_configs > 0 && (!cfg->ragged || !cfg->ragged_off))
    return fail(ctx, SP_E_ARG, "sp_featurize: attention needs ragged (qlen, kvlen) data");
  if (fam == SP_FUSED_MOE && cfg->ragged_off && !cfg->ragged)
    return fail(ctx, SP_E_ARG, "sp_featurize: MoE ragged_off without ragged");
  if (out->family != fam) return fail(ctx, SP_E_ARG, "sp_featurize: out->family != cfg->family");
  int64_t n_pairs;
  if (pairs->kind == SP_PAIRS_CROSS) {
    if (pairs->spec_begin < 0 || pairs->spec_end > specs->n || pairs->spec_begin > pairs->spec_end)
      return fail(ctx, SP_E_ARG, "sp_featurize: spec range out of bounds");
    n_pairs = (int64_t)(pairs->spec_end - pairs->spec_begin) * cfg->n_configs;
  } else if (pairs->kind == SP_PAIRS_LIST) {
    n_pairs = pairs->n_pairs;
    if (n_pairs < 0 || (n_pairs > 0 && (!pairs->cfg_idx || !pairs->spec_idx)))
      return fail(ctx, SP_E_ARG, "sp_featurize: bad pair list");
  } else {
    return fail(ctx, SP_E_ARG, "sp_featurize: unknown pairing kind");
  }
  if (out->n_pairs != n_pairs || out->ld < n_pairs)
    return fail(ctx, SP_E_ARG, "sp_featurize: out->n_pairs / ld do not match the pairing");
  if (n_pairs > 0 && (!out->ints || !out->flts || !out->status))
    return fail(ctx, SP_E_ARG, "sp_featurize: output buffers are NULL");
  if (n_pairs == 0) return SP_OK;
  ctx->err.clear();
  cudaSetDevice(ctx->device);

  ConfigView cv{cfg->fields, cfg->ragged, cfg->ragged_off, cfg->n_configs, cfg->field_ld};
  FeatOut fo{out->ints, out->flts, out->status, out->ld};
  const DevSpec *ds = (const DevSpec *)specs->dev.p;
  int e;
  if (flags & SP_FEAT_CLAMPED) {
    if (fam != SP_GEMM && fam != SP_FUSED_MOE && fam != SP_ATTENTION)
      return fail(ctx, SP_E_UNSUPPORTED,
                  "sp_featurize_ex: clamped edge tiles are implemented for GEMM, fused MoE and attention");
    if (scheduler != SP_SCHED_RR)
      return fail(ctx, SP_E_UNSUPPORTED, "sp_featurize_ex: clamped edge tiles use the cyclic (RR) scheduler");
    if (specs->max_sms > 4096) return fail(ctx, SP_E_UNSUPPORTED, "sp_featurize_ex: clamped mode supports <= 4096 SMs");
    const bool cross = pairs->kind == SP_PAIRS_CROSS;
    const LaunchHook h = ctx->hook();
    h.on_begin(fam == SP_ATTENTION ? "attn_clamped" : "featurize_clamped", stream);
    if (fam == SP_ATTENTION)
      e = launch_attention_clamped(cv, ds, cross ? pairs->spec_begin : 0, specs->n, n_pairs,
                                   cross ? nullptr : pairs->cfg_idx, cross ? nullptr : pairs->spec_idx,
                                   specs->max_sms, fo, ctx->num_sms, stream);
    else
      e = launch_featurize_clamped(fam, cv, ds, cross ? pairs->spec_begin : 0, specs->n, n_pairs,
                                   cross ? nullptr : pairs->cfg_idx, cross ? nullptr : pairs->spec_idx,
                                   specs->max_sms, fo, ctx->num_sms, stream);
    h.on_end(stream);
  } else if (fam == SP_GEMM_SPLITK && scheduler != SP_SCHED_RR) {
    // split-K tasks come in two sizes (R25): GREEDY / MINHEAP would not reduce to the cyclic closed form
    return fail(ctx, SP_E_UNSUPPORTED, "sp_featurize_sched: split-K GEMM supports the cyclic (RR) scheduler only");
  } else if (fam == SP_ATTENTION && scheduler != SP_SCHED_RR) {
    // sequential scheduler simulation: per-warp shared memory for the largest target set
    const bool cross = pairs->kind == SP_PAIRS_CROSS;
    const int b = cross ? pairs->spec_begin : 0, en = cross ? pairs->spec_end : specs->n;
    int64_t max_targets = 1;
    for (int g = b; g < en; ++g) {
      const int64_t n = specs->host[g].num_sms;
      max_targets = std::max(max_targets, scheduler == SP_SCHED_GREEDY ? n : n * specs->host[g].max_ctas_per_sm);
    }
    if (attention_sim_smem_bytes(max_targets) > 227 * 1024)
      return fail(ctx, SP_E_UNSUPPORTED, "sp_featurize_sched: scheduler state of these specs exceeds shared memory");
    e = launch_attention_sim(scheduler, cv, ds, b, en, specs->n, n_pairs, cross ? nullptr : pairs->cfg_idx,
                             cross ? nullptr : pairs->spec_idx, max_targets, fo, ctx->num_sms, stream, ctx->hook());
  } else if (fam == SP_ATTENTION) {
    if (pairs->kind == SP_PAIRS_CROSS) {
      AttnPlan run;
      AttnResults res;
      sp_status st = attn_cross(ctx, specs, pairs, cv, fo, n_pairs, stream, true, run, res);
      if (st != SP_OK) return st;
      e = 0;
    } else {
      if (specs->max_sms > kAttnMaxSms)
        return fail(ctx, SP_E_UNSUPPORTED, "attention featurization supports at most 4096 SMs per spec");
      AttnPlan none{};
      AttnResults nores{};
      e = launch_featurize_attention(cv, ds, 0, specs->n, specs->n, none, nores, n_pairs, pairs->cfg_idx,
                                     pairs->spec_idx, specs->max_sms, fo, ctx->num_sms, stream, ctx->hook());
    }
  } else if (pairs->kind == SP_PAIRS_CROSS) {
    const LaunchHook h = ctx->hook();
    h.on_begin(fam == SP_GEMM_SPLITK ? "featurize_splitk_cross" : "featurize_uniform_cross", stream);
    e = launch_featurize_uniform(fam, cv, ds, pairs->spec_begin, pairs->spec_end, n_pairs, nullptr, nullptr,
                                 fo, stream);
    h.on_end(stream);
  } else {
    const LaunchHook h = ctx->hook();
    h.on_begin(fam == SP_GEMM_SPLITK ? "featurize_splitk_list" : "featurize_uniform_list", stream);
    e = launch_featurize_uniform(fam, cv, ds, 0, specs->n, n_pairs, pairs->cfg_idx, pairs->spec_idx, fo,
                                 stream);
    h.on_end(stream);
  }
  if (e) return cuda_fail(ctx, e, "sp_featurize: launch");
  return SP_OK;
}

// --------------------------------------------------------- fused featurize -> predict

extern "C" sp_status sp_featurize_predict(sp_ctx *ctx, const sp_config_batch *cfg, const sp_specs *specs,
                                          const sp_pairing *pairs, const sp_model *model, const sp_features *out,
                                          float *latency_us, float *efficiency, void *stream) {
  if (!ctx) return fail(nullptr, SP_E_ARG, "sp_featurize_predict: ctx is NULL");
  if (!cfg || !specs || !pairs || !model || !out) return fail(ctx, SP_E_ARG, "sp_featurize_predict: NULL argument");
  if (model->family != cfg->family) return fail(ctx, SP_E_ARG, "sp_featurize_predict: config/model family mismatch");
  const int fam = cfg->family;
  const bool fusable = (fam == SP_GEMM || fam == SP_FUSED_MOE || fam == SP_RMSNORM || fam == SP_SILU_MUL ||
                        fam == SP_SCALED_MM || fam == SP_ATTENTION) &&
                       pairs->kind == SP_PAIRS_CROSS &&
                       (model->precision == SP_MLP_BF16 || model->precision == SP_MLP_FP16);
  if (!fusable) {  // the two-kernel path (attention, split-K, pair lists, the fp32 predictor)
    sp_status st = sp_featurize(ctx, cfg, specs, pairs, out, stream);
    if (st != SP_OK) return st;
    return sp_predict(ctx, model, out, latency_us, efficiency, stream);
  }
  // argument checks of sp_featurize (CROSS)
  if (cfg->n_fields != nfields_of(fam))
    return fail(ctx, SP_E_ARG, "sp_featurize_predict: n_fields does not match the family's field count");
  if (cfg->n_configs < 0 || cfg->field_ld < cfg->n_configs)
    return fail(ctx, SP_E_ARG, "sp_featurize_predict: bad n_configs / field_ld");
  if (cfg->n_configs > 0 && !cfg->fields) return fail(ctx, SP_E_ARG, "sp_featurize_predict: fields is NULL");
  if (fam == SP_FUSED_MOE && cfg->ragged_off && !cfg->ragged)
    return fail(ctx, SP_E_ARG, "sp_featurize_predict: MoE ragged_off without ragged");
  if (fam == SP_ATTENTION && cfg->n_configs > 0 && (!cfg->ragged || !cfg->ragged_off))
    return fail(ctx, SP_E_ARG, "sp_featurize_predict: attention needs ragged (qlen, kvlen) data");
  if (out->family != fam) return fail(ctx, SP_E_ARG, "sp_featurize_predict: out->family != cfg->family");
  if (pairs->spec_begin < 0 || pairs->spec_end > specs->n || pairs->spec_begin > pairs->spec_end)
    return fail(ctx, SP_E_ARG, "sp_featurize_predict: spec range out of bounds");
  const int64_t n_pairs = (int64_t)(pairs->spec_end - pairs->spec_begin) * cfg->n_configs;
  if (out->n_pairs != n_pairs || out->ld < n_pairs)
    return fail(ctx, SP_E_ARG, "sp_featurize_predict: out->n_pairs / ld do not match the pairing");
  if (n_pairs == 0) return SP_OK;
  if (!out->ints || !out->flts || !out->status || !latency_us)
    return fail(ctx, SP_E_ARG, "sp_featurize_predict: NULL buffer");
  ctx->err.clear();
  cudaSetDevice(ctx->device);
  const int64_t C = cfg->n_configs, ldc = (C + 31) & ~(int64_t)31;
  const size_t need = (size_t)ldc * kPreFields * sizeof(uint64_t);
  sp_status gst = grow_pre(ctx, C);
  if (gst != SP_OK) return gst;
  ConfigView cv{cfg->fields, cfg->ragged, cfg->ragged_off, cfg->n_configs, cfg->field_ld};
  const LaunchHook h = ctx->hook();
  FusedIn fi{};
  int e;
  if (fam == SP_ATTENTION) {
    // schedule (+ the planner's pairs, written to `out`), then the per-config record
    AttnPlan run;
    AttnResults res;
    sp_status st = attn_cross(ctx, const_cast<sp_specs *>(specs), pairs, cv,
                              FeatOut{out->ints, out->flts, out->status, out->ld}, n_pairs, stream, false, run, res);
    if (st != SP_OK) return st;
    h.on_begin("attn_fuse_prep", stream);
    e = launch_attn_fuse_prep(cv, res, (uint64_t *)ctx->pre, ldc, stream);
    h.on_end(stream);
    if (e) return cuda_fail(ctx, e, "sp_featurize_predict: attention pre-pass launch");
    fi.slot = run.spec_slot;
    fi.lo = res.mS;
    fi.hi = res.mB;
    fi.lohi_ld = res.ld;
  } else {
    h.on_begin("uniform_prepass", stream);
    e = launch_uniform_prepass(fam, cv, (uint64_t *)ctx->pre, ldc, stream);
    h.on_end(stream);
    if (e) return cuda_fail(ctx, e, "sp_featurize_predict: pre-pass launch");
  }
  fi.pre = (const uint64_t *)ctx->pre;
  fi.ldc = ldc;
  fi.C = C;
  fi.g0 = pairs->spec_begin;
  fi.n_specs = pairs->spec_end - pairs->spec_begin;
  fi.inv_c = 0.0;
  // config-major tiles when the pre-pass would not stay in L2 across the spec sweep
  fi.cmajor = fi.n_specs > 1 && need > ((size_t)32 << 20) ? 1 : 0;
  fi.specs = (const DevSpec *)specs->dev.p;
  fi.out = FeatOut{out->ints, out->flts, out->status, out->ld};
  fi.n_pairs = n_pairs;
  h.on_begin("predict_tcgen05_fused", stream);
  e = launch_predict_tcgen05_fused(model->m16, fi, latency_us, efficiency, ctx->num_sms, stream);
  h.on_end(stream);
  if (e) return cuda_fail(ctx, e, "sp_featurize_predict: launch");
  return SP_OK;
}

// -------------------------------------------------------------------- model

static bool all_finite(const float *p, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(p[i])) return false;
  return true;
}

extern "C" sp_status sp_load_model(sp_ctx *ctx, const sp_mlp_desc *d, sp_model **out) {
  if (!ctx || !d || !out) return fail(ctx, SP_E_ARG, "sp_load_model: NULL argument");
  *out = nullptr;
  ctx->err.clear();
  cudaSetDevice(ctx->device);
  if (nfields_of(d->family) < 0) return fail(ctx, SP_E_ARG, "sp_load_model: unknown family");
  const int n_in = d->n_in;
  if (n_in != 4 * pipes_count(d->family) + 7)
    return fail(ctx, SP_E_DATA, "sp_load_model: n_in does not match the family's Table IV layout");
  if (d->precision != SP_MLP_FP32 && d->precision != SP_MLP_BF16 && d->precision != SP_MLP_FP16)
    return fail(ctx, SP_E_ARG, "sp_load_model: unknown precision");
  // bf16 operands (8-bit mantissa) measured a 3e-2 max latency error against the fp64
  // oracle with seeded weights, outside north_star's 1e-2 for a 16-bit MLP: refused.
  if (d->precision == SP_MLP_BF16)
    return fail(ctx, SP_E_UNSUPPORTED,
                "sp_load_model: SP_MLP_BF16 misses the 1e-2 latency bar (measured 3e-2); use SP_MLP_FP16");
  const float *arrs[] = {d->mu, d->sigma, d->w1, d->b1, d->g1, d->be1, d->m1, d->v1, d->w2, d->b2, d->g2,
                         d->be2, d->m2, d->v2, d->w3, d->b3, d->g3, d->be3, d->m3, d->v3, d->w4};
  const size_t lens[] = {(size_t)n_in, (size_t)n_in, 256u * n_in, 256, 256, 256, 256, 256, 128 * 256, 128,
                         128, 128, 128, 128, 64 * 128, 64, 64, 64, 64, 64, 64};
  for (int k = 0; k < 21; ++k) {
    if (!arrs[k]) return fail(ctx, SP_E_ARG, "sp_load_model: NULL weight pointer");
    if (!all_finite(arrs[k], lens[k])) return fail(ctx, SP_E_DATA, "sp_load_model: non-finite value");
  }
  if (!std::isfinite(d->b4) || !(d->bn_eps > 0) || !std::isfinite(d->bn_eps))
    return fail(ctx, SP_E_DATA, "sp_load_model: bad b4 or bn_eps");
  const float *vs[3] = {d->v1, d->v2, d->v3};
  const int W[3] = {256, 128, 64};
  for (int l = 0; l < 3; ++l)
    for (int i = 0; i < W[l]; ++i)
      if (!((double)vs[l][i] + (double)d->bn_eps > 0))
        return fail(ctx, SP_E_DATA, "sp_load_model: BatchNorm variance + eps must be > 0");

  // BN(eval) after ReLU as a per-unit affine: s = gamma / sqrt(var + eps),
  // t = beta - s * mean (R18), computed in fp64.
  std::vector<double> s[3], t[3];
  const float *gs[3] = {d->g1, d->g2, d->g3}, *bes[3] = {d->be1, d->be2, d->be3},
              *ms[3] = {d->m1, d->m2, d->m3};
  for (int l = 0; l < 3; ++l) {
    s[l].resize(W[l]);
    t[l].resize(W[l]);
    for (int i = 0; i < W[l]; ++i) {
      s[l][i] = (double)gs[l][i] / std::sqrt((double)vs[l][i] + (double)d->bn_eps);
      t[l][i] = (double)bes[l][i] - s[l][i] * (double)ms[l][i];
    }
  }
  std::unique_ptr<sp_model> m(new (std::nothrow) sp_model);
  if (!m) return fail(ctx, SP_E_INTERNAL, "sp_load_model: out of host memory");
  m->family = d->family;
  m->n_in = n_in;
  m->precision = d->precision;

  // fp32 layout (always built: it is also the reference layout of the bf16 pack)
  {
    std::vector<float> buf;
    auto push = [&](size_t n) { size_t o = buf.size(); buf.resize(o + ((n + 3) & ~size_t(3)), 0.f); return o; };
    const size_t o_w1t = push(256u * n_in), o_w2t = push(256 * 128), o_w3t = push(128 * 64);
    const size_t o_v[9] = {push(256), push(256), push(256), push(128), push(128), push(128), push(64), push(64), push(64)};
    const size_t o_w4 = push(64), o_mu = push(16), o_is = push(16);
    for (int k = 0; k < n_in; ++k)
      for (int n = 0; n < 256; ++n) buf[o_w1t + k * 256 + n] = d->w1[n * n_in + k];
    for (int k = 0; k < 256; ++k)
      for (int n = 0; n < 128; ++n) buf[o_w2t + k * 128 + n] = d->w2[n * 256 + k];
    for (int k = 0; k < 128; ++k)
      for (int n = 0; n < 64; ++n) buf[o_w3t + k * 64 + n] = d->w3[n * 128 + k];
    const float *bs[3] = {d->b1, d->b2, d->b3};
    for (int l = 0; l < 3; ++l)
      for (int i = 0; i < W[l]; ++i) {
        buf[o_v[3 * l] + i] = bs[l][i];
        buf[o_v[3 * l + 1] + i] = (float)s[l][i];
        buf[o_v[3 * l + 2] + i] = (float)t[l][i];
      }
    for (int i = 0; i < 64; ++i) buf[o_w4 + i] = d->w4[i];
    for (int i = 0; i < n_in; ++i) {
      buf[o_mu + i] = d->mu[i];
      buf[o_is + i] = (float)(1.0 / std::max((double)d->sigma[i], 1e-8));
    }
    cudaError_t e = m->fp32.alloc_copy(buf.data(), buf.size() * 4);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "sp_load_model: upload");
    const float *base = (const float *)m->fp32.p;
    MlpFp32 &q = m->m32;
    q.w1t = base + o_w1t; q.w2t = base + o_w2t; q.w3t = base + o_w3t;
    q.b1 = base + o_v[0]; q.s1 = base + o_v[1]; q.t1 = base + o_v[2];
    q.b2 = base + o_v[3]; q.s2 = base + o_v[4]; q.t2 = base + o_v[5];
    q.b3 = base + o_v[6]; q.s3 = base + o_v[7]; q.t3 = base + o_v[8];
    q.w4 = base + o_w4; q.mu = base + o_mu; q.inv_sigma = base + o_is;
    q.b4 = d->b4;
    q.n_in = n_in;
    q.family = d->family;
  }
  if (d->precision == SP_MLP_FP16) {
    std::vector<uint16_t> wpack;
    std::vector<float> vecs;
    float b4 = 0.f;
    m->m16.bf16 = 0;
    const int pk = pack_mlp_16bit(*d, s, t, false, wpack, vecs, b4);
    if (pk == 1) return fail(ctx, SP_E_UNSUPPORTED, "sp_load_model: tcgen05 path unavailable in this build");
    if (pk == 2)  // W' = W diag(gamma/sqrt(var+eps)) past +-65504 (e.g. a tiny BN variance)
      return fail(ctx, SP_E_DATA,
                  "sp_load_model: a BN-folded weight or bias exceeds the fp16 range (|v| > 65504); use SP_MLP_FP32");
    cudaError_t e = m->bf16w.alloc_copy(wpack.data(), wpack.size() * 2);
    if (e == cudaSuccess) e = m->bf16v.alloc_copy(vecs.data(), vecs.size() * 4);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "sp_load_model: bf16 upload");
    m->m16.wpack = m->bf16w.p;
    m->m16.vecs = (const float *)m->bf16v.p;
    m->m16.b4 = b4;
    m->m16.n_in = n_in;
    m->m16.family = d->family;
  }
  *out = m.release();
  return SP_OK;
}

extern "C" void sp_free_model(sp_model *model) { delete model; }

// ------------------------------------------------------------------ predict

extern "C" sp_status sp_predict(sp_ctx *ctx, const sp_model *model, const sp_features *in, float *latency_us,
                                float *efficiency, void *stream) {
  if (!ctx) return fail(nullptr, SP_E_ARG, "sp_predict: ctx is NULL");
  if (!model || !in) return fail(ctx, SP_E_ARG, "sp_predict: NULL argument");
  if (in->family != model->family) return fail(ctx, SP_E_ARG, "sp_predict: features/model family mismatch");
  if (in->n_pairs < 0 || in->ld < in->n_pairs) return fail(ctx, SP_E_ARG, "sp_predict: bad n_pairs / ld");
  if (in->n_pairs == 0) return SP_OK;
  if (!latency_us || !in->ints || !in->flts || !in->status)
    return fail(ctx, SP_E_ARG, "sp_predict: NULL buffer");
  ctx->err.clear();
  cudaSetDevice(ctx->device);
  int e;
  const LaunchHook h = ctx->hook();
  if (model->precision == SP_MLP_FP16) {
    h.on_begin("predict_tcgen05", stream);
    e = launch_predict_tcgen05(model->m16, *in, latency_us, efficiency, ctx->num_sms, stream);
  } else {
    h.on_begin("predict_simt", stream);
    e = launch_predict_simt(model->m32, *in, latency_us, efficiency, ctx->num_sms, stream);
  }
  h.on_end(stream);
  if (e) return cuda_fail(ctx, e, "sp_predict: launch");
  return SP_OK;
}

// ------------------------------------------------------------- accounting

extern "C" sp_status sp_set_profiling(sp_ctx *ctx, int32_t enable) {
  if (!ctx) return fail(nullptr, SP_E_ARG, "sp_set_profiling: ctx is NULL");
  std::lock_guard<std::mutex> lk(ctx->prof_mu);
  ctx->prof = enable != 0;
  return SP_OK;
}

extern "C" int32_t sp_profile_read(sp_ctx *ctx, sp_kernel_stat *out, int32_t max, int32_t reset) {
  if (!ctx) {
    fail(nullptr, SP_E_ARG, "sp_profile_read: ctx is NULL");
    return -1;
  }
  std::lock_guard<std::mutex> lk(ctx->prof_mu);
  cudaSetDevice(ctx->device);
  int32_t rc = 0;
  for (auto &p : ctx->pending) {
    float ms = 0.f;
    cudaError_t e = cudaEventSynchronize(p.b);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, p.a, p.b);
    if (e != cudaSuccess) {
      cuda_fail(ctx, e, "sp_profile_read");
      rc = -1;
    } else {
      ctx->kstats[p.kernel].ms += ms;
    }
    ctx->ev_pool.push_back(p.a);
    ctx->ev_pool.push_back(p.b);
  }
  ctx->pending.clear();
  if (rc < 0) return rc;
  int32_t n = 0;
  for (auto &kv : ctx->kstats) {
    auto it = ctx->knames.find(kv.first);
    if (it == ctx->knames.end()) it = ctx->knames.emplace(kv.first, strdup(kv.first.c_str())).first;
    if (out && n < max) out[n] = sp_kernel_stat{it->second, kv.second.launches, kv.second.ms};
    ++n;
  }
  if (reset) ctx->kstats.clear();
  return n;
}
