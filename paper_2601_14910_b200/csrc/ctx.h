// Host-side context and helpers shared by the C-ABI translation units
// (api.cu, e2e.cu).  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "sp_internal.h"
#include "synperf.h"

struct sp_ctx {
  using LaunchHook = sp::LaunchHook;
  int device = 0;
  int num_sms = 0;
  int *counters = nullptr;  // DEVICE work counters of the attention kernel (kAttnMaxGroups)
  void *attn_res = nullptr;  // DEVICE per-config attention results (AttnResults), grow-only
  size_t attn_res_bytes = 0;
  void *pre = nullptr;  // DEVICE config pre-pass of the fused path (kPreFields u64 per config), grow-only
  size_t pre_bytes = 0;
  std::string err;
  // sp_predict_host (host.cu): grow-only device staging, two copy streams, events
  struct HostBuf {
    void *p = nullptr;
    size_t bytes = 0;
    cudaError_t need(size_t n) {
      if (n <= bytes) return cudaSuccess;
      if (p) cudaFree(p);
      p = nullptr;
      bytes = 0;
      cudaError_t e = cudaMalloc(&p, n);
      if (e == cudaSuccess) bytes = n;
      else p = nullptr;
      return e;
    }
    ~HostBuf() {
      if (p) cudaFree(p);
    }
  };
  HostBuf h_fields, h_ragged, h_roff, h_feats, h_lat[2], h_flag;
  cudaStream_t h_h2d = nullptr, h_d2h = nullptr;
  std::vector<cudaEvent_t> h_events;  // sync-only events, reused across calls
  // kernel accounting (sp_set_profiling / sp_profile_read)
  struct KStat {
    int64_t launches = 0;
    double ms = 0;
  };
  struct Pending {
    const char *kernel;
    cudaEvent_t a, b;
  };
  bool prof = false;
  std::mutex prof_mu;
  std::map<std::string, KStat> kstats;
  std::map<std::string, const char *> knames;  // stable name strings
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> ev_pool;
  const char *open_kernel = nullptr;
  cudaEvent_t open_ev = nullptr;
  ~sp_ctx() {
    if (h_h2d) cudaStreamDestroy(h_h2d);
    if (h_d2h) cudaStreamDestroy(h_d2h);
    for (auto e : h_events) cudaEventDestroy(e);
    if (counters) cudaFree(counters);
    if (attn_res) cudaFree(attn_res);
    if (pre) cudaFree(pre);
    for (auto &p : pending) {
      cudaEventDestroy(p.a);
      cudaEventDestroy(p.b);
    }
    for (auto e : ev_pool) cudaEventDestroy(e);
    for (auto &kv : knames) free(const_cast<char *>(kv.second));
  }
  cudaEvent_t event() {
    if (!ev_pool.empty()) {
      cudaEvent_t e = ev_pool.back();
      ev_pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    return e;
  }
  static void hook_begin(void *self, const char *kernel, void *stream) {
    sp_ctx *c = static_cast<sp_ctx *>(self);
    std::lock_guard<std::mutex> lk(c->prof_mu);
    ++c->kstats[kernel].launches;
    c->open_kernel = kernel;
    c->open_ev = nullptr;
    if (c->prof && (c->open_ev = c->event()) != nullptr)
      cudaEventRecord(c->open_ev, reinterpret_cast<cudaStream_t>(stream));
  }
  static void hook_end(void *self, void *stream) {
    sp_ctx *c = static_cast<sp_ctx *>(self);
    std::lock_guard<std::mutex> lk(c->prof_mu);
    if (!c->open_ev) return;
    cudaEvent_t b = c->event();
    if (!b) return;
    cudaEventRecord(b, reinterpret_cast<cudaStream_t>(stream));
    c->pending.push_back({c->open_kernel, c->open_ev, b});
    c->open_ev = nullptr;
  }
  LaunchHook hook() { return LaunchHook{&hook_begin, &hook_end, this}; }
};

namespace sp {

extern thread_local std::string g_noctx_err;

struct DevBuf {
  void *p = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf &) = delete;
  DevBuf &operator=(const DevBuf &) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc_copy(const void *host, size_t bytes) {
    cudaError_t e = cudaMalloc(&p, bytes ? bytes : 16);
    if (e != cudaSuccess) { p = nullptr; return e; }
    if (bytes) e = cudaMemcpy(p, host, bytes, cudaMemcpyHostToDevice);
    return e;
  }
};

inline sp_status fail(sp_ctx *ctx, sp_status st, const std::string &msg) {
  if (ctx) ctx->err = msg;
  else g_noctx_err = msg;
  return st;
}

inline sp_status cuda_fail(sp_ctx *ctx, int e, const char *what) {
  return fail(ctx, SP_E_INTERNAL, std::string(what) + ": " + cudaGetErrorString((cudaError_t)e));
}

}  // namespace sp
