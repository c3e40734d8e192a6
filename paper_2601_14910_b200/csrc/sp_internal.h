// Internal declarations shared by the host API (api.cu) and the kernels.
// Not part of the ABI.
#pragma once

#include <cstdint>
#include <vector>

#include "synperf.h"

namespace sp {

constexpr int kNumInts = 11;
constexpr int kNumFlts = 12;

// Slot indices of the uniform feature record (include/synperf.h sp_features).
enum IntSlot { I_NTASKS, I_OCC, I_WAVES, I_TOT_T, I_TOT_F, I_TOT_X, I_MAX_T, I_MAX_F, I_MAX_X,
               I_BYTES, I_BYTES_MAX };
enum FltSlot { F_CG_T, F_CG_F, F_CG_X, F_CS_T, F_CS_F, F_CS_X, F_GLOB_G, F_L2_G, F_GLOB_S,
               F_L2_S, F_SMEM_S, F_TTHEORY };

// Pipes per family (Table V): bit 0 Tensor, bit 1 FMA, bit 2 XU.
__host__ __device__ inline int family_pipes(int fam) {
  return (fam == SP_GEMM || fam == SP_FUSED_MOE || fam == SP_SCALED_MM || fam == SP_GEMM_SPLITK)
             ? 1
             : (fam == SP_ATTENTION ? 5 : 6);
}

// Step a1: per-spec constants derived once on the host in fp64 (Eq.4-5).
// 128-byte aligned so a warp reads one spec in a single pass.
struct alignas(16) DevSpec {
  int32_t num_sms;       // N_SM
  int32_t smem_per_sm;   // bytes
  int32_t regs_per_sm;   // 32-bit registers (R6)
  int32_t max_warps;
  int32_t max_ctas;
  int32_t tensor_ok[3];  // tensor rate present for {bf16, fp16, fp8}
  double cg_tensor[3];   // 1 / (N_SM * Th_tensor)   (Eq.5)
  double cs_tensor[3];   // 1 / Th_tensor           (Eq.4)
  double cg_fma, cs_fma, cg_xu, cs_xu;
  double glob_g;         // f / (BW_glob * 1e3): bytes -> cycles at GPU level (R8)
  double l2_g;
  double glob_s;         // f * N_SM / (BW_glob * 1e3): per-SM share BW/N_SM (R8)
  double l2_s;
  double smem_s;         // 1 / smem bytes per clk
  double inv_f;          // 1 / f (cycles -> us)
};
static_assert(sizeof(DevSpec) == 160, "DevSpec layout");

// Device feature-record view.
struct FeatOut {
  int64_t *ints;
  float *flts;
  uint8_t *status;
  int64_t ld;
};

struct ConfigView {
  const int32_t *fields;
  const int32_t *ragged;
  const int64_t *ragged_off;
  int64_t n_configs;
  int64_t ld;
};

// -------------------------------------------------------------- launchers
// All return cudaError_t cast to int (0 = success).

// Uniform families (GEMM, fused MoE, RMSNorm, SiLU&Mul): closed-form schedule.
// Fused featurize -> predict (uniform families GEMM, fused MoE, RMSNorm,
// SiLU&Mul, Scaled MM; SURVEY §8(b) "fused"): the spec-independent part of each
// config, u64 SoA [kPreFields][ldc]:
//   0 status | range_bad << 8 | (tensor dtype + 1) << 16 | T << 32
//   1..4 per-task Tensor, FMA, XU ops, bytes (totals = T x these; range-checked here)
//   5 smem per task (clamped to 32 bits) | warps << 32      6 regs
constexpr int kPreFields = 7;
int launch_uniform_prepass(int family, const ConfigView &cfg, uint64_t *pre, int64_t ldc, void *stream);

// Clamped edge tiles (NEXT-4), GEMM and fused MoE; warp per pair.
// Clamped edge tiles for attention (NEXT-4): warp per pair, every task walked.
int launch_attention_clamped(const ConfigView &cfg, const DevSpec *specs, int spec_begin, int n_specs,
                             int64_t n_pairs, const int64_t *cfg_idx, const int32_t *spec_idx, int max_sms,
                             const FeatOut &out, int num_device_sms, void *stream);
int launch_featurize_clamped(int family, const ConfigView &cfg, const DevSpec *specs, int spec_begin, int n_specs,
                             int64_t n_pairs, const int64_t *cfg_idx, const int32_t *spec_idx, int max_sms,
                             const FeatOut &out, int num_device_sms, void *stream);
int launch_featurize_uniform(int family, const ConfigView &cfg, const DevSpec *specs,
                             int spec_begin, int spec_end, int64_t n_pairs, const int64_t *cfg_idx,
                             const int32_t *spec_idx, const FeatOut &out, void *stream);

// Attention: per-task loop with per-SM shared-memory accumulators.
// Host-built spec groups for CROSS mode (see featurize_attention.cu).
struct AttnGroup {
  int32_t spec_first;    // index into group_specs
  int32_t n_specs;
  int32_t distinct_first;  // index into distinct_n / distinct_off
  int32_t n_distinct;
};
// per-warp shared memory after the accumulators: the request scratch (7 x 32 words)
constexpr int kAttnScratchWords = 224;
// Lazy residue wrap (featurize_attention.cu accumulate): every accumulator
// region has kAttnSlack words past its N; the non-atomic path needs N >= 64.
constexpr int kAttnSlack = 32;
constexpr int kAttnLazyMinN = 64;
constexpr int kAttnMaxGroups = 4096;  // work counters per launch (sp_ctx scratch)
struct AttnPlan {
  const AttnGroup *groups;     // DEVICE [n_groups]
  const int32_t *group_specs;  // DEVICE spec index (absolute)
  const int32_t *spec_dist;    // DEVICE, per group_specs entry: distinct slot (absolute)
  const int32_t *distinct_n;   // DEVICE N_SM of each distinct slot
  const int32_t *distinct_off; // DEVICE word offset of the slot in the warp's smem region
  int32_t n_groups;
  int32_t words_per_warp;      // u32 accumulator words per warp
  const int32_t *host_nd;      // HOST [n_groups]: distinct count per group (kernel template)
  const uint8_t *host_small;   // HOST [n_groups]: group holds an SM count < kAttnLazyMinN (atomic path)
  int *counters;               // DEVICE [n_groups] work counters (context scratch, zeroed per launch)
  const int32_t *spec_slot;    // DEVICE, per spec of the range: its distinct slot (absolute)
  int32_t n_slots;             // distinct slots over all groups
  int32_t min_n;               // smallest SM count of the range (attn_prepass's sparse rule)
};
// Per-config results of the schedule kernel (context scratch, cross mode):
// st/L/U [C], mS/mB [n_slots][ld].
struct AttnResults {
  int32_t *st;
  int64_t *L;
  uint64_t *U;
  int64_t *mS, *mB;
  int64_t ld;
  uint32_t *pre;  // attn_prepass record [kAttnPreWords][ld]: flags, g, FastDiv (m, s) of g, BKV, BQ, chunk
  int8_t *chunk_b;  // [ld / 32] cost class of each chunk of 32 configs: floor(log2 of its task-count sum), -1 none
  int32_t *order;   // [ld / 32] the chunks with warp work, heaviest class first (attn_order)
  int *hist;        // DEVICE [2 kAttnCostBuckets]: chunks per class, then scatter cursors (zeroed per launch)
};
constexpr int kAttnPreWords = 10;
// The schedule kernel takes its chunks of 32 configs heaviest cost class first:
// per-config cost is heavy-tailed (cfg2: T up to ~2e5 tasks, mean ~2.4e3), and
// in input order the last configs drawn by the warps leave a tail of a few busy
// warps (cfg2 featurize measured 3.33 ms in the bench's shuffled order, 3.10 ms
// with the configs grouped by floor(log2 T) descending on the host, 3.88 ms
// lightest first).
constexpr int kAttnCostBuckets = 32;
// ctx->counters: [work counters: n_groups][bucket counts + cursors: 2 kAttnCostBuckets]
constexpr int kAttnCounterInts = kAttnMaxGroups + 2 * kAttnCostBuckets;
// Optional per-launch hook (kernel accounting, sp_set_profiling): begin/end
// bracket one kernel launch on the launch stream.
struct LaunchHook {
  void (*begin)(void *self, const char *kernel, void *stream);
  void (*end)(void *self, void *stream);
  void *self;
  void on_begin(const char *k, void *st) const { if (begin) begin(self, k, st); }
  void on_end(void *st) const { if (end) end(self, st); }
};
// emit = false (cross mode, the fused path): no attn_emit_cross; the planner's pairs are still written.
int launch_featurize_attention(const ConfigView &cfg, const DevSpec *specs, int spec_begin, int spec_end,
                               int n_specs, const AttnPlan &plan, const AttnResults &res, int64_t n_pairs,
                               const int64_t *cfg_idx, const int32_t *spec_idx, int32_t max_sms,
                               const FeatOut &out, int num_device_sms, void *stream, const LaunchHook &hook,
                               bool emit = true);

// Attention under SP_SCHED_GREEDY / SP_SCHED_MINHEAP: warp per pair, sequential
// scheduler simulation (CROSS when cfg_idx == nullptr, else LIST).  max_targets =
// largest SM count (GREEDY) or SM count x max CTAs/SM (MINHEAP) over the specs.
int launch_attention_sim(int mode, const ConfigView &cfg, const DevSpec *specs, int spec_begin, int spec_end,
                         int n_specs, int64_t n_pairs, const int64_t *cfg_idx, const int32_t *spec_idx,
                         int64_t max_targets, const FeatOut &out, int num_device_sms, void *stream,
                         const LaunchHook &hook);
int64_t attention_sim_smem_bytes(int64_t max_targets);  // per warp

// MLP predictor.
struct MlpFp32 {        // DEVICE pointers, fp32
  const float *w1t;     // [n_in][256]  (transposed: k-major)
  const float *w2t;     // [256][128]
  const float *w3t;     // [128][64]
  const float *b1, *s1, *t1;  // bias, BN scale gamma/sqrt(var+eps), BN shift beta - scale*mean
  const float *b2, *s2, *t2;
  const float *b3, *s3, *t3;
  const float *w4;      // [64]
  const float *mu, *inv_sigma;  // [n_in]
  float b4;
  int32_t n_in;
  int32_t family;
};
int launch_predict_simt(const MlpFp32 &m, const sp_features &in, float *latency, float *eff,
                        int num_device_sms, void *stream);

struct MlpBf16 {  // tcgen05 path, 16-bit operands (bf16 or fp16)
  int32_t bf16;         // 1: bf16 operands, 0: fp16 operands
  const void *wpack;    // DEVICE packed 16-bit weights in the UMMA canonical layout (predict_tcgen05.cu)
  const float *vecs;    // DEVICE fp32 vectors: b2'[128], b3'[64], w4'[64], ln2/sigma[16], -mu/sigma[16]
  float b4;
  int32_t n_in;
  int32_t family;
};
// Host: BN-folded bf16 weights in the kernel's shared-memory image, plus fp32
// vectors.  s[l], t[l]: BN(eval) affine of hidden layer l (fp64).  Returns
// 0 on success, 1 if the tcgen05 path is not available (n_in), 2 if a folded
// weight rounds to +-inf in the 16-bit format or an fp32 vector is not finite.
int pack_mlp_16bit(const sp_mlp_desc &d, const std::vector<double> *s, const std::vector<double> *t, bool bf16,
                   std::vector<uint16_t> &wpack, std::vector<float> &vecs, float &b4);
int launch_predict_tcgen05(const MlpBf16 &m, const sp_features &in, float *latency, float *eff,
                           int num_device_sms, void *stream);
// The fused kernel: producers derive each pair's record from the pre-pass and
// its spec (writing `out`, the same bytes sp_featurize writes), then the MLP
// runs as in sp_predict.  Pairs: CROSS, p = (g - g0) * C + c.
struct FusedIn {
  const uint64_t *pre;
  int64_t ldc;
  int64_t C;
  int64_t n_specs;  // spec_end - spec_begin
  double inv_c;     // 1 / C (set by the launcher)
  uint32_t ns_m, ns_s;  // FastDiv constants of n_specs (set by the launcher)
  int cmajor;       // config-major tile order (large pre-pass, see predict_tcgen05.cu)
  int g0;
  const DevSpec *specs;
  FeatOut out;
  int64_t n_pairs;
  // attention (FAM = SP_ATTENTION): per spec of the range its distinct slot, and the
  // schedule kernel's per-(slot, config) class maxima (lo, hi) [n_slots][lohi_ld]
  const int32_t *slot;
  const int64_t *lo, *hi;
  int64_t lohi_ld;
};
// Attention pre-pass of the fused path (thread per config; after attn_schedule_cross
// and attn_planner_cross), u64 SoA [kPreFields][ldc]:
//   0 status | range_bad << 8 | planner << 9 | (tensor dtype + 1) << 16 | T << 32
//   1 total Tensor ops  2 total XU ops  3 total load bytes
//   4 BQ | BKV << 32    5 smem per task | warps << 32    6 regs | head dim << 32
// planner = kv_chunk -1: its records are attn_planner_cross's, read back.
int launch_attn_fuse_prep(const ConfigView &cfg, const AttnResults &res, uint64_t *pre, int64_t ldc, void *stream);
int launch_predict_tcgen05_fused(const MlpBf16 &m, const FusedIn &fi, float *latency, float *eff,
                                 int num_device_sms, void *stream);

}  // namespace sp
