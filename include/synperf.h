/*
 * synperf.h -- C-ABI of libsynperf.so, the B200-native batched SynPerf predictor.
 *
 * SynPerf (arXiv 2601.14910) predicts a kernel's latency on a GPU in two
 * stages (§IV):
 *   1. an analytical feature stage -- Kernel Decomposer F (Eq.1),
 *      Scheduling Simulator M (Eq.2) and Feature Analyzer (Eq.3-5,
 *      P:334-357) -- producing the Table IV feature vector;
 *   2. a per-kernel-category MLP mapping the features to an
 *      execution efficiency e in (0,1); latency = t_theory / e.
 * This library evaluates both stages for every (kernel config x GPU spec)
 * pair of a batch, on the GPU, in hand-written sm_100a kernels.
 *
 * Conventions
 *  - Plain C types only.  Pointers documented DEVICE must be CUDA device
 *    memory of the context's device (e.g. torch tensors' data_ptr()); HOST
 *    pointers are ordinary host memory and are only read during the call.
 *  - `stream` arguments are cudaStream_t passed as void* (NULL = legacy
 *    default stream).  sp_featurize / sp_predict / sp_featurize_predict are
 *    asynchronous on that stream.  They use CONTEXT-OWNED device scratch --
 *    the attention schedule plan of a spec range (built and uploaded with a
 *    synchronous copy the first time the range is seen), the attention
 *    per-config results and the fused pass's config pre-pass (grow-only:
 *    a call with more configs than any before reallocates).  Hence:
 *      * calls on one context must be serialized on one stream (two streams
 *        sharing a context would race on that scratch; use one context per
 *        stream for concurrency);
 *      * a call that builds a plan or grows scratch allocates and
 *        synchronizes: call sp_prepare first (or make one warm-up call at
 *        the largest size) to make the following calls allocation-free and
 *        safe to capture in a CUDA graph.
 *  - No exception crosses the ABI and the library never aborts.  Every call
 *    returns an sp_status; sp_last_error() describes the last failure (or
 *    the last warning) of a context.  There is no CPU fallback: without a
 *    usable sm_100 device, sp_create fails.
 *  - Readings of passages where the paper is silent or ambiguous are listed
 *    as R1..R25 (feature stage), E1..E9 (end-to-end composition) and T1..T9
 *    (estimator training) in DESIGN.md §3, §3b and §3c, and cited below as such.
 */
#ifndef SYNPERF_H_
#define SYNPERF_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */

typedef enum sp_status {
  SP_OK = 0,
  SP_E_ARG = 1,         /* bad argument: NULL, size, family mismatch (SPEC S:604 exit 1) */
  SP_E_DATA = 2,        /* invalid data: spec or model values (SPEC S:604 exit 2) */
  SP_E_INTERNAL = 3,    /* CUDA error or launch failure (SPEC S:604 exit 3) */
  SP_E_UNSUPPORTED = 4  /* valid but not implemented (e.g. scheduler state beyond shared memory) */
} sp_status;

/* Per-pair status written by sp_featurize (one byte per pair).  A pair with a
 * nonzero status has all int slots = -1 and all float slots = NaN; the batch
 * still succeeds.  Domain rules: SPEC S:103 (nh divisible by nkv, histogram
 * sums to M*topk), S:121 (dimensions >= 1), causal requires kvlen >= qlen;
 * exact-integer range R22. */
typedef enum sp_pair_status {
  SP_PAIR_OK = 0,
  SP_PAIR_E_DIM = 1,     /* a problem dimension < 1 (or attention config without requests) */
  SP_PAIR_E_TILE = 2,    /* a tile / block / stage field < 1 (kv_chunk < 0) */
  SP_PAIR_E_HEADS = 3,   /* nh % nkv != 0 */
  SP_PAIR_E_HIST = 4,    /* MoE histogram: negative count or sum != M*topk */
  SP_PAIR_E_CAUSAL = 5,  /* causal attention request with kvlen < qlen */
  SP_PAIR_E_RES = 6,     /* warps < 1, regs < 1 or smem < 0 */
  SP_PAIR_E_DTYPE = 7,   /* dtype not supported by the family, or spec lacks that tensor rate */
  SP_PAIR_E_RANGE = 8,   /* a total >= 2^63 (does not fit the int64 record, R22), or past the
                            kernels' 32-bit working range: T >= 2^31, per-kv-head sum
                            kv_eff/BKV >= 2^32, M*topk >= 2^31 or qlen*g >= 2^31 (an
                            implementation limit, not the paper's: the oracle answers there) */
  SP_PAIR_E_INDEX = 9    /* SP_PAIRS_LIST entry with a config or spec index out of range */
} sp_pair_status;

/* ---------------------------------------------------------------- families */

/* Kernel categories of Table V. */
typedef enum sp_family {
  SP_GEMM = 0,       /* cuBLAS GEMM, Tensor pipe */
  SP_ATTENTION = 1,  /* FlashInfer FA2 prefill/decode, Tensor + XU */
  SP_FUSED_MOE = 2,  /* SGLang fused MoE (Triton), Tensor */
  SP_RMSNORM = 3,    /* FlashInfer RMSNorm, FMA + XU */
  SP_SILU_MUL = 4,   /* FlashInfer SiLU&Mul, FMA + XU */
  SP_SCALED_MM = 5,  /* vLLM FP8 Scaled MM, block-wise quantisation, Tensor */
  SP_GEMM_SPLITK = 6 /* cuBLAS split-K GEMM (tiling reverse-engineered from profiles, P:270;
                        SURVEY 8(f) NEXT-4), Tensor; reading R25 */
} sp_family;

typedef enum sp_dtype { SP_BF16 = 0, SP_FP16 = 1, SP_FP32 = 2, SP_FP8 = 3 } sp_dtype;

/*
 * Config fields, int32, one row per field (structure of arrays), in this
 * order per family.  The generator workloads/gen.py FIELDS uses the same order.
 *
 * SP_GEMM (11):      M, N, K, TM, TN, BK, STAGES, WARPS, REGS, SMEM, DTYPE
 * SP_ATTENTION (12): BS, NH, NKV, HD, BQ, BKV, KV_CHUNK, CAUSAL, WARPS, REGS, SMEM, DTYPE
 *                    ragged: 2*BS int32 per config, (qlen, kvlen) interleaved
 *                    KV_CHUNK: 0 unsplit, > 0 split-KV chunk (R12), -1 the split-KV
 *                    planner picks it per spec (non-causal only; reading R24: the
 *                    smallest multiple of 16 whose work items nkv * sum_b nqb_b *
 *                    ceil(kvlen_b / chunk) fit N_SM x occupancy, unsplit if none needed)
 * SP_FUSED_MOE (14): M, E, TOPK, H, N, BM, BN, BK, GROUP_M, STAGES, WARPS, REGS, SMEM, DTYPE
 *                    ragged: E int32 per-expert token counts; ragged_off = -1 means
 *                    the balanced split q + [e < r], q = M*TOPK / E, r = M*TOPK % E (R16)
 * SP_RMSNORM (6):    SEQ, DIM, WARPS, REGS, SMEM, DTYPE
 * SP_SILU_MUL (6):   SEQ, DIM, WARPS, REGS, SMEM, DTYPE   (DIM = output width, R15)
 * SP_SCALED_MM (11): M, N, K, TM, TN, BK, STAGES, WARPS, REGS, SMEM, DTYPE (= SP_FP8)
 *                    GEMM's tiling (Table V lists the Tensor pipe only) with
 *                    FP8 operands at the spec's th_tensor_fp8 and block-wise scales
 *                    (reading R23): per task, A scales tm x ceil(K/128) and B scales
 *                    ceil(tn/128) x ceil(K/128), fp32 each, on top of (tm+tn) x K_pad
 *                    one-byte operands.  A spec without an FP8 tensor rate (sm_80/86)
 *                    gives SP_PAIR_E_DTYPE.
 * SP_GEMM_SPLITK (12): M, N, K, TM, TN, BK, SPLIT_K, STAGES, WARPS, REGS, SMEM, DTYPE
 *                    reading R25: the kt = ceil(K/BK) k-tiles are cut into slices of
 *                    kps = ceil(kt/SPLIT_K) k-tiles; S' = ceil(kt/kps) <= SPLIT_K
 *                    non-empty slices, the last one holding kt - (S'-1)*kps.  Tasks
 *                    are (slice z, tile i, tile j) with z outermost (cuBLAS's grid z,
 *                    dispatched last), tiles row-major: T = S' * ceil(M/TM) * ceil(N/TN);
 *                    task (z,.,.) = padded TM x TN x (k_z*BK) tile (Tensor 2*TM*TN*k_z*BK,
 *                    bytes (TM+TN)*k_z*BK*bpe).  The fp32 partial-tile reduction is a
 *                    separate kernel and is excluded (as the split-KV merge, R12).
 *
 * SMEM = per-task shared memory bytes, 0 = default footprint.
 * GROUP_M does not change any feature under cyclic dealing (it only permutes
 * uniform tiles); it is accepted for completeness of the Triton knob set.
 */
enum {
  SP_NFIELDS_GEMM = 11, SP_NFIELDS_ATTENTION = 12, SP_NFIELDS_FUSED_MOE = 14,
  SP_NFIELDS_RMSNORM = 6, SP_NFIELDS_SILU_MUL = 6, SP_NFIELDS_SCALED_MM = 11,
  SP_NFIELDS_GEMM_SPLITK = 12
};

/* -------------------------------------------------------------- hardware S */

/*
 * Hardware specification S: the Table II parameter vector of one
 * GPU.  Values for the paper's 11 GPUs are in Table VI plus the
 * fills of R19.  112 bytes, natural alignment (workloads/specs.py SPEC_DTYPE).
 */
typedef struct sp_gpu_spec {
  char name[32];
  int32_t cc_major, cc_minor;       /* compute capability, 8.0 - 12.0 */
  int32_t num_sms;                  /* N_SM, 78 - 188 */
  int32_t th_tensor_bf16;           /* Tensor pipe, ops/clk/SM, 512 - 4096 */
  int32_t th_tensor_fp16;
  int32_t th_tensor_fp8;            /* 0 = absent */
  int32_t th_fma;                   /* FMA pipe, ops/clk/SM, 64 - 128 */
  int32_t th_xu;                    /* XU pipe, ops/clk/SM, 16 */
  int32_t smem_bw_bytes_per_clk;    /* shared memory bandwidth per SM, 128 */
  int32_t smem_per_sm_bytes;        /* 100 - 228 KB */
  int32_t regfile_per_sm_bytes;     /* 256 KB */
  int32_t max_warps_per_sm;         /* occupancy limit (not in Table II) */
  int32_t max_ctas_per_sm;          /* occupancy limit */
  int32_t reserved_;
  double sm_clock_mhz;              /* f, 1410 - 2520 MHz */
  double bw_global_gbps;            /* BW_glob, 696 - 4916 GB/s (GB = 1e9 B) */
  double bw_l2_gbps;                /* BW_L2, 2430 - 10400 GB/s */
} sp_gpu_spec;

/* ----------------------------------------------------------------- batches */

typedef struct sp_config_batch {
  int32_t family;             /* sp_family */
  int32_t n_fields;           /* must equal SP_NFIELDS_<family> */
  int64_t n_configs;          /* C >= 0 */
  int64_t field_ld;           /* elements between field rows, >= n_configs */
  const int32_t *fields;      /* DEVICE int32 [n_fields][field_ld] */
  const int32_t *ragged;      /* DEVICE int32 [n_ragged]; NULL if the family has none */
  const int64_t *ragged_off;  /* DEVICE int64 [n_configs]; offset into ragged, or -1 */
  int64_t n_ragged;
} sp_config_batch;

typedef enum sp_pairing_kind {
  SP_PAIRS_CROSS = 0,  /* specs [spec_begin, spec_end) x all configs, spec-major:
                          pair p = (g - spec_begin) * n_configs + c */
  SP_PAIRS_LIST = 1    /* explicit list: pair p = (cfg_idx[p], spec_idx[p]) */
} sp_pairing_kind;

typedef struct sp_pairing {
  int32_t kind;          /* sp_pairing_kind */
  int32_t spec_begin;    /* CROSS */
  int32_t spec_end;      /* CROSS */
  int32_t reserved_;
  int64_t n_pairs;       /* LIST: number of pairs */
  const int64_t *cfg_idx;   /* LIST: DEVICE int64 [n_pairs] */
  const int32_t *spec_idx;  /* LIST: DEVICE int32 [n_pairs] */
} sp_pairing;

/*
 * Feature record per pair (SURVEY §8 uniform record; Table IV),
 * structure of arrays with leading dimension ld (>= n_pairs):
 *   ints[k*ld + p], k = 0..10 (int64):
 *     0 n_tasks T            1 occupancy            2 waves = ceil(T/(N_SM*occ))
 *     3..5 total ops N^GPU_p for p = Tensor, FMA, XU (Eq.5 numerator)
 *     6..8 max-SM ops max_j N^SM_j_p (R7)
 *     9 total load bytes B^GPU    10 max-SM load bytes max_j B^SM_j
 *   flts[k*ld + p], k = 0..11 (fp32):
 *     0..2 C^GPU_p = N^GPU_p / (N_SM Th_p) (Eq.5)   3..5 C^SM_p = max-SM ops / Th_p (Eq.4)
 *     6 C_glob^GPU  7 C_L2^GPU  (B^GPU / BW, cycles at f)
 *     8 C_glob^SM   9 C_L2^SM   (max-SM bytes / (BW/N_SM), R8)   10 C_smem^SM
 *     11 t_theory_us = max(GPU-level roofs of the family) / f (R9)
 *   status[p]: sp_pair_status.
 * Pipes absent from a family (Table V) hold 0.
 */
typedef struct sp_features {
  int32_t family;        /* sp_family of the batch that produced it */
  int32_t reserved_;
  int64_t n_pairs;
  int64_t ld;
  int64_t *ints;         /* DEVICE int64 [11][ld] */
  float *flts;           /* DEVICE fp32 [12][ld] */
  uint8_t *status;       /* DEVICE uint8 [n_pairs] */
} sp_features;

/* ---------------------------------------------------------------- MLP model */

typedef enum sp_precision {
  SP_MLP_FP32 = 0,  /* CUDA-core fp32 path: parity within 1e-5 relative of the fp64 oracle */
  SP_MLP_BF16 = 1,  /* REFUSED by sp_load_model (SP_E_UNSUPPORTED): bf16 operands (8-bit
                       mantissa) measured 3e-2 max latency error vs the fp64 oracle, outside
                       north_star's 1e-2 bar for a 16-bit MLP */
  SP_MLP_FP16 = 2   /* tcgen05/TMEM path, fp16 operands, fp32 accumulate: parity within 1e-2
                       (measured max 5e-3); same dense tensor rate as bf16 */
} sp_precision;

/*
 * Per-kernel-category estimator: 3 hidden layers of 256, 128, 64
 * units, each Linear -> ReLU -> BatchNorm(eval) -> Dropout(identity at eval),
 * then Linear(64 -> 1) -> sigmoid = efficiency (R18).  Inputs are the
 * family's Table IV vector in frozen order (per pipe present, Tensor, FMA, XU:
 * [total ops, C^GPU, max-SM ops, C^SM], then [B^GPU, C_glob^GPU, C_L2^GPU,
 * max-SM B, C_glob^SM, C_L2^SM, C_smem^SM]; 11 or 15 values), normalised as
 * (ln(1+v) - mu) / max(sigma, 1e-8) (R17).  All pointers are HOST fp32,
 * row-major [out][in]; the library copies what it needs.
 */
typedef struct sp_mlp_desc {
  int32_t family;      /* sp_family the model was trained for */
  int32_t n_in;        /* 4 * (#pipes) + 7: 11 (GEMM, MoE, Scaled MM, split-K GEMM) or 15 */
  int32_t precision;   /* sp_precision */
  int32_t reserved_;
  const float *mu, *sigma;              /* [n_in] */
  const float *w1, *b1;                 /* [256][n_in], [256] */
  const float *g1, *be1, *m1, *v1;      /* BN1 gamma, beta, running mean, running var [256] */
  const float *w2, *b2;                 /* [128][256], [128] */
  const float *g2, *be2, *m2, *v2;      /* [128] */
  const float *w3, *b3;                 /* [64][128], [64] */
  const float *g3, *be3, *m3, *v3;      /* [64] */
  const float *w4;                      /* [64] */
  float b4;
  float bn_eps;                         /* BatchNorm epsilon, > 0 (default 1e-5) */
} sp_mlp_desc;

/* ------------------------------------------------------------------ handles */

typedef struct sp_ctx sp_ctx;
typedef struct sp_specs sp_specs;
typedef struct sp_model sp_model;

/* Flags of sp_load_gpu_specs */
#define SP_STRICT 1u  /* reject values outside Table II's ranges; default: warn */

/* ---------------------------------------------------------------------- API */

/* Creates a context on CUDA device `device` (must be sm_100).  Library-owned;
 * one per device.  SP_E_ARG on a bad device, SP_E_UNSUPPORTED if it is not
 * sm_100, SP_E_INTERNAL if CUDA is unusable. */
sp_status sp_create(int device, sp_ctx **out);
void sp_destroy(sp_ctx *ctx);

/* Message of the context's last error or warning ("" if none).  Valid until
 * the next call on that context.  sp_last_error(NULL) reports failures of
 * calls that had no context (sp_create). */
const char *sp_last_error(const sp_ctx *ctx);

/* Version string and the number of SMs of the context's device. */
const char *sp_version(void);
int32_t sp_device_sms(const sp_ctx *ctx);

/*
 * a1 spec staging (Table II).  Copies n HOST records, validates them
 * (SP_E_DATA on num_sms < 1 "invalid SM count", non-positive clock,
 * bandwidth, FMA/XU throughput, smem bandwidth, register file, warps or CTAs
 * (S:39); with SP_STRICT also values outside Table II's ranges --
 * otherwise those set a warning readable through sp_last_error), derives the
 * per-spec constants used by Eq.4-5 and C_mem = B/BW and uploads
 * them.  The handle is immutable and may be shared across streams.
 */
sp_status sp_load_gpu_specs(sp_ctx *ctx, const sp_gpu_spec *host_specs, int32_t n,
                            uint32_t flags, sp_specs **out);
void sp_free_specs(sp_specs *specs);
int32_t sp_specs_count(const sp_specs *specs);

/*
 * Estimator load.  Copies the HOST description, checks
 * n_in == 4*pipes(family)+7 and that every value is finite and sigma, var,
 * bn_eps are sane (SP_E_DATA otherwise), and builds device layouts:
 * SP_MLP_FP32 keeps fp32 weights with BN as a per-unit affine; SP_MLP_FP16
 * folds each BN affine into the next layer (algebraically exact, R18) and
 * packs fp16 weights in the tcgen05 UMMA shared-memory layout.  SP_MLP_BF16
 * returns SP_E_UNSUPPORTED (see sp_precision).  SP_MLP_FP16 returns
 * SP_E_DATA when a folded weight W*diag(gamma/sqrt(var+eps)) or the layer-1
 * bias rounds past the fp16 range (|v| > 65504, e.g. a tiny BN variance);
 * SP_MLP_FP32 accepts such a model.  At predict time the fp16 path converts
 * activations with saturation (cvt.rn.satfinite): an activation past 65504 is
 * clamped to it, never inf/NaN.
 */
sp_status sp_load_model(sp_ctx *ctx, const sp_mlp_desc *desc, sp_model **out);
void sp_free_model(sp_model *model);

/*
 * Feature stage, steps a2..a9: for every pair, decompose the kernel into tasks
 * (Eq.1), deal them round-robin onto the spec's SMs (Eq.2, R5), accumulate
 * per-SM and GPU demands (Eq.3), and derive cycles and t_theory
 * (Eq.4-5, R9).  Writes out->ints/flts/status for out->n_pairs pairs.
 *   cfg:   configs of one family (DEVICE arrays).
 *   specs: from sp_load_gpu_specs.
 *   pairs: CROSS (n_pairs = (spec_end-spec_begin)*n_configs) or LIST.
 *   out:   caller-owned DEVICE SoA; out->family must equal cfg->family and
 *          out->n_pairs the pairing's pair count.
 * EDGE TILES ARE PADDED (reading R2): a partial output tile
 * counts its full tile_M x tile_N x ceil(K/BK)*BK MMA work and loads, as the
 * MMA units execute them (Table VII's 0.01% total-op error vs NCU, P:529-530,
 * is only plausible for executed, i.e. padded, tiles).  This DIFFERS from
 * SPEC's default, which clamps edge tiles to their in-range extent (S:124,
 * S:155): that reading is sp_featurize_ex(.., SP_FEAT_CLAMPED, ..) (GEMM,
 * fused MoE, attention; Scaled MM and split-K GEMM are padded only).
 * Integer slots are exact (bit-identical to the fp64 oracle); float slots are
 * computed in fp64 from the exact integers and rounded once to fp32 (R20).
 * Synchronous errors: SP_E_ARG (NULL, sizes, family/field-count mismatch,
 * spec index range), SP_E_UNSUPPORTED (attention on a spec with > 4096 SMs),
 * SP_E_INTERNAL (launch failure).  Per-pair domain errors go to status[p].
 */
sp_status sp_featurize(sp_ctx *ctx, const sp_config_batch *cfg, const sp_specs *specs,
                       const sp_pairing *pairs, const sp_features *out, void *stream);

/*
 * Reserve the context-owned scratch (see Conventions) for calls of `family`
 * with up to `n_configs` configs over specs [spec_begin, spec_end) (CROSS):
 * builds and uploads the attention schedule plan of that range and grows the
 * attention result / fused pre-pass scratch.  After it, sp_featurize,
 * sp_predict and sp_featurize_predict at those sizes neither allocate nor
 * synchronize (CUDA-graph capturable).  Synchronous.  Errors: SP_E_ARG,
 * SP_E_UNSUPPORTED (as sp_featurize), SP_E_INTERNAL (allocation).
 */
sp_status sp_prepare(sp_ctx *ctx, int32_t family, int64_t n_configs, const sp_specs *specs, int32_t spec_begin,
                     int32_t spec_end);

/*
 * Scheduling Simulator variants ("supporting the two main scheduling
 * paradigms").  sp_featurize uses SP_SCHED_RR.
 *   SP_SCHED_RR      hardware round-robin as cyclic dealing, task t -> SM
 *                    (t mod N_SM) (R5).  Exact for uniform tasks.
 *   SP_SCHED_GREEDY  hardware round-robin with retirement ("a new task
 *                    is assigned to an SM when an existing task finishes";
 *                    SPEC S:183): the first N_SM*occ tasks are dealt
 *                    cyclically, then each task goes to the SM with the least
 *                    accumulated busy time.
 *   SP_SCHED_MINHEAP persistent kernel with a software MinHeap tile scheduler
 *                    (P:281, P:427 FlashInfer FA3): W = min(N_SM*occ,
 *                    T) workers, worker w resident on SM (w mod N_SM); each
 *                    task goes to the worker with the least accumulated busy time.
 * Busy time of a task = max over the family's pipes of ops_p / Th_p;
 * ties go to the lowest SM / worker index.  For the uniform-task
 * families (GEMM, fused MoE, RMSNorm, SiLU&Mul, Scaled MM) all three give the
 * cyclic partition, so they share the closed form.  Split-K GEMM (two task
 * sizes, R25) supports SP_SCHED_RR only (SP_E_UNSUPPORTED otherwise).  Attention under GREEDY / MINHEAP
 * is simulated task by task (one warp per pair): exact, but ~100x slower than
 * SP_SCHED_RR; SP_E_UNSUPPORTED if the scheduler state of the spec range
 * (N_SM, or N_SM x max CTAs/SM, 12 bytes each) exceeds a warp's shared memory.
 */
typedef enum sp_scheduler { SP_SCHED_RR = 0, SP_SCHED_GREEDY = 1, SP_SCHED_MINHEAP = 2 } sp_scheduler;

sp_status sp_featurize_sched(sp_ctx *ctx, const sp_config_batch *cfg, const sp_specs *specs,
                             const sp_pairing *pairs, int32_t scheduler, const sp_features *out,
                             void *stream);

/*
 * Feature-stage options.  sp_featurize_ex(.., scheduler, 0, ..)
 * is sp_featurize_sched.
 *   SP_FEAT_CLAMPED  SPEC's clamped edge tiles, the alternative
 *                    to the padded reading R2: an edge tile of a GEMM (fused
 *                    MoE) computes and loads only its in-range rows and columns,
 *                    ma x na over the exact K (H): Tensor 2*ma*na*K, bytes
 *                    (ma+na)*K*bpe; an attention task only its qr in-range
 *                    query rows over its exact kv length len: Tensor 4*qr*len*hd,
 *                    XU qr*len + qr*ceil(len/BKV), bytes (qr + 2*len)*hd*bpe.
 *                    Tasks are then non-uniform; the busiest SM is found exactly
 *                    (GEMM: closed form per SM; MoE: runs of equal tasks;
 *                    attention: every task walked; one warp per pair).  GEMM,
 *                    fused MoE and attention with SP_SCHED_RR only
 *                    (SP_E_UNSUPPORTED otherwise); <= 4096 SMs per spec.
 */
#define SP_FEAT_CLAMPED 1u

sp_status sp_featurize_ex(sp_ctx *ctx, const sp_config_batch *cfg, const sp_specs *specs,
                          const sp_pairing *pairs, int32_t scheduler, uint32_t flags, const sp_features *out,
                          void *stream);

/*
 * Predictor stage, steps a10..a12: for each pair p < in->n_pairs,
 * x = normalised Table IV vector of in (O8-O9), e = sigmoid(MLP(x)),
 * latency_us[p] = t_theory_us[p] / e.  efficiency may be NULL.  Pairs with
 * status != 0 yield NaN.  latency_us / efficiency: DEVICE fp32 [n_pairs].
 * SP_E_ARG if in->family != the model's family.
 */
sp_status sp_predict(sp_ctx *ctx, const sp_model *model, const sp_features *in, float *latency_us,
                     float *efficiency, void *stream);

/*
 * Fused feature + predictor stage (SURVEY §8(b) "fused"): the result of
 * sp_featurize followed by sp_predict -- the same feature records in `out`,
 * bit for bit, and the same latencies -- with the record computation moved into
 * the predictor's producer warps, so the records are written while the tensor
 * cores run the MLP instead of in a separate HBM-bound pass.  Applies to the
 * uniform-task families (GEMM, fused MoE, RMSNorm, SiLU&Mul, Scaled MM) with
 * SP_PAIRS_CROSS and a 16-bit (tcgen05) model; anything else runs the two
 * calls in sequence.  A small per-config pre-pass (56 B per config, in a
 * context-owned grow-only scratch: the first call with more configs than
 * before allocates; see sp_prepare) runs first.  Asynchronous on `stream`; errors as
 * sp_featurize and sp_predict.
 */
sp_status sp_featurize_predict(sp_ctx *ctx, const sp_config_batch *cfg, const sp_specs *specs,
                               const sp_pairing *pairs, const sp_model *model, const sp_features *out,
                               float *latency_us, float *efficiency, void *stream);

/*
 * Host-buffer end-to-end prediction: SPEC's predict_latency batched
 * over the CROSS pairing of specs [spec_begin, spec_end) x all configs --
 * the call a user makes with configs in host memory.
 *   host_cfg:     as sp_config_batch, but fields / ragged / ragged_off are
 *                 HOST pointers (pinned memory gives asynchronous copies;
 *                 pageable memory works, with staged copies)
 *   host_latency: HOST fp32 [spec_end - spec_begin][n_configs], spec-major as
 *                 sp_featurize numbers pairs; NaN for pairs with status != 0
 *   slice_weights / n_slices: the configs are cut into slices pipelined over
 *                 three streams (H2D of slice i+1 and D2H of slice i-1 overlap
 *                 the kernels of slice i).  NULL weights: n_slices equal
 *                 slices (0: the default, 8; attention defaults to the
 *                 weights (1, 2, 3, 2)); otherwise n_slices relative weights.
 *                 A wide spec axis (>= 64 specs and >= 4 slices per spec)
 *                 is sliced by spec instead (configs uploaded once).
 *   stream:       the kernels run on it; the copies on two library streams
 *                 ordered after the work already on `stream`.
 * Each slice copies only its own range of the ragged data, planned from the
 * host offsets at the slice boundaries and checked on the device; a batch
 * whose ragged data is not laid out config by config is redone with one whole
 * copy (same result).  Blocks until host_latency is written.  Uses context-
 * owned grow-only device staging (the first call at a new size allocates):
 * calls on one context must not run concurrently.  Errors: SP_E_ARG (NULL,
 * sizes, range), then as sp_featurize_predict; SP_E_INTERNAL on a CUDA error.
 */
sp_status sp_predict_host(sp_ctx *ctx, const sp_config_batch *host_cfg, const sp_specs *specs,
                          int32_t spec_begin, int32_t spec_end, const sp_model *model, float *host_latency,
                          const float *slice_weights, int32_t n_slices, void *stream);

/*
 * Performance-gap diagnosis (PAPER §VII).  A
 * second estimator trained with quantile loss at q = 0.8 predicts the
 * "Potential Performance Ceiling" efficiency y_p80; it is an
 * ordinary sp_model run through sp_predict (its `efficiency` output).  For
 * every pair, with measured latency m:
 *   y_actual = t_theory_us / m          (efficiency, P:489's definition)
 *   gap      = y_p80 - y_actual          ("perf_gap")
 *   underperforming <=> gap > 0.1        (strict)
 * all in fp32 (IEEE division and subtraction).  Pairs with status != 0, a
 * NaN operand or m <= 0 are skipped (counted in neither total).
 *   in:        features of the pairs (t_theory_us = flts[11], status)
 *   eff_p80:   DEVICE fp32 [n_pairs], sp_predict's efficiency of the P80 model
 *   measured_us: DEVICE fp32 [n_pairs]
 *   pairs:     how pair p maps to a spec: SP_PAIRS_CROSS (spec = spec_begin +
 *              p / n_configs, spec-major as sp_featurize writes) or
 *              SP_PAIRS_LIST (spec_idx[p]); G = number of spec slots
 *              (CROSS: spec_end - spec_begin; LIST: n_specs below)
 *   n_configs: configs per spec (CROSS); n_specs: slots (LIST)
 * Outputs (DEVICE, caller-owned, zeroed by the call; gap may be NULL):
 *   gap        fp32 [n_pairs] (NaN for skipped pairs)
 *   counts     int64 [G][2]: {valid pairs, underperforming pairs} per spec
 *   hist       int64 [G][n_bins]: gap histogram on [gap_lo, gap_hi), the end
 *              bins also collect the gaps below / above (the CDF of Fig. 7)
 * Asynchronous on `stream`.
 */
#define SP_GAP_THRESHOLD 0.1f
sp_status sp_perf_gap(sp_ctx *ctx, const sp_features *in, const float *eff_p80, const float *measured_us,
                      const sp_pairing *pairs, int64_t n_configs, int32_t n_specs, int32_t n_bins,
                      float gap_lo, float gap_hi, float *gap, int64_t *counts, int64_t *hist, void *stream);

/*
 * Kernel accounting, for measurement (bench.py's roofline and launch count,
 * DESIGN.md section 6).  Every kernel launched by sp_featurize / sp_predict is
 * counted per kernel name.  With profiling enabled (off by default) each such
 * launch is also bracketed by two CUDA events recorded on the caller's stream,
 * so the per-kernel device time is measured in place, inside the caller's
 * timed region.  sp_profile_read waits for the pending events, writes up to
 * `max` entries (kernel name: static library-owned string; launches; summed
 * device milliseconds, 0 for launches made while profiling was off) and
 * returns the number of kernels seen; reset != 0 clears the totals.  Returns
 * -1 on a NULL context or a CUDA error (message in sp_last_error).
 */
typedef struct sp_kernel_stat {
  const char *kernel;
  int64_t launches;
  double total_ms;
} sp_kernel_stat;

sp_status sp_set_profiling(sp_ctx *ctx, int32_t enable);
int32_t sp_profile_read(sp_ctx *ctx, sp_kernel_stat *out, int32_t max, int32_t reset);

/* ===================================================================
 * End-to-end serving composition (PAPER §V-D; SURVEY §8(f) NEXT-1,
 * BASELINE config 4).  A Workload Generator turns a model and a batch of
 * requests into "a sequence of kernel invocations that represents a real
 * inference scenario"; kernels run "sequentially without overlap" and the
 * end-to-end latency is "the sum of all predicted kernel durations";
 * All-Reduce (TP) and Send/Recv (PP) latencies come from a regression over
 * profiled (volume, latency) points.  Readings E1..E9
 * fix what the paper leaves open:
 *   E1 per layer: RMSNorm, QKV GEMM, Attention, O GEMM, [AllReduce], RMSNorm,
 *      GateUp GEMM, SiLU&Mul, Down GEMM, [AllReduce]; then final RMSNorm and
 *      LM-head GEMM once per forward pass; pp-1 Send/Recv per forward pass
 *      (SPEC S:556).
 *   E2 static batch: step 0 prefills every request (qlen = kvlen = input_len,
 *      causal); decode step k = 1 .. max(output_len)-1 runs the requests with
 *      output_len > k in batch order, qlen 1, kvlen = input_len + k.
 *   E3 token count M = sum of qlen over the step's requests; the LM head runs
 *      on one row per sequence.
 *   E4 GEMM tiles by M: <= 64 -> 64x128 (BK 64, 4 stages, 4 warps, 128 regs);
 *      <= 256 -> 128x128 (4 stages, 8 warps, 168 regs); else 128x256
 *      (3 stages, 8 warps, 232 regs).
 *   E5 attention (FA2): heads nh/tp, nkv/tp; prefill BQ 128, BKV 64, causal,
 *      4 warps, 168 regs; decode BQ 16, BKV 64, non-causal, 4 warps, 64 regs,
 *      kv_chunk 1024 if n_active*nkv/tp < 128 else unsplit.
 *   E6 RMSNorm (dim = hidden) and SiLU&Mul (dim = intermediate/tp):
 *      clamp(ceil(dim/256), 1, 32) warps, 32 regs.
 *   E7 comm bytes M*hidden*2; latency interpolated linearly in ln(bytes)
 *      over the spec's calibration points, clamped flat at both ends.
 *   E8 per trace: sum over its steps; breakdown by category (Table I).
 *   E9 bf16 everywhere (2 bytes per element).
 * The expansion runs on the GPU; the resulting config batches go through
 * sp_featurize / sp_predict like any other; sp_e2e_compose sums them.
 * =================================================================== */

/* SPEC ModelConfig + ParallelConfig: a dense SwiGLU transformer. */
typedef struct sp_serving_model {
  int32_t n_layers, hidden, n_heads, n_kv_heads, head_dim, intermediate, vocab;
  int32_t tp;     /* tensor parallel degree >= 1: heads, kv heads, intermediate, vocab divisible */
  int32_t pp;     /* pipeline parallel degree >= 1: n_layers divisible */
  int32_t dtype;  /* SP_BF16 (E9) */
} sp_serving_model;

/* Breakdown categories of sp_e2e_compose (Table I's kernel classes). */
enum { SP_E2E_CAT_GEMM = 0, SP_E2E_CAT_ATTENTION = 1, SP_E2E_CAT_RMSNORM = 2,
       SP_E2E_CAT_SILU_MUL = 3, SP_E2E_CAT_COMM = 4, SP_E2E_NCAT = 5 };

typedef struct sp_e2e_plan sp_e2e_plan;

/* Sizes of an expanded plan.  Config batches (sp_e2e_plan_batch):
 *   SP_ATTENTION: one config per step, steps of trace r contiguous
 *                 (n_steps configs, n_ragged int32 (qlen, kvlen) entries);
 *   SP_GEMM:      4 * n_slots + max_batch configs: kind k in {QKV, O, GateUp,
 *                 Down} at k*n_slots + slot, LM head at 4*n_slots + (seqs-1);
 *   SP_RMSNORM, SP_SILU_MUL: n_slots configs.
 * A slot is a token count: slot j < max_batch holds M = j+1 (decode steps);
 * slot max_batch + r holds trace r's prefill M = sum of its input lengths. */
typedef struct sp_e2e_info {
  int32_t n_traces;
  int32_t max_batch;   /* largest number of requests in a trace */
  int64_t n_requests;
  int64_t n_steps;     /* sum over traces of max(output_len) */
  int64_t n_ragged;    /* 2 * sum of output_len */
  int64_t n_slots;     /* max_batch + n_traces */
  int64_t n_configs[5];  /* per sp_family; 0 for SP_FUSED_MOE */
} sp_e2e_info;

/*
 * Builds the invocation plan of R request traces (E1-E9) for `model`.
 *   req_off:    HOST int64 [n_traces+1], trace r = requests [req_off[r], req_off[r+1])
 *   input_len, output_len: HOST int32 [req_off[n_traces]]
 * Copies the requests to the device on `stream` and expands them there (one
 * warp per step); the plan owns all device memory it needs (allocated here,
 * reused by later sp_e2e_plan_update calls that fit).  Errors: SP_E_ARG (NULL,
 * counts, divisibility of heads / kv heads / intermediate / vocab by tp or of
 * layers by pp, dtype != SP_BF16), SP_E_DATA (a trace without requests, a
 * length < 1, or a token count >= 2^31), SP_E_INTERNAL (CUDA).
 * The plan is valid for use on `stream` once the call returns (stream order).
 */
sp_status sp_e2e_plan_create(sp_ctx *ctx, const sp_serving_model *model, int32_t n_traces,
                             const int64_t *req_off, const int32_t *input_len,
                             const int32_t *output_len, void *stream, sp_e2e_plan **out);
/* Re-expands new traces into an existing plan (same model), growing its
 * buffers only if needed.  Same arguments and errors as sp_e2e_plan_create. */
sp_status sp_e2e_plan_update(sp_e2e_plan *plan, int32_t n_traces, const int64_t *req_off,
                             const int32_t *input_len, const int32_t *output_len, void *stream);
/* Re-runs the expansion kernels from the requests already resident in the
 * plan (no host work, no copy): the device-side step of a timed loop. */
sp_status sp_e2e_plan_expand(sp_e2e_plan *plan, void *stream);
void sp_free_e2e_plan(sp_e2e_plan *plan);
sp_status sp_e2e_plan_info(const sp_e2e_plan *plan, sp_e2e_info *out);
/* The plan's config batch of one family (DEVICE pointers owned by the plan,
 * valid until the next update / free).  SP_E_ARG for SP_FUSED_MOE. */
sp_status sp_e2e_plan_batch(const sp_e2e_plan *plan, int32_t family, sp_config_batch *out);

/* Communication estimator (SPEC CommModel S:545): per spec, one
 * calibration table per collective at this plan's world size, all on the same
 * byte grid.  HOST fp64 arrays: bytes [n_points] strictly increasing > 0;
 * allreduce_us, sendrecv_us [n_specs][n_points] finite, >= 0, non-decreasing
 * in bytes.  Spec g of the table = spec g of the sp_specs handle used
 * with it.  SP_E_DATA on a table violating these rules. */
typedef struct sp_comm_desc {
  int32_t n_specs;
  int32_t n_points;   /* 1 .. 64 */
  const double *bytes;
  const double *allreduce_us;
  const double *sendrecv_us;
} sp_comm_desc;
typedef struct sp_comm_model sp_comm_model;
sp_status sp_load_comm_model(sp_ctx *ctx, const sp_comm_desc *desc, sp_comm_model **out);
void sp_free_comm_model(sp_comm_model *comm);

/* Per-family predicted latencies of the plan's batches (DEVICE fp32), each
 * spec-major over specs [spec_begin, spec_end) as sp_predict writes them after
 * sp_featurize with SP_PAIRS_CROSS: lat[(g - spec_begin) * n_configs + c]. */
typedef struct sp_e2e_latencies {
  const float *gemm;
  const float *attention;
  const float *rmsnorm;
  const float *silu_mul;
} sp_e2e_latencies;

/*
 * Composition (E8): for every spec g of [spec_begin, spec_end) and step
 * s, the step latency is the sum of its invocations' latencies
 *   L*(2 rms + qkv + attn + o + gate_up + silu + down + 2 [tp>1] allreduce)
 *   + (pp-1) sendrecv + rms + lm_head,
 * and trace r's latency the sum of its steps (fp64).  Outputs (DEVICE,
 * caller-owned, each may be NULL):
 *   step_us   fp32 [G][n_steps]
 *   trace_us  fp64 [G][n_traces]               (total)
 *   trace_cat fp64 [G][n_traces][SP_E2E_NCAT]  (breakdown; sums to trace_us)
 * G = spec_end - spec_begin.  comm may be NULL when tp == pp == 1; it must
 * cover spec_end specs otherwise.  A NaN latency (a pair with status != 0)
 * propagates.  Asynchronous on `stream`; no allocation.
 */
sp_status sp_e2e_compose(sp_ctx *ctx, const sp_e2e_plan *plan, int32_t spec_begin, int32_t spec_end,
                         const sp_comm_model *comm, const sp_e2e_latencies *lat, float *step_us,
                         double *trace_us, double *trace_cat, void *stream);

/* ===================================================================
 * Estimator training on the GPU (PAPER §V-C; §VII-A P:670;
 * SURVEY §8(f) NEXT-4).  One minibatch step of the per-category MLP:
 *   target  t = t_theory_us / measured_us        (execution efficiency)
 *   input   x = normalised Table IV vector        (O8-O9 with the model's mu/sigma, R17)
 *   forward, per hidden layer: z = h W^T + b, a = relu(z),
 *           batch-statistics BatchNorm a_hat = (a - mean)/sqrt(var + eps) (biased var),
 *           y = gamma a_hat + beta, inverted Dropout(p) -> h; e = sigmoid(h3 . w4 + b4)
 *   loss    MAPE mean |e - t| / max(t, 1e-6) or pinball(q)
 *   update  AdamW: decoupled weight decay on every parameter, bias-corrected
 *           moments; running BN statistics with momentum and unbiased variance.
 * Readings T1..T9 fix what the paper leaves open.  The dropout
 * keep mask is counter-based (T3): splitmix64 finaliser of seed + ctr*0x9E3779B97F4A7C15,
 * ctr = ((step*4 + layer)*2^20 + row)*2^8 + col; keep iff bits 63..40 >= round(p*2^24).
 * Arithmetic is fp32 (CUDA cores); reductions run in a fixed order, so a step is
 * deterministic.  Oracle: oracle/train.py (fp64).
 * =================================================================== */

typedef enum sp_loss { SP_LOSS_MAPE = 0, SP_LOSS_PINBALL = 1 } sp_loss;

typedef struct sp_train_config {
  int32_t loss;          /* sp_loss */
  float quantile;        /* pinball q in (0,1); 0.8 for the P80 ceiling */
  float lr;              /* 1e-3 */
  float weight_decay;    /* decoupled; 0.01 (T5: the paper gives no value) */
  float beta1, beta2, adam_eps;  /* 0.9, 0.999, 1e-8 */
  float dropout;         /* p in [0,1); 0.1 */
  float bn_momentum;     /* 0.1 */
  int32_t max_batch;     /* largest minibatch, 2 .. 2^20 (sizes the trainer's buffers) */
  uint64_t seed;         /* dropout generator seed (T3) */
} sp_train_config;

typedef struct sp_trainer sp_trainer;

/* Creates a trainer on ctx's device from HOST initial weights (desc: same
 * layout and checks as sp_load_model; precision is ignored, training is fp32;
 * mu/sigma are the fixed input normalisation).  Allocates its device buffers
 * once (parameters, AdamW moments, activations for max_batch rows).
 * SP_E_ARG / SP_E_DATA on bad arguments, SP_E_INTERNAL on allocation failure. */
sp_status sp_train_create(sp_ctx *ctx, const sp_mlp_desc *init, const sp_train_config *cfg,
                          sp_trainer **out);
void sp_train_destroy(sp_trainer *tr);

/* One training step over the minibatch rows batch_idx[0..B) (DEVICE int64
 * pair indices into `in`, which must have the model's family; every indexed
 * pair must have status 0 and measured_us > 0).  measured_us: DEVICE fp32
 * [in->n_pairs].  loss_out: DEVICE fp32 [1] receiving the pre-update batch
 * loss, or NULL.  Advances the trainer's step counter (the dropout counter and
 * AdamW's t), which lives in device memory: the call can be captured in a CUDA
 * graph and replayed, each replay taking the next step.  Asynchronous on
 * `stream`; no allocation.  SP_E_ARG if B < 2 or B > max_batch. */
sp_status sp_train_step(sp_trainer *tr, const sp_features *in, const float *measured_us,
                        const int64_t *batch_idx, int64_t B, float *loss_out, void *stream);

/* Eval-mode loss (running statistics, no dropout) over rows idx[0..n) (DEVICE
 * int64), processed in chunks of max_batch: the validation loss that early
 * stopping monitors.  loss_out: DEVICE fp32 [1].  Asynchronous. */
sp_status sp_train_eval(sp_trainer *tr, const sp_features *in, const float *measured_us,
                        const int64_t *idx, int64_t n, float *loss_out, void *stream);

/* Number of floats sp_train_export writes: P + 2*(256+128+64), with
 * P = 256*n_in + 3*256 + 128*256 + 3*128 + 64*128 + 3*64 + 64 + 1 trainable
 * parameters in the order w1 b1 g1 be1 w2 b2 g2 be2 w3 b3 g3 be3 w4 b4
 * (weights row-major [out][in]), followed by the running statistics
 * m1 v1 m2 v2 m3 v3. */
int64_t sp_train_export_count(const sp_trainer *tr);

/* Waits for the trainer's pending work on `stream` and copies the current
 * parameters and running statistics into host_out[sp_train_export_count]. */
sp_status sp_train_export(sp_trainer *tr, float *host_out, void *stream);

/* Waits for the trainer's pending work on `stream` and copies the gradients of
 * the last sp_train_step (the P trainable parameters, same order) into
 * host_out[P]; P = sp_train_export_count - 2*(256+128+64).  For testing and
 * diagnosis. */
sp_status sp_train_export_grads(sp_trainer *tr, float *host_out, void *stream);

/* Normalisation statistics (R17; reading T7): per input feature k of the
 * family's Table IV vector, mean and population standard deviation of
 * ln(1 + v_k) over pairs idx[0..n) (DEVICE int64) of `in`, accumulated in fp64
 * in a fixed order.  Writes HOST mu_out[n_in], sigma_out[n_in]; synchronises
 * `stream`. */
sp_status sp_fit_norm(sp_ctx *ctx, const sp_features *in, const int64_t *idx, int64_t n, float *mu_out,
                      float *sigma_out, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* SYNPERF_H_ */
