/*
 * oracle/synperf_oracle.c -- plain, slow, fp64 CPU oracle of SynPerf's batched
 * prediction hot path (arXiv 2601.14910, "SynPerf").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / `--impl reference` legs may load this library.
 * The product path (paper_2601_14910_b200/) never imports, links or executes
 * it, and this file shares no code, header, table or constant generator with
 * the CUDA path: the two meet only at their inputs (workloads/).
 *
 * What it computes, per (kernel config X, GPU spec S) pair, step by step in the
 * paper's order (PAPER.md line numbers "P:n"; readings R1..R22 of SURVEY.md
 * §8(c), restated in DESIGN.md):
 *   O1 Kernel Decomposer F, Eq.1: enumerate every task tau_i in the
 *      kernel's natural order with its per-pipe op counts (Eq.3, P:335-338;
 *      element-wise counts) and its load bytes B_i.
 *   O2 Occupancy ("registers, shared memory, warp-slots") and waves
 *      ceil(T / (N_SM * occ)).
 *   O3 Scheduling Simulator M, Eq.2: hardware round-robin, task t
 *      dealt to SM (t mod N_SM) (R5), accumulated into explicit per-SM arrays.
 *      Scheduler modes (flags >> 4):
 *        1 GREEDY  hardware RR with retirement ("a new task is assigned
 *                  to an SM when an existing task finishes"): the
 *                  first N_SM*occ tasks are dealt cyclically, then each task
 *                  goes to the SM with the least accumulated busy time;
 *        2 MINHEAP persistent kernel with a software MinHeap scheduler (P:281,
 *                  P:427 FlashInfer FA3): W = min(N_SM*occ, T)
 *                  workers pinned round-robin to SMs, each task to the worker
 *                  with the least accumulated busy time.
 *      Busy time of a task = max over the family's pipes of its theoretical
 *      cycles ops_p / Th_p, kept exact as an integer in units of
 *      1/lcm(Th_p) cycle; ties go to the lowest index.
 *   O4 GPU totals: summed over the task list itself, independently of the
 *      per-SM arrays, so conservation (sum_j S_j = total) is a real check.
 *   O5 Max-SM: max_j S_j per quantity independently (R7).
 *   O6 Theoretical cycles, Eq.4 and Eq.5; memory cycles
 *      C_mem = B / BW_mem at GPU level (global, L2) and SM level
 *      (global, L2 per-SM shares BW/N_SM (R8), shared memory).
 *   O7 t_theory = max over the GPU-level roofs present / f (R9).
 *   O8-O11 Performance Estimator: Table IV vector in frozen
 *      order, log1p z-score normalisation (R17), MLP 256-128-64 with
 *      Linear -> ReLU -> BatchNorm (eval) -> Dropout(identity) (R18, unfused),
 *      sigmoid efficiency, latency = t_theory / efficiency.
 *
 * All floating point is fp64, no fast-math, no reassociation beyond what the
 * formulas state.  Integers are int64.  Nothing is blocked, fused or reordered.
 *
 * Parity pins for every function live in tests/test_oracle_pins.py; the one
 * function without an independent pin is the MLP's *realism* (no trained
 * weights exist) -- "parity unpinned" for realism, see DESIGN.md.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------- input formats (defined by workloads/, documented in include/synperf.h) */

enum { FAM_GEMM = 0, FAM_ATTENTION = 1, FAM_MOE = 2, FAM_RMSNORM = 3, FAM_SILU = 4, FAM_SCALED = 5,
       FAM_SPLITK = 6 };
enum { DT_BF16 = 0, DT_FP16 = 1, DT_FP32 = 2, DT_FP8 = 3 };

/* per-pair status codes (include/synperf.h sp_pair_status) */
enum {
  ST_OK = 0, ST_DIM = 1, ST_TILE = 2, ST_HEADS = 3, ST_HIST = 4,
  ST_CAUSAL = 5, ST_RES = 6, ST_DTYPE = 7, ST_RANGE = 8, ST_INDEX = 9
};

/* field order of each family (workloads/gen.py FIELDS) */
enum { G_M, G_N, G_K, G_TM, G_TN, G_BK, G_STAGES, G_WARPS, G_REGS, G_SMEM, G_DTYPE };
enum { A_BS, A_NH, A_NKV, A_HD, A_BQ, A_BKV, A_CHUNK, A_CAUSAL, A_WARPS, A_REGS, A_SMEM, A_DTYPE };
enum { E_M, E_E, E_TOPK, E_H, E_N, E_BM, E_BN, E_BK, E_GROUPM, E_STAGES, E_WARPS, E_REGS, E_SMEM, E_DTYPE };
enum { R_SEQ, R_DIM, R_WARPS, R_REGS, R_SMEM, R_DTYPE };
enum { K_M, K_N, K_K, K_TM, K_TN, K_BK, K_SPLIT, K_STAGES, K_WARPS, K_REGS, K_SMEM, K_DTYPE };

/* Table II record, byte layout of workloads/specs.py SPEC_DTYPE (112 B) */
typedef struct {
  char name[32];
  int32_t cc_major, cc_minor, num_sms;
  int32_t th_tensor_bf16, th_tensor_fp16, th_tensor_fp8, th_fma, th_xu;
  int32_t smem_bw_bytes_per_clk, smem_per_sm_bytes, regfile_per_sm_bytes;
  int32_t max_warps_per_sm, max_ctas_per_sm, pad_;
  double sm_clock_mhz, bw_global_gbps, bw_l2_gbps;
} orc_spec;

/* oracle flags */
#define ORC_CLAMPED 1 /* SPEC's clamped edge tiles (R2 alternative), oracle-only */
#define ORC_SCHED_SHIFT 4 /* scheduler mode in bits 4..5: 0 RR, 1 GREEDY, 2 MINHEAP */
enum { SCHED_RR = 0, SCHED_GREEDY = 1, SCHED_MINHEAP = 2 };

/* output slots (SURVEY §8 uniform record) */
enum { I_NTASKS, I_OCC, I_WAVES, I_TOT_T, I_TOT_F, I_TOT_X, I_MAX_T, I_MAX_F, I_MAX_X,
       I_BYTES, I_BYTES_MAX, N_I };
enum { F_CG_T, F_CG_F, F_CG_X, F_CS_T, F_CS_F, F_CS_X, F_GLOB_G, F_L2_G, F_GLOB_S, F_L2_S,
       F_SMEM_S, F_TTHEORY, N_F };

#define INT64_LIM 9223372036854775807LL

/* Demands are accumulated in 128-bit integers so that the exact-range rule
 * (status 8 when a count does not fit in int64, R22) is decided exactly. */
typedef __int128 i128;
#define SAT128 ((i128)1 << 100)

static int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
static int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }

static int bytes_per_elem(int dtype) {
  switch (dtype) {
    case DT_BF16: case DT_FP16: return 2;
    case DT_FP32: return 4;
    default: return 0;
  }
}

/* ---------------- O3/O4 accumulation state for one pair ---------------- */

/* quantity index: 0 = Tensor ops, 1 = FMA ops, 2 = XU ops, 3 = load bytes */
typedef struct {
  int64_t n_sm;
  int64_t t;          /* tasks enumerated so far (= next task index) */
  i128 *sm_sum;       /* [n_sm][4] explicit per-SM sums  S_j(X) */
  int64_t *sm_count;  /* [n_sm] tasks per SM */
  i128 total[4];      /* sum over the task list */
  int mode;           /* SCHED_*; non-RR modes collect the task list first */
  i128 *list;         /* [cap][4] task demands in task order (GREEDY / MINHEAP) */
  int64_t cap;
} orc_sched;

/* One task tau_t with demands d[4]: Eq.2 cyclic dealing (R5) + O4 totals.
 * GREEDY / MINHEAP: the task is recorded and dealt later (schedule_list). */
static void emit_task(orc_sched *s, i128 ops_t, i128 ops_f, i128 ops_x, i128 bytes) {
  i128 d[4] = {ops_t, ops_f, ops_x, bytes};
  if (s->mode != SCHED_RR) {
    if (s->t == s->cap) {
      s->cap = s->cap ? 2 * s->cap : 1024;
      s->list = (i128 *)realloc(s->list, (size_t)s->cap * 4 * sizeof(i128));
    }
    for (int q = 0; q < 4; ++q) {
      s->list[s->t * 4 + q] = d[q];
      if (s->total[q] < SAT128) s->total[q] += d[q];
    }
    s->t += 1;
    return;
  }
  int64_t j = s->t % s->n_sm; /* M: task t -> SM (t mod N_SM) */
  for (int q = 0; q < 4; ++q) {
    /* saturate far above int64 (only the > INT64_MAX decision matters there) */
    if (s->sm_sum[j * 4 + q] < SAT128) s->sm_sum[j * 4 + q] += d[q];
    if (s->total[q] < SAT128) s->total[q] += d[q];
  }
  s->sm_count[j] += 1;
  s->t += 1;
}

/* ---------------- O1 decomposers (Eq.1, one per family) ---------------- */

/* Scaled MM (Table V; FP8 with block-wise quantisation; reading
 * R23): GEMM's output tiles, operands one byte each, and every task also
 * loads its fp32 scales -- one per (row of A, 128-wide K block) and one per
 * (128x128 block of B): tm*ceil(K/128) + ceil(tn/128)*ceil(K/128) floats. */
static void decompose_scaled_mm(const int64_t *x, orc_sched *s) {
  int64_t M = x[G_M], N = x[G_N], K = x[G_K], tm = x[G_TM], tn = x[G_TN], bk = x[G_BK];
  int64_t kpad = cdiv(K, bk) * bk;
  int64_t kblocks = cdiv(K, 128);
  for (int64_t i = 0; i < cdiv(M, tm); ++i) {
    for (int64_t j = 0; j < cdiv(N, tn); ++j) {
      i128 operand_bytes = (i128)(tm + tn) * kpad * 1;               /* FP8: 1 byte per element */
      i128 scale_bytes = ((i128)tm * kblocks + (i128)cdiv(tn, 128) * kblocks) * 4;  /* fp32 scales */
      emit_task(s, (i128)2 * tm * tn * kpad, 0, 0, operand_bytes + scale_bytes);
    }
  }
}

/* Split-K GEMM (cuBLAS's split-K variants, tiling inferred from profiles
 * P:270; Table V P:409 Tensor pipe; reading R25).  The K loop of kt =
 * ceil(K/BK) k-tiles is cut into slices of kps = ceil(kt/SPLIT_K) k-tiles,
 * slice z holding min(kps, kt - z*kps) of them; slices are enumerated while
 * they hold at least one k-tile.  Grid order: slice z outermost (grid z is
 * dispatched last), then output tiles row-major as in GEMM.  Each task is a
 * padded tm x tn tile over its slice's k_z*BK extent.  The fp32 reduction of
 * the partial tiles is another kernel and is not part of this one (R25). */
static void decompose_gemm_splitk(const int64_t *x, orc_sched *s) {
  int64_t M = x[K_M], N = x[K_N], K = x[K_K], tm = x[K_TM], tn = x[K_TN], bk = x[K_BK];
  int64_t bpe = bytes_per_elem((int)x[K_DTYPE]);
  int64_t kt = cdiv(K, bk), kps = cdiv(kt, x[K_SPLIT]);
  for (int64_t z = 0; z * kps < kt; ++z) {
    int64_t kz = imin(kps, kt - z * kps); /* k-tiles of slice z */
    for (int64_t i = 0; i < cdiv(M, tm); ++i)
      for (int64_t j = 0; j < cdiv(N, tn); ++j)
        emit_task(s, (i128)2 * tm * tn * kz * bk, 0, 0, (i128)(tm + tn) * kz * bk * bpe);
  }
}

/* GEMM (Table V; Eq.3 alpha = 2): output tiles row-major,
 * i over ceil(M/tm) outer, j over ceil(N/tn) inner (R4).  Padded (R2): every
 * tile is a full tm x tn x K_pad MMA with K_pad = ceil(K/BK)*BK (R1);
 * loads = (tm + tn) * K_pad elements (A and B panels). */
static void decompose_gemm(const int64_t *x, int flags, orc_sched *s) {
  int64_t M = x[G_M], N = x[G_N], K = x[G_K], tm = x[G_TM], tn = x[G_TN], bk = x[G_BK];
  int64_t bpe = bytes_per_elem((int)x[G_DTYPE]);
  int64_t kpad = cdiv(K, bk) * bk;
  for (int64_t i = 0; i < cdiv(M, tm); ++i) {
    for (int64_t j = 0; j < cdiv(N, tn); ++j) {
      if (flags & ORC_CLAMPED) {
        int64_t ma = imin(tm, M - i * tm), na = imin(tn, N - j * tn);
        emit_task(s, (i128)2 * ma * na * K, 0, 0, (i128)(ma + na) * K * bpe);
      } else {
        emit_task(s, (i128)2 * tm * tn * kpad, 0, 0, (i128)(tm + tn) * kpad * bpe);
      }
    }
  }
}

/* Fused MoE (Table V; §V-B; R16): expert e receives t_e
 * tokens (histogram, or balanced q + [e < r]); tasks are expert-major, then
 * m-block over ceil(t_e/BM), then n-block over ceil(N/BN); each task is a
 * padded BM x BN x H_pad GEMM tile, H_pad = ceil(H/BK)*BK. */
static void decompose_moe(const int64_t *x, const int32_t *hist, int flags, orc_sched *s) {
  int64_t M = x[E_M], E = x[E_E], topk = x[E_TOPK], H = x[E_H], N = x[E_N];
  int64_t bm = x[E_BM], bn = x[E_BN], bk = x[E_BK];
  int64_t bpe = bytes_per_elem((int)x[E_DTYPE]);
  int64_t hpad = cdiv(H, bk) * bk;
  int64_t q = (M * topk) / E, r = (M * topk) % E;
  for (int64_t e = 0; e < E; ++e) {
    int64_t te = hist ? (int64_t)hist[e] : q + (e < r ? 1 : 0);
    for (int64_t mb = 0; mb < cdiv(te, bm); ++mb) {
      for (int64_t nb = 0; nb < cdiv(N, bn); ++nb) {
        if (flags & ORC_CLAMPED) {
          int64_t ma = imin(bm, te - mb * bm), na = imin(bn, N - nb * bn);
          emit_task(s, (i128)2 * ma * na * H, 0, 0, (i128)(ma + na) * H * bpe);
        } else {
          emit_task(s, (i128)2 * bm * bn * hpad, 0, 0, (i128)(bm + bn) * hpad * bpe);
        }
      }
    }
  }
}

/* RMSNorm (Table V, FMA+XU; R14): one task per row; per row
 * FMA = 3*dim (square-accumulate, scale, weight multiply), XU = 1 (rsqrt,
 * Table III), loads = input row + weight vector = 2*dim elements. */
static void decompose_rmsnorm(const int64_t *x, orc_sched *s) {
  int64_t seq = x[R_SEQ], dim = x[R_DIM], bpe = bytes_per_elem((int)x[R_DTYPE]);
  for (int64_t row = 0; row < seq; ++row) emit_task(s, 0, (i128)3 * dim, 1, (i128)2 * dim * bpe);
}

/* SiLU&Mul (Table V, FMA+XU; R15): one task per row; dim = output
 * width; per element FMA 4, XU 2 (ex2 + rcp, Table III); loads = gate +
 * up halves = 2*dim elements. */
static void decompose_silu(const int64_t *x, orc_sched *s) {
  int64_t seq = x[R_SEQ], dim = x[R_DIM], bpe = bytes_per_elem((int)x[R_DTYPE]);
  for (int64_t row = 0; row < seq; ++row) emit_task(s, 0, (i128)4 * dim, (i128)2 * dim, (i128)2 * dim * bpe);
}

/* Attention, FlashInfer FA2 (Table V; Eq.3 alpha = 4; P:262
 * causal non-uniform tasks; R10-R13).  GQA group g = nh/nkv; request b has
 * R_b = qlen_b * g packed query rows and nqb_b = ceil(R_b/BQ) q-blocks; task
 * order: kv-head h outermost, then request b, q-block i, kv-chunk c (R4).
 * For q-block i the last query token is q_last = floor((min((i+1)BQ, R_b)-1)/g);
 * causal: kv_need = min(kvlen, kvlen - qlen + q_last + 1), else kv_need = kvlen;
 * split-KV (R12): n_ch = ceil(kv_need/kv_chunk) chunks of
 * len_c = min(kv_chunk, kv_need - c*kv_chunk) (kv_chunk = 0: one chunk);
 * kv_eff = ceil(len_c/BKV)*BKV.  Per task: Tensor 4*BQ*kv_eff*hd; XU = one exp2
 * per score + one rescale exp2 per row per KV block = BQ*kv_eff + BQ*kv_eff/BKV;
 * loads = Q tile + K and V tiles = (BQ*hd + 2*kv_eff*hd) elements. */
static void decompose_attention(const int64_t *x, const int32_t *req, int flags, orc_sched *s) {
  int64_t bs = x[A_BS], nh = x[A_NH], nkv = x[A_NKV], hd = x[A_HD];
  int64_t bq = x[A_BQ], bkv = x[A_BKV], chunk = x[A_CHUNK], causal = x[A_CAUSAL];
  int64_t bpe = bytes_per_elem((int)x[A_DTYPE]);
  int64_t g = nh / nkv;
  for (int64_t h = 0; h < nkv; ++h) {
    for (int64_t b = 0; b < bs; ++b) {
      int64_t qlen = req[2 * b], kvlen = req[2 * b + 1];
      int64_t rows = qlen * g;
      for (int64_t i = 0; i < cdiv(rows, bq); ++i) {
        int64_t q_last = (imin((i + 1) * bq, rows) - 1) / g;
        int64_t kv_need = causal ? imin(kvlen, kvlen - qlen + q_last + 1) : kvlen;
        int64_t n_ch = chunk > 0 ? cdiv(kv_need, chunk) : 1;
        for (int64_t c = 0; c < n_ch; ++c) {
          int64_t len = chunk > 0 ? imin(chunk, kv_need - c * chunk) : kv_need;
          if (flags & ORC_CLAMPED) {
            int64_t qr = imin(bq, rows - i * bq);
            emit_task(s, (i128)4 * qr * len * hd, 0, (i128)qr * len + (i128)qr * cdiv(len, bkv),
                      ((i128)qr * hd + (i128)2 * len * hd) * bpe);
          } else {
            int64_t kv_eff = cdiv(len, bkv) * bkv;
            emit_task(s, (i128)4 * bq * kv_eff * hd, 0, (i128)bq * kv_eff + (i128)bq * (kv_eff / bkv),
                      ((i128)bq * hd + (i128)2 * kv_eff * hd) * bpe);
          }
        }
      }
    }
  }
}

/* ---------------- domain checks (include/synperf.h "per-pair domain") ---- */

static int is_tensor_family(int fam) {
  return fam == FAM_GEMM || fam == FAM_ATTENTION || fam == FAM_MOE || fam == FAM_SCALED || fam == FAM_SPLITK;
}

/* Validates one config against the paper's domain (every dimension >= 1,
 * heads divisible, causal kv >= q, a histogram summing to M*topk, ...) and
 * counts its tasks T and, for attention, the per-kv-head kv-unit sum
 * U = sum of kv_eff/BKV over one head's tasks (tests compare them with the
 * GPU's exact-range limits).  The oracle itself has no 32-bit limit: it
 * enumerates whatever the config defines (R22: only a count that does not fit
 * the int64 record is out of range, decided after the enumeration).
 * Counts saturate at SAT128.  Returns a status. */
static int validate(int fam, const int64_t *x, const int32_t *rag, i128 *T_out, i128 *U_out) {
  *T_out = 0;
  *U_out = 0;
  switch (fam) {
    case FAM_SCALED: case FAM_GEMM: {
      if (x[G_M] < 1 || x[G_N] < 1 || x[G_K] < 1) return ST_DIM;
      if (x[G_TM] < 1 || x[G_TN] < 1 || x[G_BK] < 1 || x[G_STAGES] < 1) return ST_TILE;
      if (x[G_WARPS] < 1 || x[G_REGS] < 1 || x[G_SMEM] < 0) return ST_RES;
      if (fam == FAM_SCALED ? x[G_DTYPE] != DT_FP8 : (x[G_DTYPE] != DT_BF16 && x[G_DTYPE] != DT_FP16))
        return ST_DTYPE;
      *T_out = (i128)cdiv(x[G_M], x[G_TM]) * cdiv(x[G_N], x[G_TN]);
      return ST_OK;
    }
    case FAM_SPLITK: {
      if (x[K_M] < 1 || x[K_N] < 1 || x[K_K] < 1) return ST_DIM;
      if (x[K_TM] < 1 || x[K_TN] < 1 || x[K_BK] < 1 || x[K_SPLIT] < 1 || x[K_STAGES] < 1) return ST_TILE;
      if (x[K_WARPS] < 1 || x[K_REGS] < 1 || x[K_SMEM] < 0) return ST_RES;
      if (x[K_DTYPE] != DT_BF16 && x[K_DTYPE] != DT_FP16) return ST_DTYPE;
      int64_t kt = cdiv(x[K_K], x[K_BK]), slices = cdiv(kt, cdiv(kt, x[K_SPLIT]));
      *T_out = (i128)slices * cdiv(x[K_M], x[K_TM]) * cdiv(x[K_N], x[K_TN]);
      return ST_OK;
    }
    case FAM_MOE: {
      if (x[E_M] < 1 || x[E_E] < 1 || x[E_TOPK] < 1 || x[E_H] < 1 || x[E_N] < 1) return ST_DIM;
      if (x[E_BM] < 1 || x[E_BN] < 1 || x[E_BK] < 1 || x[E_STAGES] < 1) return ST_TILE;
      if (x[E_WARPS] < 1 || x[E_REGS] < 1 || x[E_SMEM] < 0) return ST_RES;
      if (x[E_DTYPE] != DT_BF16 && x[E_DTYPE] != DT_FP16) return ST_DTYPE;
      int64_t mt = x[E_M] * x[E_TOPK];
      i128 T = 0;
      if (rag) {
        int64_t sum = 0;
        for (int64_t e = 0; e < x[E_E]; ++e) {
          if (rag[e] < 0) return ST_HIST;
          sum += rag[e];
        }
        if (sum != mt) return ST_HIST;
        for (int64_t e = 0; e < x[E_E]; ++e) T += cdiv(rag[e], x[E_BM]);
      } else {
        int64_t q = mt / x[E_E], r = mt % x[E_E];
        T = (i128)r * cdiv(q + 1, x[E_BM]) + (i128)(x[E_E] - r) * cdiv(q, x[E_BM]);
      }
      *T_out = T * cdiv(x[E_N], x[E_BN]);
      return ST_OK;
    }
    case FAM_RMSNORM: case FAM_SILU: {
      if (x[R_SEQ] < 1 || x[R_DIM] < 1) return ST_DIM;
      if (x[R_WARPS] < 1 || x[R_REGS] < 1 || x[R_SMEM] < 0) return ST_RES;
      if (bytes_per_elem((int)x[R_DTYPE]) == 0) return ST_DTYPE;
      *T_out = x[R_SEQ];
      return ST_OK;
    }
    case FAM_ATTENTION: {
      if (x[A_BS] < 1 || x[A_NH] < 1 || x[A_NKV] < 1 || x[A_HD] < 1) return ST_DIM;
      if (x[A_BQ] < 1 || x[A_BKV] < 1 || x[A_CHUNK] < 0) return ST_TILE; /* -1 is resolved before (R24) */
      if (x[A_WARPS] < 1 || x[A_REGS] < 1 || x[A_SMEM] < 0) return ST_RES;
      if (x[A_DTYPE] != DT_BF16 && x[A_DTYPE] != DT_FP16) return ST_DTYPE;
      if (x[A_NH] % x[A_NKV] != 0) return ST_HEADS;
      int64_t g = x[A_NH] / x[A_NKV];
      for (int64_t b = 0; b < x[A_BS]; ++b) {
        int64_t qlen = rag[2 * b], kvlen = rag[2 * b + 1];
        if (qlen < 1 || kvlen < 1) return ST_DIM;
        if (x[A_CAUSAL] && kvlen < qlen) return ST_CAUSAL;
      }
      /* per-head task count L and kv-unit sum U, counted item by item */
      i128 L = 0, U = 0;
      for (int64_t b = 0; b < x[A_BS]; ++b) {
        int64_t qlen = rag[2 * b], kvlen = rag[2 * b + 1], rows = qlen * g;
        for (int64_t i = 0; i < cdiv(rows, x[A_BQ]) && L < SAT128; ++i) {
          int64_t q_last = (imin((i + 1) * x[A_BQ], rows) - 1) / g;
          int64_t kv_need = x[A_CAUSAL] ? imin(kvlen, kvlen - qlen + q_last + 1) : kvlen;
          int64_t chunk = x[A_CHUNK];
          int64_t n_ch = chunk > 0 ? cdiv(kv_need, chunk) : 1;
          for (int64_t c = 0; c < n_ch; ++c) {
            int64_t len = chunk > 0 ? imin(chunk, kv_need - c * chunk) : kv_need;
            U += cdiv(len, x[A_BKV]);
          }
          L += n_ch;
        }
      }
      *T_out = L * x[A_NKV];
      *U_out = U;
      return ST_OK;
    }
  }
  return ST_DIM;
}

/* O2: per-task resource footprint and occupancy, R6 register units. */
static int64_t occupancy(int fam, const int64_t *x, const orc_spec *sp) {
  i128 smem = 0;
  int64_t warps = 0, regs = 0;
  switch (fam) {
    case FAM_SCALED: /* one-byte FP8 operand stages */
      warps = x[G_WARPS]; regs = x[G_REGS];
      smem = x[G_SMEM] > 0 ? (i128)x[G_SMEM] : (i128)x[G_STAGES] * (x[G_TM] + x[G_TN]) * x[G_BK] * 1;
      break;
    case FAM_GEMM:
      warps = x[G_WARPS]; regs = x[G_REGS];
      smem = x[G_SMEM] > 0 ? (i128)x[G_SMEM]
                           : (i128)x[G_STAGES] * (x[G_TM] + x[G_TN]) * x[G_BK] * bytes_per_elem((int)x[G_DTYPE]);
      break;
    case FAM_SPLITK:
      warps = x[K_WARPS]; regs = x[K_REGS];
      smem = x[K_SMEM] > 0 ? (i128)x[K_SMEM]
                           : (i128)x[K_STAGES] * (x[K_TM] + x[K_TN]) * x[K_BK] * bytes_per_elem((int)x[K_DTYPE]);
      break;
    case FAM_MOE:
      warps = x[E_WARPS]; regs = x[E_REGS];
      smem = x[E_SMEM] > 0 ? (i128)x[E_SMEM]
                           : (i128)x[E_STAGES] * (x[E_BM] + x[E_BN]) * x[E_BK] * bytes_per_elem((int)x[E_DTYPE]);
      break;
    case FAM_ATTENTION:
      warps = x[A_WARPS]; regs = x[A_REGS];
      smem = x[A_SMEM] > 0 ? (i128)x[A_SMEM]
                           : (i128)(x[A_BQ] + 2 * x[A_BKV]) * x[A_HD] * bytes_per_elem((int)x[A_DTYPE]);
      break;
    default:
      warps = x[R_WARPS]; regs = x[R_REGS];
      smem = x[R_SMEM] > 0 ? (i128)x[R_SMEM] : (i128)warps * 4;
      break;
  }
  i128 occ = sp->max_ctas_per_sm;
  if (smem > 0) {
    i128 q = (i128)sp->smem_per_sm_bytes / smem;
    if (q < occ) occ = q;
  }
  i128 rq = (i128)(sp->regfile_per_sm_bytes / 4) / ((i128)regs * 32 * warps);
  if (rq < occ) occ = rq;
  i128 wq = (i128)sp->max_warps_per_sm / warps;
  if (wq < occ) occ = wq;
  return occ < 1 ? 1 : (int64_t)occ;
}

/* Pipes present per family (Table V): bit 0 Tensor, 1 FMA, 2 XU */
static int pipes_of(int fam) {
  switch (fam) {
    case FAM_GEMM: case FAM_MOE: case FAM_SCALED: case FAM_SPLITK: return 1;
    case FAM_ATTENTION: return 1 | 4;
    default: return 2 | 4;
  }
}

static void set_error(int64_t *ints, double *flts) {
  for (int k = 0; k < N_I; ++k) ints[k] = -1;
  for (int k = 0; k < N_F; ++k) flts[k] = NAN;
}

/* ---------------- O3 non-cyclic schedulers (NEXT-2) ---------------- */

static int64_t gcd64(int64_t a, int64_t b) {
  while (b) {
    int64_t r = a % b;
    a = b;
    b = r;
  }
  return a;
}

/* GREEDY: tasks 0..N*occ-1 dealt cyclically (the RR rounds until every SM is
 * saturated), then task t to the SM with the least busy time (ties: lowest
 * SM).  cost[t] = busy time of task t.  Writes sm_of[t]. */
static void greedy_assign(const i128 *cost, int64_t n, int64_t n_sm, int64_t occ, int64_t *sm_of) {
  i128 *busy = (i128 *)calloc((size_t)n_sm, sizeof(i128));
  for (int64_t t = 0; t < n; ++t) {
    int64_t j;
    if (t < n_sm * occ) {
      j = t % n_sm;
    } else {
      j = 0;
      for (int64_t k = 1; k < n_sm; ++k)
        if (busy[k] < busy[j]) j = k;
    }
    busy[j] += cost[t];
    sm_of[t] = j;
  }
  free(busy);
}

/* MINHEAP: W = min(N*occ, n) workers, worker w resident on SM (w mod N);
 * task t to the worker with the least accumulated busy time (ties: lowest
 * worker) -- a linear scan gives the heap's answer.  Writes worker_of[t]
 * and sm_of[t]. */
static void minheap_assign(const i128 *cost, int64_t n, int64_t n_sm, int64_t occ, int64_t *worker_of,
                           int64_t *sm_of) {
  int64_t W = n_sm * occ < n ? n_sm * occ : n;
  if (W < 1) W = 1;
  i128 *load = (i128 *)calloc((size_t)W, sizeof(i128));
  for (int64_t t = 0; t < n; ++t) {
    int64_t w = 0;
    for (int64_t k = 1; k < W; ++k)
      if (load[k] < load[w]) w = k;
    load[w] += cost[t];
    if (worker_of) worker_of[t] = w;
    sm_of[t] = w % n_sm;
  }
  free(load);
}

/* Deal the recorded task list of s with scheduler `mode` into the per-SM
 * arrays.  th[p] = pipe throughputs (ops/clk/SM), pipes = Table V bitmask. */
static void schedule_list(orc_sched *s, int mode, int64_t occ, const int64_t *th, int pipes) {
  int64_t lc = 1; /* lcm of the pipes' throughputs: busy time in 1/lc cycles is an integer */
  for (int p = 0; p < 3; ++p)
    if (pipes & (1 << p)) lc = lc / gcd64(lc, th[p]) * th[p];
  i128 *cost = (i128 *)malloc((size_t)(s->t ? s->t : 1) * sizeof(i128));
  int64_t *sm_of = (int64_t *)malloc((size_t)(s->t ? s->t : 1) * sizeof(int64_t));
  for (int64_t t = 0; t < s->t; ++t) {
    i128 c = 0;
    for (int p = 0; p < 3; ++p) {
      if (!(pipes & (1 << p))) continue;
      i128 v = s->list[t * 4 + p] * (i128)(lc / th[p]); /* ops_p / Th_p cycles, in 1/lc units */
      if (v > c) c = v;
    }
    cost[t] = c;
  }
  if (mode == SCHED_GREEDY) greedy_assign(cost, s->t, s->n_sm, occ, sm_of);
  else minheap_assign(cost, s->t, s->n_sm, occ, NULL, sm_of);
  for (int64_t t = 0; t < s->t; ++t) {
    int64_t j = sm_of[t];
    for (int q = 0; q < 4; ++q)
      if (s->sm_sum[j * 4 + q] < SAT128) s->sm_sum[j * 4 + q] += s->list[t * 4 + q];
    s->sm_count[j] += 1;
  }
  free(cost);
  free(sm_of);
}

/* R24 split-KV planner (FlashInfer's decode planner; the decomposition F
 * depends on S): for a non-causal attention config with kv_chunk = -1
 * on spec sp, max_grid = N_SM * occupancy work items; no split (0) if
 * nkv * sum_b nqb_b >= max_grid, else the smallest chunk = 16c, c = 1, 2, ...,
 * with nkv * sum_b nqb_b * ceil(kvlen_b / chunk) <= max_grid -- 0 again if that
 * chunk covers the longest request.  A literal upward scan. */
static int64_t plan_kv_chunk(const int64_t *x, const int32_t *rag, const orc_spec *sp, int64_t occ) {
  int64_t g = x[A_NH] / x[A_NKV], max_grid = (int64_t)sp->num_sms * occ, w0 = 0, maxkv = 0;
  for (int64_t b = 0; b < x[A_BS]; ++b) {
    w0 += cdiv((int64_t)rag[2 * b] * g, x[A_BQ]);
    if (rag[2 * b + 1] > maxkv) maxkv = rag[2 * b + 1];
  }
  if (w0 * x[A_NKV] >= max_grid) return 0;
  for (int64_t c = 1;; ++c) {
    int64_t chunk = 16 * c, items = 0;
    for (int64_t b = 0; b < x[A_BS]; ++b) items += cdiv((int64_t)rag[2 * b] * g, x[A_BQ]) * cdiv(rag[2 * b + 1], chunk);
    if (items * x[A_NKV] <= max_grid) return chunk >= maxkv ? 0 : chunk;
  }
}

/* One (config, spec) pair through O1..O7.  ints[N_I], flts[N_F]. */
static int featurize_pair(int fam, const int64_t *x_in, const int32_t *rag, const orc_spec *sp,
                          int flags, int64_t *ints, double *flts) {
  int64_t x[16];
  i128 T = 0, U = 0;
  memcpy(x, x_in, sizeof x);
  int st;
  if (fam == FAM_ATTENTION && x[A_CHUNK] == -1 && !x[A_CAUSAL]) {
    x[A_CHUNK] = 0; /* domain checks first, with the unsplit extent */
    st = validate(fam, x, rag, &T, &U);
    if (st == ST_OK) {
      x[A_CHUNK] = plan_kv_chunk(x, rag, sp, occupancy(fam, x, sp));
      st = validate(fam, x, rag, &T, &U);
    }
  } else {
    st = validate(fam, x, rag, &T, &U);
  }
  int64_t tensor_th = 0;
  if (st == ST_OK && is_tensor_family(fam)) {
    int dt = (int)((fam == FAM_GEMM || fam == FAM_SCALED) ? x[G_DTYPE]
                   : fam == FAM_MOE                         ? x[E_DTYPE]
                   : fam == FAM_SPLITK                      ? x[K_DTYPE]
                                                            : x[A_DTYPE]);
    tensor_th = dt == DT_BF16 ? sp->th_tensor_bf16 : dt == DT_FP16 ? sp->th_tensor_fp16 : sp->th_tensor_fp8;
    if (tensor_th <= 0) st = ST_DTYPE;
  }
  if (st != ST_OK) {
    set_error(ints, flts);
    return st;
  }

  orc_sched s;
  memset(&s, 0, sizeof s);
  s.n_sm = sp->num_sms;
  s.sm_sum = (i128 *)calloc((size_t)s.n_sm * 4, sizeof(i128));
  s.sm_count = (int64_t *)calloc((size_t)s.n_sm, sizeof(int64_t));
  s.mode = (flags >> ORC_SCHED_SHIFT) & 3;

  switch (fam) { /* O1 + O3 + O4 */
    case FAM_GEMM: decompose_gemm(x, flags, &s); break;
    case FAM_SCALED: decompose_scaled_mm(x, &s); break;
    case FAM_SPLITK: decompose_gemm_splitk(x, &s); break;
    case FAM_MOE: decompose_moe(x, rag, flags, &s); break;
    case FAM_RMSNORM: decompose_rmsnorm(x, &s); break;
    case FAM_SILU: decompose_silu(x, &s); break;
    case FAM_ATTENTION: decompose_attention(x, rag, flags, &s); break;
  }
  if (s.mode != SCHED_RR) { /* O3 for GREEDY / MINHEAP over the recorded task list */
    int64_t th_sched[3] = {tensor_th, sp->th_fma, sp->th_xu};
    schedule_list(&s, s.mode, occupancy(fam, x, sp), th_sched, pipes_of(fam));
    free(s.list);
  }

  /* O5: per-quantity max over SMs (R7) */
  i128 mx128[4] = {0, 0, 0, 0};
  for (int64_t j = 0; j < s.n_sm; ++j)
    for (int q = 0; q < 4; ++q)
      if (s.sm_sum[j * 4 + q] > mx128[q]) mx128[q] = s.sm_sum[j * 4 + q];

  /* exact-range rule (R22): every count must fit in int64; max <= total */
  int range_ok = 1;
  for (int q = 0; q < 4; ++q)
    if (s.total[q] > (i128)INT64_LIM) range_ok = 0;
  free(s.sm_sum);
  free(s.sm_count);
  if (!range_ok) {
    set_error(ints, flts);
    return ST_RANGE;
  }
  int64_t mx[4], tot[4];
  for (int q = 0; q < 4; ++q) {
    mx[q] = (int64_t)mx128[q];
    tot[q] = (int64_t)s.total[q];
  }

  /* O2 */
  int64_t occ = occupancy(fam, x, sp);
  ints[I_NTASKS] = s.t;
  ints[I_OCC] = occ;
  ints[I_WAVES] = cdiv(s.t, (int64_t)sp->num_sms * occ);
  ints[I_TOT_T] = tot[0];
  ints[I_TOT_F] = tot[1];
  ints[I_TOT_X] = tot[2];
  ints[I_MAX_T] = mx[0];
  ints[I_MAX_F] = mx[1];
  ints[I_MAX_X] = mx[2];
  ints[I_BYTES] = tot[3];
  ints[I_BYTES_MAX] = mx[3];

  /* O6: Eq.4 C_p = N_ops,p / Th_p ; Eq.5 C_p^GPU = N^GPU / (N_SM Th_p) */
  double nsm = (double)sp->num_sms, f = sp->sm_clock_mhz;
  double th[3] = {(double)tensor_th, (double)sp->th_fma, (double)sp->th_xu};
  int pipes = pipes_of(fam);
  for (int p = 0; p < 3; ++p) {
    if (pipes & (1 << p)) {
      flts[F_CG_T + p] = (double)tot[p] / (nsm * th[p]);
      flts[F_CS_T + p] = (double)mx[p] / th[p];
    } else {
      flts[F_CG_T + p] = 0.0;
      flts[F_CS_T + p] = 0.0;
    }
  }
  /* C_mem = B / BW in SM-clock cycles: B bytes / (BW GB/s * 1e3 B/us) * f cycles/us (R8) */
  double B = (double)tot[3], Bm = (double)mx[3];
  flts[F_GLOB_G] = B / (sp->bw_global_gbps * 1e3) * f;
  flts[F_L2_G] = B / (sp->bw_l2_gbps * 1e3) * f;
  flts[F_GLOB_S] = Bm / (sp->bw_global_gbps * 1e3 / nsm) * f;
  flts[F_L2_S] = Bm / (sp->bw_l2_gbps * 1e3 / nsm) * f;
  flts[F_SMEM_S] = Bm / (double)sp->smem_bw_bytes_per_clk;

  /* O7: t_theory = max(GPU-level roofs present) / f (R9) */
  double roof = fmax(flts[F_GLOB_G], flts[F_L2_G]);
  for (int p = 0; p < 3; ++p)
    if (pipes & (1 << p)) roof = fmax(roof, flts[F_CG_T + p]);
  flts[F_TTHEORY] = roof / f;
  return ST_OK;
}

/* Gather config c's fields (int32 SoA [n_fields][ld]) into int64 */
static void load_config(const int32_t *fields, int64_t ld, int64_t c, int nf, int64_t *x) {
  for (int k = 0; k < nf; ++k) x[k] = fields[(int64_t)k * ld + c];
}

static int n_fields_of(int fam) {
  switch (fam) {
    case FAM_GEMM: case FAM_SCALED: return 11;
    case FAM_ATTENTION: case FAM_SPLITK: return 12;
    case FAM_MOE: return 14;
    default: return 6;
  }
}

/*
 * Batched featurization.  Pair p uses config cfg_idx[p] and spec spec_idx[p].
 * Outputs SoA: ints[k * n_pairs + p] (k < 11), flts[k * n_pairs + p] (k < 12),
 * status[p].  Returns 0, or -1 on a bad family.
 */
int orc_featurize(int fam, int64_t n_configs, const int32_t *fields, int64_t field_ld,
                  const int32_t *ragged, const int64_t *ragged_off, const orc_spec *specs,
                  int64_t n_specs, int64_t n_pairs, const int64_t *cfg_idx, const int64_t *spec_idx, int flags,
                  int64_t *ints, double *flts, uint8_t *status, int nthreads) {
  if (fam < 0 || fam > FAM_SPLITK) return -1;
  int nf = n_fields_of(fam);
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
  for (int64_t p = 0; p < n_pairs; ++p) {
    int64_t x[16], pi[N_I];
    double pf[N_F];
    int64_t c = cfg_idx[p];
    if (c < 0 || c >= n_configs || spec_idx[p] < 0 || spec_idx[p] >= n_specs) {
      set_error(pi, pf);
      status[p] = ST_INDEX;
      for (int k = 0; k < N_I; ++k) ints[(int64_t)k * n_pairs + p] = pi[k];
      for (int k = 0; k < N_F; ++k) flts[(int64_t)k * n_pairs + p] = pf[k];
      continue;
    }
    load_config(fields, field_ld, c, nf, x);
    const int32_t *rag = NULL;
    if (ragged_off && ragged_off[c] >= 0) rag = ragged + ragged_off[c];
    if (fam == FAM_ATTENTION && !rag) {
      set_error(pi, pf);
      status[p] = ST_DIM;
    } else {
      status[p] = (uint8_t)featurize_pair(fam, x, rag, &specs[spec_idx[p]], flags, pi, pf);
    }
    for (int k = 0; k < N_I; ++k) ints[(int64_t)k * n_pairs + p] = pi[k];
    for (int k = 0; k < N_F; ++k) flts[(int64_t)k * n_pairs + p] = pf[k];
  }
  return 0;
}

/* Per-SM arrays of the cyclic schedule for the test suite's partition checks:
 * sm_of[t] = SM of task t (Eq.2 partition). */
void orc_schedule_rr(int64_t n_tasks, int64_t n_sm, int64_t *sm_of) {
  for (int64_t t = 0; t < n_tasks; ++t) sm_of[t] = t % n_sm;
}

/* The two non-cyclic schedulers on an explicit cost list (tests pin them with
 * SPEC S:191-193's examples): sm_of[t] (and worker_of[t] for MINHEAP). */
void orc_schedule_greedy(const int64_t *cost, int64_t n, int64_t n_sm, int64_t occ, int64_t *sm_of) {
  i128 *c = (i128 *)malloc((size_t)(n ? n : 1) * sizeof(i128));
  for (int64_t t = 0; t < n; ++t) c[t] = cost[t];
  greedy_assign(c, n, n_sm, occ, sm_of);
  free(c);
}
void orc_schedule_minheap(const int64_t *cost, int64_t n, int64_t n_sm, int64_t occ, int64_t *worker_of,
                          int64_t *sm_of) {
  i128 *c = (i128 *)malloc((size_t)(n ? n : 1) * sizeof(i128));
  for (int64_t t = 0; t < n; ++t) c[t] = cost[t];
  minheap_assign(c, n, n_sm, occ, worker_of, sm_of);
  free(c);
}

/* Per-task demand list of one config on one spec (tests: conservation,
 * monotone kv extent, brute-force comparisons).  Writes up to cap tasks as
 * [ops_T, ops_F, ops_X, bytes] rows; returns the task count, or -status. */
int64_t orc_task_list(int fam, const int32_t *fields, int64_t field_ld, int64_t c,
                      const int32_t *rag, int flags, int64_t n_sm, int64_t *out, int64_t cap) {
  int64_t x[16];
  i128 T = 0, U = 0;
  load_config(fields, field_ld, c, n_fields_of(fam), x);
  int st = validate(fam, x, rag, &T, &U);
  if (st != ST_OK) return -st;
  if (T > cap) return -(int64_t)100;
  orc_sched s;
  memset(&s, 0, sizeof s);
  /* one "SM" per task slot, so sm_sum rows are the per-task demands in order */
  s.n_sm = T > 0 ? (int64_t)T : 1;
  (void)n_sm;
  s.sm_sum = (i128 *)calloc((size_t)s.n_sm * 4, sizeof(i128));
  s.sm_count = (int64_t *)calloc((size_t)s.n_sm, sizeof(int64_t));
  switch (fam) {
    case FAM_GEMM: decompose_gemm(x, flags, &s); break;
    case FAM_SCALED: decompose_scaled_mm(x, &s); break;
    case FAM_SPLITK: decompose_gemm_splitk(x, &s); break;
    case FAM_MOE: decompose_moe(x, rag, flags, &s); break;
    case FAM_RMSNORM: decompose_rmsnorm(x, &s); break;
    case FAM_SILU: decompose_silu(x, &s); break;
    case FAM_ATTENTION: decompose_attention(x, rag, flags, &s); break;
  }
  for (int64_t k = 0; k < s.t * 4; ++k) out[k] = (int64_t)s.sm_sum[k];
  int64_t n = s.t;
  free(s.sm_sum);
  free(s.sm_count);
  return n;
}

/* Task count T and (attention) the per-kv-head kv-unit sum U of config c, as
 * validate() counts them; returns the domain status (tests: the GPU's
 * exact-range limits, include/synperf.h SP_PAIR_E_RANGE, are asserted where
 * these cross 2^31 and 2^32).  Saturated counts read as INT64_MAX. */
int orc_count(int fam, const int32_t *fields, int64_t field_ld, int64_t c, const int32_t *rag, int64_t *T,
              int64_t *U) {
  int64_t x[16];
  i128 t = 0, u = 0;
  load_config(fields, field_ld, c, n_fields_of(fam), x);
  int st = validate(fam, x, rag, &t, &u);
  *T = t > (i128)INT64_LIM ? INT64_LIM : (int64_t)t;
  *U = u > (i128)INT64_LIM ? INT64_LIM : (int64_t)u;
  return st;
}

/* ---------------- O8-O11 Performance Estimator ---------------- */

/* Host fp32 model description (same arrays the C-ABI's sp_mlp_desc points at). */
typedef struct {
  int32_t family, n_in, precision, pad_;
  const float *mu, *sigma;          /* [n_in] normalisation stats (R17) */
  const float *w1, *b1;             /* [256][n_in], [256] */
  const float *g1, *be1, *m1, *v1;  /* BN1 gamma, beta, running mean, var [256] */
  const float *w2, *b2;             /* [128][256], [128] */
  const float *g2, *be2, *m2, *v2;
  const float *w3, *b3;             /* [64][128], [64] */
  const float *g3, *be3, *m3, *v3;
  const float *w4;                  /* [64] */
  float b4, bn_eps;
} orc_mlp;

/* O8: Table IV order: per pipe present (Tensor, FMA, XU):
 * [total ops, C^GPU, max-SM ops, C^SM], then the 7 MIO features. */
static int build_input(int fam, const int64_t *ints, const double *flts, double *v) {
  int pipes = pipes_of(fam), n = 0;
  for (int p = 0; p < 3; ++p) {
    if (!(pipes & (1 << p))) continue;
    v[n++] = (double)ints[I_TOT_T + p];
    v[n++] = flts[F_CG_T + p];
    v[n++] = (double)ints[I_MAX_T + p];
    v[n++] = flts[F_CS_T + p];
  }
  v[n++] = (double)ints[I_BYTES];
  v[n++] = flts[F_GLOB_G];
  v[n++] = flts[F_L2_G];
  v[n++] = (double)ints[I_BYTES_MAX];
  v[n++] = flts[F_GLOB_S];
  v[n++] = flts[F_L2_S];
  v[n++] = flts[F_SMEM_S];
  return n;
}

/* One hidden layer, unfused (O10): a = W h + b; r = max(a,0);
 * out = gamma (r - mean) / sqrt(var + eps) + beta; dropout = identity (eval). */
static void hidden_layer(int n_out, int n_in, const float *w, const float *b, const float *g,
                         const float *be, const float *m, const float *var, double eps,
                         const double *h, double *out) {
  for (int o = 0; o < n_out; ++o) {
    double a = (double)b[o];
    for (int k = 0; k < n_in; ++k) a += (double)w[(int64_t)o * n_in + k] * h[k];
    double r = a > 0.0 ? a : 0.0;
    out[o] = (double)g[o] * (r - (double)m[o]) / sqrt((double)var[o] + eps) + (double)be[o];
  }
}

/* O9-O11 for one feature vector v[n_in]; returns the logit z. */
static double mlp_logit(const orc_mlp *md, const double *v) {
  double x[16], h1[256], h2[128], h3[64];
  for (int i = 0; i < md->n_in; ++i) {
    double sd = (double)md->sigma[i] > 1e-8 ? (double)md->sigma[i] : 1e-8;
    x[i] = (log1p(v[i]) - (double)md->mu[i]) / sd;
  }
  double eps = (double)md->bn_eps;
  hidden_layer(256, md->n_in, md->w1, md->b1, md->g1, md->be1, md->m1, md->v1, eps, x, h1);
  hidden_layer(128, 256, md->w2, md->b2, md->g2, md->be2, md->m2, md->v2, eps, h1, h2);
  hidden_layer(64, 128, md->w3, md->b3, md->g3, md->be3, md->m3, md->v3, eps, h2, h3);
  double z = (double)md->b4;
  for (int k = 0; k < 64; ++k) z += (double)md->w4[k] * h3[k];
  return z;
}

/*
 * Batched prediction from oracle features (ints/flts SoA as written by
 * orc_featurize).  efficiency e = 1/(1+exp(-z)) (sigmoid);
 * latency_us = t_theory / e.  Status != 0 -> NaN.
 */
int orc_predict(const orc_mlp *md, int64_t n_pairs, const int64_t *ints, const double *flts,
                const uint8_t *status, double *latency_us, double *efficiency, double *logit,
                int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
  for (int64_t p = 0; p < n_pairs; ++p) {
    int64_t pi[N_I];
    double pf[N_F], v[16];
    for (int k = 0; k < N_I; ++k) pi[k] = ints[(int64_t)k * n_pairs + p];
    for (int k = 0; k < N_F; ++k) pf[k] = flts[(int64_t)k * n_pairs + p];
    if (status[p] != ST_OK) {
      latency_us[p] = NAN;
      if (efficiency) efficiency[p] = NAN;
      if (logit) logit[p] = NAN;
      continue;
    }
    build_input(md->family, pi, pf, v);
    double z = mlp_logit(md, v);
    double e = 1.0 / (1.0 + exp(-z));
    latency_us[p] = pf[F_TTHEORY] / e;
    if (efficiency) efficiency[p] = e;
    if (logit) logit[p] = z;
  }
  return 0;
}

/* Normalised MLP input of one pair (tests: compare against torch.nn). */
int orc_mlp_input(const orc_mlp *md, const int64_t *pi, const double *pf, double *x_out) {
  double v[16];
  int n = build_input(md->family, pi, pf, v);
  for (int i = 0; i < n; ++i) {
    double sd = (double)md->sigma[i] > 1e-8 ? (double)md->sigma[i] : 1e-8;
    x_out[i] = (log1p(v[i]) - (double)md->mu[i]) / sd;
  }
  return n;
}

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
