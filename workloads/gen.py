"""Seeded synthetic config generators for the BASELINE.json workloads.

Input-only module: it draws kernel configurations X (Eq.1 inputs) with
the shapes and ranges of the paper's datasets (§V-B) and the config
recipes of SURVEY.md §8(d).  It contains none of the method's arithmetic — no
tiles, tasks, schedules or features — so that the CUDA path and the CPU oracle
share nothing but their inputs.

A batch is a structure of arrays: `fields` is int32 [n_fields, n_configs] in the
per-family field order below (the same order include/synperf.h documents), plus
an optional ragged int32 array addressed by int64 per-config offsets:
  * ATTENTION: (qlen, kvlen) pairs, bs of them per config, interleaved.
  * FUSED_MOE: E per-expert token counts, or offset -1 for the balanced split.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# ---- family codes (include/synperf.h sp_family) ----
GEMM, ATTENTION, FUSED_MOE, RMSNORM, SILU_MUL, SCALED_MM, GEMM_SPLITK = 0, 1, 2, 3, 4, 5, 6
FAMILY_NAMES = {GEMM: "gemm", ATTENTION: "attention", FUSED_MOE: "fused_moe",
                RMSNORM: "rmsnorm", SILU_MUL: "silu_mul", SCALED_MM: "scaled_mm",
                GEMM_SPLITK: "gemm_splitk"}

# ---- dtype codes (include/synperf.h sp_dtype) ----
BF16, FP16, FP32, FP8 = 0, 1, 2, 3

FIELDS = {
    GEMM: ["M", "N", "K", "TM", "TN", "BK", "STAGES", "WARPS", "REGS", "SMEM", "DTYPE"],
    ATTENTION: ["BS", "NH", "NKV", "HD", "BQ", "BKV", "KV_CHUNK", "CAUSAL",
                "WARPS", "REGS", "SMEM", "DTYPE"],
    FUSED_MOE: ["M", "E", "TOPK", "H", "N", "BM", "BN", "BK", "GROUP_M", "STAGES",
                "WARPS", "REGS", "SMEM", "DTYPE"],
    RMSNORM: ["SEQ", "DIM", "WARPS", "REGS", "SMEM", "DTYPE"],
    SILU_MUL: ["SEQ", "DIM", "WARPS", "REGS", "SMEM", "DTYPE"],
    SCALED_MM: ["M", "N", "K", "TM", "TN", "BK", "STAGES", "WARPS", "REGS", "SMEM", "DTYPE"],
    GEMM_SPLITK: ["M", "N", "K", "TM", "TN", "BK", "SPLIT_K", "STAGES", "WARPS", "REGS", "SMEM",
                  "DTYPE"],
}
N_FIELDS = {f: len(v) for f, v in FIELDS.items()}


@dataclass
class ConfigBatch:
    family: int
    fields: np.ndarray  # int32 [n_fields, n_configs], C-contiguous
    ragged: np.ndarray | None = None  # int32 [n_ragged]
    ragged_off: np.ndarray | None = None  # int64 [n_configs]

    @property
    def n_configs(self) -> int:
        return int(self.fields.shape[1])

    def field(self, name: str) -> np.ndarray:
        return self.fields[FIELDS[self.family].index(name)]

    def subset(self, idx) -> "ConfigBatch":
        """Configs idx (an index array), with ragged data re-packed."""
        idx = np.asarray(idx, dtype=np.int64)
        fields = np.ascontiguousarray(self.fields[:, idx])
        if self.ragged is None:
            return ConfigBatch(self.family, fields)
        off = self.ragged_off[idx]
        ln = np.where(off >= 0, ragged_lengths(self)[idx], 0)
        start = np.zeros(len(idx), dtype=np.int64)
        start[1:] = np.cumsum(ln)[:-1]
        total = int(ln.sum())
        src = np.repeat(off - start, ln) + np.arange(total, dtype=np.int64)
        ragged = self.ragged[src].astype(np.int32)
        new_off = np.where(off >= 0, start, -1).astype(np.int64)
        return ConfigBatch(self.family, fields, ragged, new_off)


def ragged_lengths(b: ConfigBatch) -> np.ndarray:
    if b.family == ATTENTION:
        return 2 * b.field("BS").astype(np.int64)
    if b.family == FUSED_MOE:
        return np.where(b.ragged_off >= 0, b.field("E").astype(np.int64), 0)
    return np.zeros(b.n_configs, np.int64)


def _logu_int(rng, lo, hi, n):
    """Integers log-uniform on [lo, hi] (inclusive)."""
    v = np.exp(rng.uniform(np.log(lo), np.log(hi + 1), n))
    return np.clip(np.floor(v), lo, hi).astype(np.int64)


def _pack(family, cols: dict, n) -> np.ndarray:
    out = np.zeros((N_FIELDS[family], n), dtype=np.int32)
    for i, name in enumerate(FIELDS[family]):
        out[i] = np.asarray(cols.get(name, 0), dtype=np.int64)
    return out


# GEMM tile menu of SURVEY §8(d) config 1: (tm, tn) with warps/regs by tile area
_GEMM_TILES = np.array([(64, 64), (64, 128), (128, 64), (128, 128), (128, 256), (256, 128)])


def _gemm_tiles(rng, n):
    t = _GEMM_TILES[rng.integers(0, len(_GEMM_TILES), n)]
    tm, tn = t[:, 0], t[:, 1]
    area = tm * tn
    warps = np.where(area <= 8192, 4, 8)
    regs = np.where(area <= 4096, 128, np.where(area <= 8192, 168, 232))
    bk = rng.choice([32, 64], n)
    stages = rng.choice([3, 4, 5], n)
    return tm, tn, bk, stages, warps, regs


def gen_gemm(n: int, seed: int, m_range=(2, 131072), n_range=(384, 152064),
             k_range=(256, 53248)) -> ConfigBatch:
    """BASELINE config 1 recipe: GEMM ranges of §V-B, log-uniform."""
    rng = np.random.default_rng(seed)
    M = _logu_int(rng, *m_range, n)
    N = _logu_int(rng, *n_range, n)
    K = _logu_int(rng, *k_range, n)
    tm, tn, bk, stages, warps, regs = _gemm_tiles(rng, n)
    cols = dict(M=M, N=N, K=K, TM=tm, TN=tn, BK=bk, STAGES=stages, WARPS=warps,
                REGS=regs, SMEM=0, DTYPE=BF16)
    return ConfigBatch(GEMM, _pack(GEMM, cols, n))


def gen_attention(n_prefill: int, n_decode: int, seed: int, max_bs=16,
                  qlen_max=20097, kvlen_max=20481, groups=(1, 2, 4, 8, 16)) -> ConfigBatch:
    """BASELINE config 2 recipe, ranges of §V-B.

    bs ~ U{1..16}; nkv in {1,2,4,8}; group g in {1,2,4,8,16}, nh = nkv*g in [2,128];
    hd in {64,128}.  Prefill (causal): per request qlen ~ logU[1, 20097],
    kvlen ~ U[qlen, 20481] ("vary randomly within each batch");
    BQ in {64,128}, BKV in {32,64}, unsplit.  Decode: qlen = 1,
    kvlen ~ logU[4, 20481], BQ = 16, BKV in {32,64}, kv_chunk in {0,256,...,2048}.
    Configs are prefill first, then decode (callers shuffle before sharding).
    `groups` replaces the GQA group menu (tests: groups that do not divide BQ,
    e.g. Qwen2.5-14B's 40/8 = 5).
    """
    rng = np.random.default_rng(seed)
    n = n_prefill + n_decode
    bs = rng.integers(1, max_bs + 1, n)
    nkv = rng.choice([1, 2, 4, 8], n)
    groups = list(groups)
    g = rng.choice(groups, n)
    bad = (nkv * g) < 2
    while bad.any():
        g[bad] = rng.choice(groups, int(bad.sum()))
        bad = (nkv * g) < 2
    nh = nkv * g
    hd = rng.choice([64, 128], n)
    is_pf = np.arange(n) < n_prefill
    bq = np.where(is_pf, rng.choice([64, 128], n), 16)
    bkv = rng.choice([32, 64], n)
    chunk = np.where(is_pf, 0, rng.choice([0, 256, 512, 1024, 2048], n))
    causal = is_pf.astype(np.int64)
    warps = 4
    regs = np.where(is_pf, 128, 64)
    total = int(bs.sum())
    req_pf = np.repeat(is_pf, bs)
    q_pf = _logu_int(rng, 1, qlen_max, total)
    qlen = np.where(req_pf, q_pf, 1)
    kv_pf = qlen + np.floor(rng.uniform(0, 1, total) * (kvlen_max - qlen + 1)).astype(np.int64)
    kv_pf = np.clip(kv_pf, qlen, kvlen_max)
    kv_dec = _logu_int(rng, 4, kvlen_max, total)
    kvlen = np.where(req_pf, kv_pf, kv_dec)
    ragged = np.empty(2 * total, dtype=np.int32)
    ragged[0::2] = qlen
    ragged[1::2] = kvlen
    off = np.zeros(n, dtype=np.int64)
    off[1:] = np.cumsum(2 * bs)[:-1]
    cols = dict(BS=bs, NH=nh, NKV=nkv, HD=hd, BQ=bq, BKV=bkv, KV_CHUNK=chunk,
                CAUSAL=causal, WARPS=warps, REGS=regs, SMEM=0, DTYPE=BF16)
    return ConfigBatch(ATTENTION, _pack(ATTENTION, cols, n), ragged, off)


def gen_moe(n: int, seed: int, zipf_a=1.1) -> ConfigBatch:
    """BASELINE config 3 recipe: fused-MoE space of §V-B x Triton
    knobs of §VII-C.  Half the configs use the balanced split (offset
    -1), half carry a Zipf(1.1) per-expert histogram summing to M*topk."""
    rng = np.random.default_rng(seed)
    M = _logu_int(rng, 2, 8192, n)
    E = rng.choice([8, 16, 32, 64, 128], n)
    topk = rng.choice([2, 4, 6, 8], n)
    H = rng.choice([1024, 2048, 3072, 4096], n)
    N = rng.choice([512, 768, 1024, 1536, 2048, 3072], n)
    bm = rng.choice([16, 32, 64, 128], n)
    bn = rng.choice([32, 64, 128, 256], n)
    bk = rng.choice([32, 64, 128], n)
    gm = rng.choice([1, 8, 16, 32, 64], n)
    stages = rng.choice([2, 3, 4, 5], n)
    warps = rng.choice([4, 8], n)
    regs = rng.choice([96, 128, 168, 255], n)
    use_hist = rng.uniform(0, 1, n) < 0.5
    off = np.full(n, -1, dtype=np.int64)
    chunks = []
    pos = 0
    for c in np.nonzero(use_hist)[0]:
        e = int(E[c])
        w = 1.0 / np.arange(1, e + 1) ** zipf_a
        w = w[rng.permutation(e)]
        h = rng.multinomial(int(M[c] * topk[c]), w / w.sum())
        off[c] = pos
        pos += e
        chunks.append(h)
    ragged = (np.concatenate(chunks) if chunks else np.zeros(0)).astype(np.int32)
    cols = dict(M=M, E=E, TOPK=topk, H=H, N=N, BM=bm, BN=bn, BK=bk, GROUP_M=gm,
                STAGES=stages, WARPS=warps, REGS=regs, SMEM=0, DTYPE=BF16)
    return ConfigBatch(FUSED_MOE, _pack(FUSED_MOE, cols, n), ragged, off)


def gen_scaled_mm(n: int, seed: int) -> ConfigBatch:
    """FP8 Scaled MM (block-wise quantisation) space of §V-B:
    M ~ logU[2, 131072], N ~ logU[384, 8192], K ~ logU[256, 8192]; CUTLASS
    block-scaled tiles (tm, tn) in {64x128, 128x128, 128x256}, BK 128, 3-5 stages."""
    rng = np.random.default_rng(seed)
    M = _logu_int(rng, 2, 131072, n)
    N = _logu_int(rng, 384, 8192, n)
    K = _logu_int(rng, 256, 8192, n)
    tiles = np.array([(64, 128), (128, 128), (128, 256)])[rng.integers(0, 3, n)]
    area = tiles[:, 0] * tiles[:, 1]
    cols = dict(M=M, N=N, K=K, TM=tiles[:, 0], TN=tiles[:, 1], BK=128, STAGES=rng.choice([3, 4, 5], n),
                WARPS=np.where(area <= 8192, 4, 8), REGS=np.where(area <= 16384, 168, 232), SMEM=0,
                DTYPE=FP8)
    return ConfigBatch(SCALED_MM, _pack(SCALED_MM, cols, n))


def gen_gemm_splitk(n: int, seed: int) -> ConfigBatch:
    """Split-K GEMMs: the GEMM space of §V-B restricted to the shapes
    cuBLAS splits -- few output tiles against a long K (M ~ logU[1, 4096],
    N ~ logU[384, 16384], K ~ logU[1024, 53248]) -- with the GEMM tile set and
    SPLIT_K ~ U{1..16} (1 = no split; values above the k-tile count exercise
    the empty-slice rule of reading R25)."""
    rng = np.random.default_rng(seed)
    M = _logu_int(rng, 1, 4096, n)
    N = _logu_int(rng, 384, 16384, n)
    K = _logu_int(rng, 1024, 53248, n)
    tiles = np.array([(64, 64), (64, 128), (128, 64), (128, 128), (128, 256), (256, 128)])[rng.integers(0, 6, n)]
    area = tiles[:, 0] * tiles[:, 1]
    cols = dict(M=M, N=N, K=K, TM=tiles[:, 0], TN=tiles[:, 1], BK=rng.choice([32, 64], n),
                SPLIT_K=rng.integers(1, 17, n), STAGES=rng.choice([3, 4, 5], n),
                WARPS=np.where(area <= 8192, 4, 8),
                REGS=np.where(area <= 8192, 128, np.where(area <= 16384, 168, 232)), SMEM=0,
                DTYPE=rng.choice([BF16, FP16], n))
    return ConfigBatch(GEMM_SPLITK, _pack(GEMM_SPLITK, cols, n))


def gen_rowwise(family: int, n: int, seed: int) -> ConfigBatch:
    """RMSNorm (seq in [2,131072], dim in [128,16384]) or SiLU&Mul
    (seq in [2,131072], dim in [768,106496]), log-uniform."""
    rng = np.random.default_rng(seed)
    seq = _logu_int(rng, 2, 131072, n)
    if family == RMSNORM:
        dim = _logu_int(rng, 128, 16384, n)
    else:
        dim = _logu_int(rng, 768, 106496, n)
    warps = rng.choice([4, 8, 16, 32], n)
    regs = rng.choice([32, 40, 64], n)
    cols = dict(SEQ=seq, DIM=dim, WARPS=warps, REGS=regs, SMEM=0, DTYPE=BF16)
    return ConfigBatch(family, _pack(family, cols, n))


# ---- serving shapes (public model cards; not in the paper) for configs 4/5 ----
MODEL_CARDS = {
    # layers, hidden, heads, kv heads, head dim, intermediate, vocab
    "llama3-8b": (32, 4096, 32, 8, 128, 14336, 128256),
    "qwen2.5-14b": (48, 5120, 40, 8, 128, 13824, 152064),
}


def gen_serving_gemms(n: int, seed: int) -> ConfigBatch:
    """BASELINE config 5 kernel side: GEMMs with serving (N, K) of Llama-3-8B /
    Qwen2.5-14B linear layers, M = tokens ~ logU[1, 16384], config-1 tile menu."""
    rng = np.random.default_rng(seed)
    shapes = []
    for (L, h, nh, nkv, hd, inter, vocab) in MODEL_CARDS.values():
        shapes += [((nh + 2 * nkv) * hd, h), (h, nh * hd), (2 * inter, h), (h, inter), (vocab, h)]
    shapes = np.array(shapes)
    pick = shapes[rng.integers(0, len(shapes), n)]
    M = _logu_int(rng, 1, 16384, n)
    tm, tn, bk, stages, warps, regs = _gemm_tiles(rng, n)
    cols = dict(M=M, N=pick[:, 0], K=pick[:, 1], TM=tm, TN=tn, BK=bk, STAGES=stages,
                WARPS=warps, REGS=regs, SMEM=0, DTYPE=BF16)
    return ConfigBatch(GEMM, _pack(GEMM, cols, n))


def make_batch(family: int, cols: dict, ragged=None, ragged_off=None) -> ConfigBatch:
    """Hand-built batch from per-field lists (tests, worked examples)."""
    n = len(next(iter(cols.values())))
    fields = _pack(family, cols, n)
    rg = None if ragged is None else np.asarray(ragged, dtype=np.int32)
    ro = None if ragged_off is None else np.asarray(ragged_off, dtype=np.int64)
    return ConfigBatch(family, fields, rg, ro)


def shuffle(b: ConfigBatch, seed: int) -> tuple[ConfigBatch, np.ndarray]:
    """Seeded permutation of configs (cost balance before sharding)."""
    perm = np.random.default_rng(seed).permutation(b.n_configs)
    return b.subset(perm), perm


# ---- BASELINE config 4: serving request traces (inputs of the E2E composition) ----

# (layers, hidden, heads, kv heads, head dim, intermediate, vocab) -> a dict per model
def serving_model(name: str, tp: int = 1, pp: int = 1) -> dict:
    L, h, nh, nkv, hd, inter, vocab = MODEL_CARDS[name]
    return dict(n_layers=L, hidden=h, n_heads=nh, n_kv_heads=nkv, head_dim=hd,
                intermediate=inter, vocab=vocab, tp=tp, pp=pp)


# §VI-E: arxiv_* inputs average 2,630 tokens, splitwise_* 982; outputs 5..4,056;
# static batches named arxiv_8 / splitwise_64 etc. (Table VIII)
TRACE_DATASETS = {"arxiv": 2630.0, "splitwise": 982.0}
TRACE_BATCHES = (8, 12, 16, 48, 64)


@dataclass
class RequestTraces:
    """R static batches of requests: batch r holds requests
    [req_off[r], req_off[r+1]) with input / output token counts."""
    req_off: np.ndarray  # int64 [R+1]
    input_len: np.ndarray  # int32 [n_requests]
    output_len: np.ndarray  # int32 [n_requests]

    @property
    def n_traces(self) -> int:
        return len(self.req_off) - 1

    def trace(self, r: int):
        a, b = int(self.req_off[r]), int(self.req_off[r + 1])
        return self.input_len[a:b], self.output_len[a:b]

    def subset(self, idx) -> "RequestTraces":
        ins, outs, off = [], [], [0]
        for r in idx:
            i, o = self.trace(int(r))
            ins.append(i)
            outs.append(o)
            off.append(off[-1] + len(i))
        return RequestTraces(np.array(off, np.int64), np.concatenate(ins).astype(np.int32),
                             np.concatenate(outs).astype(np.int32))


def gen_serving_traces(n_traces: int, seed: int, batches=TRACE_BATCHES, out_max: int = 4056,
                       in_max: int = 20000, sigma: float = 0.6) -> RequestTraces:
    """BASELINE config 4 traces: trace r is a static batch of size
    batches[r % len(batches)] drawn from dataset arxiv (even r) or splitwise
    (odd r).  Input lengths ~ lognormal with the dataset's mean,
    clipped to [16, in_max]; output lengths ~ logU[5, out_max]."""
    rng = np.random.default_rng(seed)
    names = list(TRACE_DATASETS)
    ins, outs, off = [], [], [0]
    for r in range(n_traces):
        bs = int(batches[r % len(batches)])
        mean = TRACE_DATASETS[names[r % len(names)]]
        mu = np.log(mean) - sigma * sigma / 2
        i = np.clip(np.round(rng.lognormal(mu, sigma, bs)), 16, in_max).astype(np.int32)
        o = _logu_int(rng, 5, out_max, bs).astype(np.int32)
        ins.append(i)
        outs.append(o)
        off.append(off[-1] + bs)
    return RequestTraces(np.array(off, np.int64), np.concatenate(ins), np.concatenate(outs))


def make_traces(batches: list) -> RequestTraces:
    """Hand-built traces: [[(input_len, output_len), ...] per batch]."""
    ins, outs, off = [], [], [0]
    for b in batches:
        ins += [int(i) for i, _ in b]
        outs += [int(o) for _, o in b]
        off.append(off[-1] + len(b))
    return RequestTraces(np.array(off, np.int64), np.array(ins, np.int32), np.array(outs, np.int32))
