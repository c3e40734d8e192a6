"""Oracle of the end-to-end serving-iteration composition (SURVEY §8(f) NEXT-1,
BASELINE config 4): a plain, slow, literal CPU implementation.

TEST INFRASTRUCTURE ONLY (like oracle/oracle.py): tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / `--impl reference` legs are the only permitted
callers.  It shares no code with paper_2601_14910_b200/; both sides consume the
request traces of workloads/gen.py.

What it follows
---------------
* PAPER §V-D: a Workload Generator "creates a sequence of kernel
  invocations that represents a real inference scenario"; "we assume sequential
  kernel execution without overlap"; the end-to-end latency is "calculated by
  summing all predicted kernel durations".
* PAPER §V-D: communication kernels (All-Reduce for TP, Send/Recv for
  PP) are estimated by a data-driven regression over profiled
  (volume, latency) points; SPEC S:561-566 reads it as piecewise-linear
  interpolation in log(bytes), clamped at the ends.
* SPEC S:556 (generate_trace): per layer RMSNorm -> QKV GEMM -> Attention ->
  O GEMM -> AllReduce(tp>1) -> RMSNorm -> GateUp GEMM -> SiLU&Mul -> Down GEMM
  -> AllReduce(tp>1); final RMSNorm + LM-head GEMM once per forward pass; PP
  inserts Send/Recv at stage boundaries.  S:573: decode step k uses
  kvlen = input_len + k.
* Readings E1..E9 of DESIGN.md §3b (where the paper is silent): step structure,
  token counts, GEMM/attention tiling, comm bytes.

Every invocation of every layer of every step is materialised in template
order, featurised and predicted on its own through the fp64 oracle
(oracle/oracle.py), and summed in fp64 in that order.  No deduplication, no
closed forms.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from workloads.gen import (ATTENTION, BF16, GEMM, RMSNORM, SILU_MUL, make_batch)

# categories of the breakdown ("per-category shares", Table I)
CAT_GEMM, CAT_ATTENTION, CAT_RMSNORM, CAT_SILU, CAT_COMM = 0, 1, 2, 3, 4
N_CAT = 5
CAT_OF_FAMILY = {GEMM: CAT_GEMM, ATTENTION: CAT_ATTENTION, RMSNORM: CAT_RMSNORM,
                 SILU_MUL: CAT_SILU}
BPE = 2  # bf16 activations (E9)


@dataclass
class ServingModel:
    """SPEC ModelConfig + ParallelConfig."""
    n_layers: int
    hidden: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    intermediate: int
    vocab: int
    tp: int = 1
    pp: int = 1


@dataclass
class Invocation:
    """One kernel invocation of the trace: a compute kernel (family + config
    fields, + (qlen, kvlen) requests for attention) or a collective."""
    kind: str  # "gemm", "attention", "rmsnorm", "silu_mul", "allreduce", "sendrecv"
    family: int = -1
    cols: dict = field(default_factory=dict)
    requests: list = field(default_factory=list)  # attention: [(qlen, kvlen), ...]
    comm_bytes: int = 0
    name: str = ""


def validate(m: ServingModel) -> None:
    """Divisibility rules ("errors: divisibility violations")."""
    for what, v in (("n_heads", m.n_heads), ("n_kv_heads", m.n_kv_heads),
                    ("intermediate", m.intermediate), ("vocab", m.vocab)):
        if v % m.tp:
            raise ValueError(f"{what}={v} not divisible by tp={m.tp}")
    if m.n_layers % m.pp:
        raise ValueError(f"n_layers={m.n_layers} not divisible by pp={m.pp}")
    if (m.n_heads // m.tp) % (m.n_kv_heads // m.tp):
        raise ValueError("heads per rank not divisible by kv heads per rank")


# ------------------------------------------------------------- kernel configs

def gemm_invocation(name: str, M: int, N: int, K: int) -> Invocation:
    """Reading E4: cuBLAS-like tile choice by the token count M.
    M <= 64: 64x128 tile, BK 64, 4 stages; M <= 256: 128x128, BK 64, 4 stages;
    otherwise 128x256, BK 64, 3 stages.  warps 4 if tm*tn <= 8192 else 8;
    regs 128 / 168 / 232 for tile areas <= 8192 / <= 16384 / larger."""
    if M <= 64:
        tm, tn, bk, stages = 64, 128, 64, 4
    elif M <= 256:
        tm, tn, bk, stages = 128, 128, 64, 4
    else:
        tm, tn, bk, stages = 128, 256, 64, 3
    area = tm * tn
    warps = 4 if area <= 8192 else 8
    if area <= 8192:
        regs = 128
    elif area <= 16384:
        regs = 168
    else:
        regs = 232
    cols = dict(M=[M], N=[N], K=[K], TM=[tm], TN=[tn], BK=[bk], STAGES=[stages],
                WARPS=[warps], REGS=[regs], SMEM=[0], DTYPE=[BF16])
    return Invocation("gemm", GEMM, cols, name=name)


def attention_invocation(m: ServingModel, requests: list, prefill: bool) -> Invocation:
    """Reading E5 (FlashInfer FA2).  Heads per TP rank nh/tp, nkv/tp.
    Prefill: causal, BQ 128, BKV 64, unsplit, 4 warps, 168 regs.
    Decode: qlen 1, BQ 16, BKV 64, non-causal, 4 warps, 64 regs, split-KV chunk
    1024 if n_active * nkv/tp < 128 else unsplit."""
    nh, nkv = m.n_heads // m.tp, m.n_kv_heads // m.tp
    bs = len(requests)
    if prefill:
        bq, bkv, chunk, causal, regs = 128, 64, 0, 1, 168
    else:
        bq, bkv, causal, regs = 16, 64, 0, 64
        chunk = 1024 if bs * nkv < 128 else 0
    cols = dict(BS=[bs], NH=[nh], NKV=[nkv], HD=[m.head_dim], BQ=[bq], BKV=[bkv],
                KV_CHUNK=[chunk], CAUSAL=[causal], WARPS=[4], REGS=[regs], SMEM=[0],
                DTYPE=[BF16])
    return Invocation("attention", ATTENTION, cols, list(requests), name="attention")


def rowwise_warps(dim: int) -> int:
    """Reading E6: one 16-byte vector (8 bf16) per thread, clamp(ceil(dim/256), 1, 32) warps."""
    w = -(-dim // 256)
    return max(1, min(32, w))


def rmsnorm_invocation(seq: int, dim: int, name: str) -> Invocation:
    cols = dict(SEQ=[seq], DIM=[dim], WARPS=[rowwise_warps(dim)], REGS=[32], SMEM=[0],
                DTYPE=[BF16])
    return Invocation("rmsnorm", RMSNORM, cols, name=name)


def silu_invocation(seq: int, dim: int) -> Invocation:
    cols = dict(SEQ=[seq], DIM=[dim], WARPS=[rowwise_warps(dim)], REGS=[32], SMEM=[0],
                DTYPE=[BF16])
    return Invocation("silu_mul", SILU_MUL, cols, name="silu_mul")


# ------------------------------------------------------------- trace generator

def forward_pass(m: ServingModel, requests: list, prefill: bool) -> list:
    """The kernel sequence of one forward pass (reading E1/E3).
    requests: [(qlen, kvlen)] of the active sequences in batch order."""
    M = sum(q for q, _ in requests)  # tokens processed this step (E3)
    n_seq = len(requests)
    h, tp = m.hidden, m.tp
    inv = []
    for layer in range(m.n_layers):
        if m.pp > 1 and layer > 0 and layer % (m.n_layers // m.pp) == 0:
            inv.append(Invocation("sendrecv", comm_bytes=M * h * BPE, name="sendrecv"))
        inv.append(rmsnorm_invocation(M, h, "input_norm"))
        inv.append(gemm_invocation("qkv", M, (m.n_heads + 2 * m.n_kv_heads) // tp * m.head_dim, h))
        inv.append(attention_invocation(m, requests, prefill))
        inv.append(gemm_invocation("o_proj", M, h, m.n_heads // tp * m.head_dim))
        if tp > 1:
            inv.append(Invocation("allreduce", comm_bytes=M * h * BPE, name="allreduce"))
        inv.append(rmsnorm_invocation(M, h, "post_attn_norm"))
        inv.append(gemm_invocation("gate_up", M, 2 * m.intermediate // tp, h))
        inv.append(silu_invocation(M, m.intermediate // tp))
        inv.append(gemm_invocation("down", M, h, m.intermediate // tp))
        if tp > 1:
            inv.append(Invocation("allreduce", comm_bytes=M * h * BPE, name="allreduce"))
    inv.append(rmsnorm_invocation(M, h, "final_norm"))
    inv.append(gemm_invocation("lm_head", n_seq, m.vocab // tp, h))  # last position per sequence
    return inv


def steps_of_trace(input_len, output_len) -> list:
    """Reading E2: a static batch.  Step 0 prefills every request
    (qlen = kvlen = input_len, causal).  Decode step k = 1 .. max(output_len)-1
    runs the requests with output_len > k, in batch order, each with qlen 1 and
    kvlen = input_len + k.  Returns [(prefill, [(qlen, kvlen), ...])]."""
    ins = [int(x) for x in input_len]
    outs = [int(x) for x in output_len]
    if not ins or len(ins) != len(outs) or min(ins) < 1 or min(outs) < 1:
        raise ValueError("a trace needs >= 1 request with input_len >= 1 and output_len >= 1")
    steps = [(True, [(q, q) for q in ins])]
    for k in range(1, max(outs)):
        steps.append((False, [(1, i + k) for i, o in zip(ins, outs) if o > k]))
    return steps


def generate_trace(m: ServingModel, input_len, output_len) -> list:
    """SPEC generate_trace: [[Invocation, ...] per step]."""
    validate(m)
    return [forward_pass(m, req, pf) for pf, req in steps_of_trace(input_len, output_len)]


# ------------------------------------------------------------- comm estimator

def predict_comm(points_bytes, points_us, nbytes: float) -> float:
    """SPEC predict_comm: piecewise-linear interpolation of latency
    in ln(bytes) over calibration points sorted by bytes; below the smallest
    point the smallest point's latency, above the largest the largest's
    (reading E7: clamped flat at both ends)."""
    xs = [float(b) for b in points_bytes]
    ys = [float(u) for u in points_us]
    if nbytes <= xs[0]:
        return ys[0]
    if nbytes >= xs[-1]:
        return ys[-1]
    for i in range(len(xs) - 1):
        if xs[i] <= nbytes <= xs[i + 1]:
            t = (math.log(nbytes) - math.log(xs[i])) / (math.log(xs[i + 1]) - math.log(xs[i]))
            return ys[i] + t * (ys[i + 1] - ys[i])
    raise AssertionError("unreachable")


# ------------------------------------------------------------- composition

def kernel_latency_fn(specs, models, orc):
    """Estimator per compute invocation: featurise the single config on every
    spec with the fp64 oracle (O1-O7), then the family's MLP (O8-O11).
    Returns f(inv) -> np.ndarray [n_specs] of latency_us."""

    def f(inv: Invocation) -> np.ndarray:
        if inv.family == ATTENTION:
            rag = []
            for q, kv in inv.requests:
                rag += [q, kv]
            b = make_batch(ATTENTION, inv.cols, ragged=rag, ragged_off=[0])
        else:
            b = make_batch(inv.family, inv.cols)
        feats = orc.featurize(b, specs)
        lat, _, _ = orc.predict(models[inv.family], feats)
        return lat

    return f


def comm_latency_fn(comm):
    """comm: {"bytes": [P], "allreduce_us": [G][P], "sendrecv_us": [G][P]} or None.
    Returns f(inv) -> np.ndarray [G]."""

    def f(inv: Invocation) -> np.ndarray:
        if comm is None:
            raise ValueError("trace has collectives but no comm model was given")
        table = comm["allreduce_us"] if inv.kind == "allreduce" else comm["sendrecv_us"]
        return np.array([predict_comm(comm["bytes"], row, inv.comm_bytes) for row in table])

    return f


def predict_e2e(trace: list, n_specs: int, kernel_fn, comm_fn):
    """SPEC predict_e2e: sequential sum of every invocation's
    predicted latency, per spec, in trace order (fp64).
    Returns (step_us [G][n_steps], total_us [G], breakdown [G][N_CAT])."""
    steps = np.zeros((n_specs, len(trace)), np.float64)
    cats = np.zeros((n_specs, N_CAT), np.float64)
    for s, invs in enumerate(trace):
        for inv in invs:
            if inv.kind in ("allreduce", "sendrecv"):
                lat = comm_fn(inv)
                cat = CAT_COMM
            else:
                lat = kernel_fn(inv)
                cat = CAT_OF_FAMILY[inv.family]
            for g in range(n_specs):
                steps[g, s] += lat[g]
                cats[g, cat] += lat[g]
    return steps, steps.sum(axis=1), cats
