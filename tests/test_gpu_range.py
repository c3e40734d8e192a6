"""The GPU kernels' exact-range limits (R22; include/synperf.h SP_PAIR_E_RANGE)
against the oracle, which has none.

The CUDA path keeps per-config counts in 32-bit registers: task count
T < 2^31, packed rows qlen*g < 2^31, M*topk < 2^31 and a per-kv-head kv-unit
sum U < 2^32.  The oracle computes the paper's answer whatever the size.  So:
  * just below a limit the GPU answers, and its record equals the oracle's
    (element by element where the oracle can enumerate the tasks in seconds,
    else its task count equals the oracle's count);
  * at or past a limit the GPU reports status 8 while the oracle's count is
    past the same bound (and the oracle still answers, status 0).
"""
import numpy as np
import pytest
import torch

from workloads import gen, specs

pytestmark = pytest.mark.gpu

I31, U32 = (1 << 31) - 1, (1 << 32) - 1


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_14910_b200 as sp

    return sp


@pytest.fixture(scope="module")
def ctx(sp):
    return sp.Context(0)


def gpu_record(sp, ctx, b, sa):
    sh = ctx.load_gpu_specs(sa)
    db = sp.DeviceBatch.from_host(b, ctx.torch_device)
    f = sp.Features.empty(b.family, len(sa) * b.n_configs, ctx.torch_device)
    ctx.featurize(db, sh, f, sp.cross(0, len(sa)))
    torch.cuda.synchronize()
    return sp.features_to_host(f)


def batch(family, rows, ragged=None):
    cols = {k: [r[k] for r in rows] for k in gen.FIELDS[family]}
    if ragged is None:
        return gen.make_batch(family, cols)
    flat, off = [], []
    for reqs in ragged:
        off.append(len(flat))
        for x in reqs:
            flat.extend(x if isinstance(x, tuple) else (x,))
    return gen.make_batch(family, cols, flat, off)


def check(sp, ctx, orc, b, expect_range, full):
    """expect_range[c]: the GPU must report status 8 for config c on every spec;
    full[c]: the oracle enumerates config c, compare the whole record."""
    sa = specs.paper_gpu_specs()
    gi, gf, gs = gpu_record(sp, ctx, b, sa)
    C = b.n_configs
    for c in range(C):
        st, T, U = orc.count(b, c)
        assert st == 0, (c, st)
        crosses = T > I31 or U > U32
        cols = np.arange(len(sa)) * C + c
        if expect_range[c]:
            assert (gs[cols] == 8).all(), (c, gs[cols])
        else:
            assert (gs[cols] == 0).all(), (c, gs[cols])
            assert (gi[0, cols] == T).all(), (c, gi[0, cols], T)
        if b.family == gen.ATTENTION:
            q = b.ragged[b.ragged_off[c]::2][: b.field("BS")[c]].astype(np.int64)
            g = int(b.field("NH")[c] // b.field("NKV")[c])
            crosses = crosses or (q * g > I31).any()
        if b.family == gen.FUSED_MOE:
            crosses = crosses or int(b.field("M")[c]) * int(b.field("TOPK")[c]) > I31
        assert crosses == expect_range[c], (c, T, U)
    idx = [c for c in range(C) if full[c]]
    if idx:
        ci = np.repeat(np.array(idx, np.int64)[None], len(sa), 0).ravel()
        si = np.repeat(np.arange(len(sa)), len(idx))
        o = orc.featurize(b, sa, cfg_idx=ci, spec_idx=si)
        assert (o.status == 0).all()  # the oracle answers past the GPU's limits too
        cols = si * C + ci
        keep = gs[cols] == 0
        assert np.array_equal(gi[:, cols][:, keep], o.ints[:, keep])
        np.testing.assert_allclose(gf[:, cols][:, keep].astype(np.float64), o.flts[:, keep], rtol=1e-5, atol=0)


def gemm_row(**kw):
    d = dict(M=1, N=1, K=16, TM=1, TN=1, BK=16, STAGES=1, WARPS=1, REGS=1, SMEM=0, DTYPE=0)
    d.update(kw)
    return d


def test_gemm_task_count_boundary(sp, ctx, orc):
    rows = [gemm_row(M=I31), gemm_row(M=1 << 30, N=2), gemm_row(M=I31, N=2), gemm_row(M=1 << 15, N=1 << 15)]
    check(sp, ctx, orc, batch(gen.GEMM, rows), [False, True, True, False], [False] * 4)


def test_scaled_mm_task_count_boundary(sp, ctx, orc):
    rows = [gemm_row(M=I31, DTYPE=3), gemm_row(M=1 << 30, N=2, DTYPE=3)]
    b = batch(gen.SCALED_MM, rows)
    sa = specs.paper_gpu_specs()
    gi, gf, gs = gpu_record(sp, ctx, b, sa)
    C = b.n_configs
    fp8 = sa["th_tensor_fp8"] > 0
    for c, rng in ((0, False), (1, True)):
        st, T, _ = orc.count(b, c)
        assert st == 0 and (T > I31) == rng
        s = gs[np.arange(len(sa)) * C + c]
        if rng:  # the config-level range check precedes the spec's FP8-rate check
            assert (s == 8).all()
        else:
            assert (s[~fp8] == 7).all() and (s[fp8] == 0).all()
            assert (gi[0, np.arange(len(sa))[fp8] * C + c] == T).all()


def test_splitk_task_count_boundary(sp, ctx, orc):
    row = dict(M=1 << 30, N=1, K=16, TM=1, TN=1, BK=16, SPLIT_K=1, STAGES=1, WARPS=1, REGS=1, SMEM=0, DTYPE=0)
    rows = [row, dict(row, K=32, SPLIT_K=2), dict(row, M=131072, N=131072, TM=16, TN=16, K=65536, SPLIT_K=64)]
    check(sp, ctx, orc, batch(gen.GEMM_SPLITK, rows), [False, True, True], [False] * 3)


def test_moe_boundaries(sp, ctx, orc):
    row = dict(M=(1 << 30) - 1, E=1, TOPK=2, H=16, N=16, BM=1 << 30, BN=16, BK=16, GROUP_M=1, STAGES=2,
               WARPS=4, REGS=64, SMEM=0, DTYPE=0)
    rows = [row,                                   # M*topk = 2^31 - 2: answered, enumerable
            dict(row, M=1 << 30),                  # M*topk = 2^31: range
            dict(row, M=(1 << 30) - 1, TOPK=1, BM=1, N=2, BN=1),  # T = 2^31 - 2
            dict(row, M=1 << 30, TOPK=1, BM=1, N=2, BN=1)]        # T = 2^31
    b = batch(gen.FUSED_MOE, rows)  # balanced split (no histogram)
    check(sp, ctx, orc, b, [False, True, False, True], [True, True, False, False])


def attn_row(**kw):
    # hd = 1 keeps every total < 2^63 (the record's own range) at these extents
    d = dict(BS=1, NH=8, NKV=1, HD=1, BQ=1 << 28, BKV=1 << 27, KV_CHUNK=0, CAUSAL=1, WARPS=4, REGS=64,
             SMEM=0, DTYPE=0)
    d.update(kw)
    return d


def test_attention_packed_rows_boundary(sp, ctx, orc):
    q0, q1 = (1 << 28) - 1, 1 << 28  # x g = 8: 2^31 - 8 and 2^31 packed rows
    rows = [attn_row(), attn_row(), attn_row(CAUSAL=0)]
    b = batch(gen.ATTENTION, rows, ragged=[[(q0, q0)], [(q1, q1)], [(q1, 5)]])
    check(sp, ctx, orc, b, [False, True, True], [True, True, True])


def test_attention_unit_sum_boundary(sp, ctx, orc):
    """Per-head kv units U = sum kv_eff/BKV just below and at/after 2^32, on
    the sparse path (T <= min N), the accumulator path (T = 200 > every N) and
    the 64-bit fold (nkv * U >= 2^32)."""
    kv2 = I31                        # 2 x (2^31 - 1) = 2^32 - 2
    kv200 = U32 // 200               # 200 x 21474836 = 4294967200
    r = dict(NH=1, NKV=1, BQ=1, BKV=1, CAUSAL=0)
    rows = [attn_row(BS=2, **r), attn_row(BS=3, **r),
            attn_row(BS=200, **r), attn_row(BS=201, **r),
            attn_row(BS=200, **dict(r, NH=2, NKV=2))]
    rag = [[(1, kv2)] * 2, [(1, kv2)] * 3, [(1, kv200)] * 200, [(1, kv200)] * 201, [(1, kv200)] * 200]
    check(sp, ctx, orc, batch(gen.ATTENTION, rows, ragged=rag), [False, True, False, True, False],
          [True, True, True, True, True])


def test_attention_task_count_boundary(sp, ctx, orc):
    """Per-head task count L = 2^31 (two requests of 2^30 q-blocks) and
    L * nkv = 2^31 (L = 2^30, nkv = 2): status 8 before any task is walked."""
    r = dict(NH=1, NKV=1, BQ=1, BKV=64, CAUSAL=0)
    rows = [attn_row(BS=2, **r), attn_row(BS=1, **dict(r, NH=2, NKV=2))]
    rag = [[(1 << 30, 1)] * 2, [(1 << 30, 1)]]
    check(sp, ctx, orc, batch(gen.ATTENTION, rows, ragged=rag), [True, True], [False, False])
