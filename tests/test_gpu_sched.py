"""GREEDY / MINHEAP scheduler modes on the GPU (sp_featurize_sched, through the
C-ABI) vs the fp64 oracle with the same scheduler.
Bar: integer slots and status bit-exact, float slots within 1e-5."""
import json
import os

import numpy as np
import pytest
import torch

from workloads import gen, specs

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "scheduler_examples.json")))


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_14910_b200 as sp

    return sp


@pytest.fixture(scope="module")
def ctx(sp):
    return sp.Context(0)


def oflag(orc, mode):
    return {"rr": 0, "greedy": orc.SCHED_GREEDY, "minheap": orc.SCHED_MINHEAP}[mode]


def run(sp, ctx, batch, sa, mode, pairs=None):
    sh = ctx.load_gpu_specs(sa)
    db = sp.DeviceBatch.from_host(batch, ctx.torch_device)
    if pairs is None:
        n, pr = len(sa) * batch.n_configs, sp.cross(0, len(sa))
    else:
        ci, si = pairs
        n = len(ci)
        pr = sp.pair_list(torch.from_numpy(np.asarray(ci, np.int64)).cuda(),
                          torch.from_numpy(np.asarray(si, np.int32)).cuda())
    f = sp.Features.empty(batch.family, n, ctx.torch_device)
    ctx.featurize(db, sh, f, pr, scheduler=mode)
    torch.cuda.synchronize()
    return sp.features_to_host(f)


def check(g, o):
    gi, gf, gs = g
    assert np.array_equal(gs, o.status)
    bad = np.nonzero((gi != o.ints).any(0))[0]
    assert bad.size == 0, f"int mismatch at {bad[:8]}: gpu {gi[:, bad[0]]} oracle {o.ints[:, bad[0]]}"
    ok = ~np.isnan(o.flts)
    assert np.array_equal(np.isnan(gf), ~ok)
    np.testing.assert_allclose(gf[ok].astype(np.float64), o.flts[ok], rtol=1e-5, atol=0)


def tiny_spec(n_sm, occ):
    s = specs.spec_by_name("A100")
    s["num_sms"] = n_sm
    s["max_ctas_per_sm"] = occ
    return s


@pytest.mark.parametrize("mode", ["greedy", "minheap"])
def test_attention_parity_cross(sp, ctx, orc, mode):
    b = gen.gen_attention(24, 24, 91, max_bs=5, qlen_max=3000, kvlen_max=6000)
    sa = specs.paper_gpu_specs()
    check(run(sp, ctx, b, sa, mode), orc.featurize(b, sa, flags=oflag(orc, mode)))


@pytest.mark.parametrize("mode", ["greedy", "minheap"])
def test_attention_parity_list_odd_sms(sp, ctx, orc, mode):
    b = gen.gen_attention(10, 10, 92, max_bs=4, qlen_max=2000, kvlen_max=4000)
    base = specs.paper_gpu_specs()
    sa = np.concatenate([base, np.concatenate([tiny_spec(n, o) for n, o in
                                               ((1, 1), (3, 2), (31, 3), (33, 1), (97, 4))])])
    rng = np.random.default_rng(4)
    ci = rng.integers(0, b.n_configs, 300)
    si = rng.integers(0, len(sa), 300)
    check(run(sp, ctx, b, sa, mode, (ci, si)), orc.featurize(b, sa, ci, si, flags=oflag(orc, mode)))


@pytest.mark.parametrize("k", range(5))
def test_attention_hand_cases(sp, ctx, k):
    g = GOLD["attention_greedy"]
    case = g["cases"][k]
    cols = {n: [v] for n, v in g["config"].items()}
    b = gen.make_batch(gen.ATTENTION, cols, ragged=np.array(g["requests"]).ravel(), ragged_off=[0])
    gi, _, gs = run(sp, ctx, b, tiny_spec(g["n_sm"], case["occ"]), case["mode"])
    assert gs[0] == 0
    assert gi[6, 0] == max(case["sm_units"]) * g["ops_per_unit"]


@pytest.mark.parametrize("mode", ["greedy", "minheap"])
@pytest.mark.parametrize("fam", [gen.GEMM, gen.FUSED_MOE, gen.RMSNORM, gen.SILU_MUL])
def test_uniform_families_equal_rr(sp, ctx, mode, fam):
    b = {gen.GEMM: lambda: gen.gen_gemm(200, 11), gen.FUSED_MOE: lambda: gen.gen_moe(200, 12),
         gen.RMSNORM: lambda: gen.gen_rowwise(gen.RMSNORM, 200, 13),
         gen.SILU_MUL: lambda: gen.gen_rowwise(gen.SILU_MUL, 200, 14)}[fam]()
    sa = specs.paper_gpu_specs()
    a, c = run(sp, ctx, b, sa, "rr"), run(sp, ctx, b, sa, mode)
    for x, y in zip(a, c):
        assert np.array_equal(x, y, equal_nan=True)


def test_unsupported_scheduler_state(sp, ctx):
    b = gen.gen_attention(2, 2, 93, max_bs=2, qlen_max=100, kvlen_max=200)
    s = tiny_spec(4096, 32)
    with pytest.raises(sp.SynPerfError, match="SP_E_UNSUPPORTED"):
        run(sp, ctx, b, s, "minheap")
