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


# ---------------------------------------------------------------- NEXT-3 gap diagnosis

@pytest.mark.parametrize("kind", ["cross", "list"])
def test_perf_gap_parity(sp, ctx, orc, kind):
    """sp_perf_gap vs oracle/gap.py: fp32 gap bit-exact, counts and histogram exact."""
    from oracle import gap as OG
    from workloads import models

    b = gen.gen_moe(400, 31)
    sa = specs.paper_gpu_specs()
    sh = ctx.load_gpu_specs(sa)
    db = sp.DeviceBatch.from_host(b, ctx.torch_device)
    G = len(sa)
    n = G * b.n_configs
    f = sp.Features.empty(b.family, n, ctx.torch_device)
    ctx.featurize(db, sh, f)
    p80m = ctx.load_model(models.random_mlp(b.family, 77), "fp16")
    lat = torch.empty(n, dtype=torch.float32, device="cuda")
    eff = torch.empty(n, dtype=torch.float32, device="cuda")
    ctx.predict(p80m, f, lat, eff)
    _, gf, gs = sp.features_to_host(f)
    rng = np.random.default_rng(9)
    meas = (gf[11] / rng.uniform(0.05, 1.0, n)).astype(np.float32)  # measured latencies
    meas[rng.uniform(0, 1, n) < 0.01] = 0.0  # some invalid measurements
    meas_d = torch.from_numpy(meas).cuda()
    if kind == "cross":
        gap, counts, hist = ctx.perf_gap(f, eff, meas_d, sp.cross(0, G), n_configs=b.n_configs, n_bins=64)
        spec_of = np.arange(n) // b.n_configs
    else:
        spec_of = rng.integers(0, 5, n)
        pl = sp.pair_list(torch.arange(n, dtype=torch.int64).cuda(),
                          torch.from_numpy(spec_of.astype(np.int32)).cuda())
        gap, counts, hist = ctx.perf_gap(f, eff, meas_d, pl, n_specs=5, n_bins=64)
    torch.cuda.synchronize()
    og, oc, oh = OG.perf_gap(gf[11], gs, eff.cpu().numpy(), meas, spec_of, int(counts.shape[0]), n_bins=64)
    assert np.array_equal(gap.cpu().numpy(), og, equal_nan=True)
    assert np.array_equal(counts.cpu().numpy(), oc)
    assert np.array_equal(hist.cpu().numpy(), oh)
    assert oc[:, 1].sum() > 0 and oc[:, 0].sum() < n


# ---------------------------------------------------------------- R24 split-KV planner

def planner_batch(seed, n=80):
    """Decode configs, a third with kv_chunk = -1 (planner), mixed with fixed chunks."""
    b = gen.gen_attention(0, n, seed, max_bs=12, kvlen_max=8000)
    ch = b.fields[gen.FIELDS[gen.ATTENTION].index("KV_CHUNK")]
    ch[::3] = -1
    return b


@pytest.mark.parametrize("mode", ["rr", "greedy", "minheap"])
def test_planner_parity_cross(sp, ctx, orc, mode):
    b = planner_batch(95)
    base = specs.paper_gpu_specs()
    sa = np.concatenate([base, np.concatenate([tiny_spec(n, o) for n, o in ((8, 1), (33, 2), (64, 1))])])
    check(run(sp, ctx, b, sa, mode), orc.featurize(b, sa, flags=oflag(orc, mode)))


def test_planner_parity_list(sp, ctx, orc):
    b = planner_batch(96)
    sa = specs.paper_gpu_specs()
    rng = np.random.default_rng(5)
    ci, si = rng.integers(0, b.n_configs, 400), rng.integers(0, len(sa), 400)
    check(run(sp, ctx, b, sa, "rr", (ci, si)), orc.featurize(b, sa, ci, si))
