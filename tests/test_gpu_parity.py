"""GPU (CUDA path, through the C-ABI) vs the fp64 CPU oracle, element by element.

Bar (BASELINE.json north_star): every integer slot and status bit-exact;
fp32 float features within 1e-5 relative of the fp64 oracle; latency within
1e-5 relative for the fp32 MLP and 1e-2 for the 16-bit (fp16) tcgen05 MLP.
"""
import numpy as np
import pytest
import torch

from workloads import gen, models, specs

pytestmark = pytest.mark.gpu

FEAT_RTOL = 1e-5
LAT_RTOL_FP32 = 1e-5
LAT_RTOL_16 = 1e-2


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_14910_b200 as sp

    return sp


@pytest.fixture(scope="module")
def ctx(sp):
    return sp.Context(0)


def gpu_features(sp, ctx, batch, spec_arr, pairs=None, specs_handle=None):
    sh = specs_handle or ctx.load_gpu_specs(spec_arr)
    db = sp.DeviceBatch.from_host(batch, ctx.torch_device)
    if pairs is None:
        n = len(spec_arr) * batch.n_configs
        pr = sp.cross(0, len(spec_arr))
    else:
        ci, si = pairs
        n = len(ci)
        pr = sp.pair_list(torch.from_numpy(np.asarray(ci, np.int64)).cuda(),
                          torch.from_numpy(np.asarray(si, np.int32)).cuda())
    f = sp.Features.empty(batch.family, n, ctx.torch_device)
    ctx.featurize(db, sh, f, pr)
    torch.cuda.synchronize()
    return f, sp.features_to_host(f)


def assert_feature_parity(g, o, where=""):
    gi, gf, gs = g
    assert np.array_equal(gs, o.status), f"status mismatch {where}: {np.nonzero(gs != o.status)[0][:10]}"
    bad = np.nonzero((gi != o.ints).any(0))[0]
    assert bad.size == 0, f"int mismatch {where} at pairs {bad[:10]}: gpu {gi[:, bad[0]]} oracle {o.ints[:, bad[0]]}"
    of = o.flts
    nan_g, nan_o = np.isnan(gf), np.isnan(of)
    assert np.array_equal(nan_g, nan_o), f"NaN pattern mismatch {where}"
    ok = ~nan_o
    np.testing.assert_allclose(gf[ok].astype(np.float64), of[ok], rtol=FEAT_RTOL, atol=0,
                               err_msg=f"float features {where}")


FAMILY_BATCHES = {
    "gemm": lambda: gen.gen_gemm(700, 1001),
    "attention": lambda: gen.gen_attention(150, 150, 1002, max_bs=6, qlen_max=4000, kvlen_max=6000),
    # GQA groups that do not divide BQ (Qwen2.5-14B: 40/8 = 5): the general causal q_last path
    "attention_gqa": lambda: gen.gen_attention(200, 100, 1012, max_bs=6, qlen_max=4000, kvlen_max=6000,
                                               groups=(3, 5, 6, 12)),
    "moe": lambda: gen.gen_moe(600, 1003),
    "rmsnorm": lambda: gen.gen_rowwise(gen.RMSNORM, 500, 1004),
    "silu": lambda: gen.gen_rowwise(gen.SILU_MUL, 500, 1005),
    "scaled_mm": lambda: gen.gen_scaled_mm(500, 1006),
    "gemm_splitk": lambda: gen.gen_gemm_splitk(600, 1007),
}


@pytest.mark.parametrize("fam", list(FAMILY_BATCHES))
def test_featurize_cross_parity(sp, ctx, orc, fam):
    b = FAMILY_BATCHES[fam]()
    sa = specs.paper_gpu_specs()
    _, g = gpu_features(sp, ctx, b, sa)
    o = orc.featurize(b, sa)
    if fam == "scaled_mm":  # no FP8 tensor rate on sm_80/86 (A40, A100, RTX A6000)
        assert ((o.status == 0) | (o.status == 7)).all() and (o.status == 0).any()
    else:
        assert (o.status == 0).all()
    assert_feature_parity(g, o, fam)


@pytest.mark.parametrize("fam", list(FAMILY_BATCHES))
def test_featurize_list_parity(sp, ctx, orc, fam):
    b = FAMILY_BATCHES[fam]()
    sa = specs.paper_gpu_specs()
    rng = np.random.default_rng(7)
    n = 900
    ci = rng.integers(0, b.n_configs, n)
    si = rng.integers(0, len(sa), n)
    ci[:3] = [-1, b.n_configs, 0]   # out-of-range indices -> SP_PAIR_E_INDEX
    si[2] = len(sa)
    _, g = gpu_features(sp, ctx, b, sa, pairs=(ci, si))
    o = orc.featurize(b, sa, cfg_idx=ci, spec_idx=si)
    assert (o.status[:3] == 9).all()
    assert_feature_parity(g, o, fam + " list")


def odd_specs():
    """SM counts below, at and around the warp width, and a large one."""
    base = specs.paper_gpu_specs()
    out = np.concatenate([base[:4]] * 2)
    for i, n in enumerate([1, 7, 31, 32, 33, 64, 97, 1000]):
        out[i]["num_sms"] = n
    return out


@pytest.mark.parametrize("fam", list(FAMILY_BATCHES))
def test_featurize_odd_sm_counts(sp, ctx, orc, fam):
    b = FAMILY_BATCHES[fam]().subset(np.arange(60))
    sa = odd_specs()
    _, g = gpu_features(sp, ctx, b, sa)
    assert_feature_parity(g, orc.featurize(b, sa), fam + " odd SMs")


def test_attention_edge_cases(sp, ctx, orc):
    """qlen = 1, kvlen < BKV, nkv = nh, causal + split-KV, non-causal split-KV with one and
    several q-blocks per request, T < N, T multiple of N, long single requests, domain errors."""
    cols = {k: [] for k in gen.FIELDS[gen.ATTENTION]}
    rag, off = [], []

    def add(bs_reqs, **kw):
        d = dict(NH=8, NKV=2, HD=128, BQ=64, BKV=64, KV_CHUNK=0, CAUSAL=1, WARPS=4, REGS=128, SMEM=0,
                 DTYPE=0)
        d.update(kw)
        d["BS"] = len(bs_reqs) if "BS" not in kw else kw["BS"]
        for k in cols:
            cols[k].append(d[k])
        off.append(len(rag))
        for q, kv in bs_reqs:
            rag.extend([q, kv])

    add([(1, 3)])                              # qlen 1, kvlen < BKV
    add([(1, 1)], NH=4, NKV=4)                 # nkv = nh (group 1)
    add([(300, 5000), (2000, 2000)], KV_CHUNK=512)   # causal + split-KV (generic path)
    add([(77, 77)] * 5, KV_CHUNK=64, BQ=16)    # many small chunks
    add([(1, 20481)] * 16, NH=128, NKV=8, BQ=16, KV_CHUNK=2048, CAUSAL=0)  # decode, split
    # non-causal split-KV with several q-blocks per request (chunk index = task mod n_ch, a
    # FastDiv of n_ch = 5) next to one-q-block requests (chunk index = task index) in one config
    add([(300, 5000), (40, 3000), (1, 700), (64, 1024)], NH=8, NKV=2, BQ=64, KV_CHUNK=1024, CAUSAL=0)
    add([(1, 3000)] * 12 + [(33, 2500)], NH=8, NKV=2, BQ=16, KV_CHUNK=512, CAUSAL=0)
    add([(20097, 20481)], NH=32, NKV=8, BQ=128, BKV=32)   # long prefill
    add([(108 * 64, 108 * 64)], NH=1, NKV=1, CAUSAL=0)    # T = 108 q-blocks (multiple of N=108)
    add([(5, 9)], NH=6, NKV=4)                 # nh % nkv != 0 -> status 3
    add([(9, 5)])                              # causal kv < q -> status 5
    add([(0, 5)])                              # qlen 0 -> status 1
    add([(5, 5)], BQ=0)                        # tile 0 -> status 2
    add([(5, 5)], DTYPE=3)                     # fp8 -> status 7
    add([(5, 5)], WARPS=0)                     # resources -> status 6
    b = gen.make_batch(gen.ATTENTION, cols, rag, off)
    sa = np.concatenate([specs.paper_gpu_specs(), odd_specs()])
    _, g = gpu_features(sp, ctx, b, sa)
    o = orc.featurize(b, sa)
    assert set(np.unique(o.status)) >= {0, 1, 2, 3, 5, 6, 7}
    assert_feature_parity(g, o, "attention edges")


def test_splitk_refuses_non_cyclic_schedulers(sp, ctx):
    """Split-K tasks come in two sizes, so GREEDY / MINHEAP do not reduce to the
    cyclic closed form: the call is refused rather than answered with RR."""
    b = FAMILY_BATCHES["gemm_splitk"]().subset(np.arange(50))
    sa = specs.paper_gpu_specs()
    sh = ctx.load_gpu_specs(sa)
    db = sp.DeviceBatch.from_host(b, ctx.torch_device)
    f = sp.Features.empty(b.family, len(sa) * b.n_configs, ctx.torch_device)
    for sched in ("greedy", "minheap"):
        with pytest.raises(sp.SynPerfError):
            ctx.featurize(db, sh, f, scheduler=sched)


def test_splitk_edge_cases(sp, ctx, orc):
    """Split-K: the hand-derived golden cases (wrapping / disjoint task classes,
    empty slices), SPLIT_K far above the k-tile count, a single k-tile, one
    output tile, SPLIT_K = 0 (tile error)."""
    cols = {k: [] for k in gen.FIELDS[gen.GEMM_SPLITK]}

    def add(**kw):
        d = dict(M=256, N=256, K=1000, TM=128, TN=128, BK=64, SPLIT_K=3, STAGES=3, WARPS=8, REGS=168,
                 SMEM=0, DTYPE=0)
        d.update(kw)
        for k in cols:
            cols[k].append(d[k])

    for sk, k in ((3, 1000), (7, 1000), (20, 1000), (2, 960)):
        add(SPLIT_K=sk, K=k)
    add(SPLIT_K=100000, K=53248)
    add(SPLIT_K=16, K=64)                       # one k-tile: one slice
    add(M=1, N=1, SPLIT_K=5)                    # one output tile
    add(SPLIT_K=0)                              # SP_PAIR_E_TILE
    add(DTYPE=3)                                # FP8 is the Scaled MM family's: SP_PAIR_E_DTYPE
    b = gen.make_batch(gen.GEMM_SPLITK, cols)
    sa = np.concatenate([odd_specs(), specs.paper_gpu_specs()])
    sa[0]["num_sms"], sa[1]["num_sms"] = 5, 8
    _, g = gpu_features(sp, ctx, b, sa)
    o = orc.featurize(b, sa)
    assert set(np.unique(o.status)) == {0, 2, 7}  # the range limit: tests/test_gpu_range.py
    assert_feature_parity(g, o, "split-K edges")


def test_uniform_edge_cases(sp, ctx, orc):
    g_cols = dict(M=[1, 4096, 131072, 7, 0, 5, 5], N=[1, 4096, 152064, 9, 5, 5, 5],
                  K=[1, 4096, 53248, 3, 5, 5, 5], TM=[128, 128, 256, 1, 8, 0, 8],
                  TN=[128, 128, 128, 1, 8, 8, 8], BK=[64, 64, 64, 1, 8, 8, 8],
                  STAGES=[3, 3, 5, 1, 1, 1, 1], WARPS=[8, 8, 8, 1, 1, 1, 1],
                  REGS=[232, 232, 232, 1, 1, 1, 1], SMEM=[0, 0, 0, 300000, 0, 0, 0],
                  DTYPE=[0, 1, 0, 1, 0, 0, 3])
    b = gen.make_batch(gen.GEMM, g_cols)
    sa = np.concatenate([specs.paper_gpu_specs(), odd_specs()])
    sa[3]["th_tensor_fp16"] = 0  # missing fp16 rate -> status 7 for fp16 configs
    _, g = gpu_features(sp, ctx, b, sa)
    assert_feature_parity(g, orc.featurize(b, sa), "gemm edges")
    m_cols = dict(M=[4, 4, 8192, 3], E=[2, 2, 128, 8], TOPK=[2, 2, 8, 2], H=[64, 64, 4096, 100],
                  N=[64, 64, 3072, 100], BM=[16, 16, 16, 16], BN=[16, 16, 32, 16],
                  BK=[16, 16, 32, 16], GROUP_M=[1, 1, 1, 1], STAGES=[2, 2, 5, 2],
                  WARPS=[4, 4, 8, 4], REGS=[64, 64, 255, 64], SMEM=[0, 0, 0, 0], DTYPE=[0, 0, 0, 0])
    hist = [8, 0, 3, 4]
    m = gen.make_batch(gen.FUSED_MOE, m_cols, hist, [0, 2, -1, -1])
    _, g = gpu_features(sp, ctx, m, sa)
    o = orc.featurize(m, sa)
    assert o.status[1] == 4 and o.status[0] == 0
    assert_feature_parity(g, o, "moe edges")


def test_attention_records_independent_of_config_order(sp, ctx):
    """The schedule kernel takes chunks of 32 configs heaviest cost class first
    (attn_prepass + attn_order): a config's record must not depend on the order
    or neighbours its chunk gives it.  Records of a batch, of the same batch
    reversed and of it sorted by cost, compared bit for bit after undoing the
    permutation (every integer, float and status slot)."""
    b = gen.gen_attention(2000, 2000, 61, max_bs=8, qlen_max=6000, kvlen_max=9000)
    sa = specs.paper_gpu_specs()
    C = b.n_configs
    _, (gi, gf, gs) = gpu_features(sp, ctx, b, sa)
    rev = np.arange(C)[::-1].copy()
    rows = b.ragged[0::2].astype(np.int64)
    cost = np.bincount(np.repeat(np.arange(C), b.field("BS")), weights=rows, minlength=C)
    for perm in (rev, np.argsort(-cost, kind="stable")):
        _, (pi, pf, ps) = gpu_features(sp, ctx, b.subset(perm), sa)
        inv = np.empty(C, np.int64)
        inv[perm] = np.arange(C)
        # pair p = g * C + c (CROSS, spec-major): undo the config permutation per spec
        idx = (np.arange(len(sa))[:, None] * C + inv[None, :]).ravel()
        assert np.array_equal(ps[idx], gs)
        assert np.array_equal(pi[:, idx], gi)
        assert np.array_equal(pf[:, idx].view(np.uint32), gf.view(np.uint32))


def test_moe_histogram_edge_cases(sp, ctx, orc):
    """Fused-MoE histograms the warp pass reduces in 32-bit partials (R16, status 4
    = SP_PAIR_E_HIST): a negative count, counts whose exact sum is 2^32 + M topk
    (a wrapping 32-bit sum would accept it), one expert holding M topk ~ 1.9e9
    tokens, E > 128 (the tail loop), E = 1, and E = 33 (a partial second row);
    every record against the oracle, bit-exact."""
    big = 2 ** 31 - 1
    hists = [
        [5, -1, 4],                   # negative count, sum = M topk
        [big, big, 10],               # exact sum 2^32 + 8: invalid
        [1879048192],                 # M topk = 2^28 * 7, one expert
        list(range(1, 201)),          # E = 200: sum 20100
        list(range(1, 201)),          # E = 200, wrong sum
        [6],                          # E = 1
        [1] * 32 + [7],               # E = 33
        [0, 0, 8],                    # zero-token experts
    ]
    mt = [8, 8, 1879048192, 20100, 20100, 6, 39, 8]
    topk = [2, 2, 7, 4, 4, 1, 3, 2]
    n = len(hists)
    M = [m // k for m, k in zip(mt, topk)]
    M[4] += 1  # config 4: the histogram sums to 20100, M topk = 20104
    off = np.cumsum([0] + [len(h) for h in hists[:-1]]).tolist()
    cols = dict(M=M, E=[len(h) for h in hists], TOPK=topk, H=[1024] * n, N=[512] * n,
                BM=[16, 16, 64, 32, 32, 16, 16, 16], BN=[64] * n, BK=[32] * n, GROUP_M=[1] * n,
                STAGES=[3] * n, WARPS=[4] * n, REGS=[128] * n, SMEM=[0] * n, DTYPE=[0] * n)
    b = gen.make_batch(gen.FUSED_MOE, cols, sum(hists, []), off)
    sa = np.concatenate([specs.paper_gpu_specs(), odd_specs()])
    _, g = gpu_features(sp, ctx, b, sa)
    o = orc.featurize(b, sa)
    st = o.status.reshape(len(sa), n)[0]
    assert st.tolist() == [4, 4, 0, 0, 4, 0, 0, 0], st
    assert_feature_parity(g, o, "moe histograms")
    # the fused pass (pre-pass + producers) reads the same histogram results
    f = sp.Features.empty(b.family, len(sa) * n, "cuda:0")
    lat = torch.empty(f.n_pairs, dtype=torch.float32, device="cuda:0")
    ctx.featurize_predict(sp.DeviceBatch.from_host(b, "cuda:0"), ctx.load_gpu_specs(sa),
                          ctx.load_model(models.random_mlp(b.family, 8), "fp16"), f, lat)
    torch.cuda.synchronize()
    assert_feature_parity(sp.features_to_host(f), o, "moe histograms (fused)")


def test_full_size_sampled_cfg2(sp, ctx, orc):
    """BASELINE config 2 at full size (1e6 configs x 11 specs), in the launch
    configuration bench.py times (sp_featurize, then the fp16 tcgen05 sp_predict
    over all 1.1e7 pairs: ~580 tiles per CTA); 3000 sampled pairs checked one by
    one -- features bit-exact / 1e-5, latencies at north_star's 1e-2."""
    b = gen.gen_attention(500_000, 500_000, 1002)
    b, _ = gen.shuffle(b, 7)
    sa = specs.paper_gpu_specs()
    f, _ = gpu_features(sp, ctx, b, sa)
    model = models.random_mlp(b.family, 5)
    mh = ctx.load_model(model, "fp16")
    lat = torch.empty(f.n_pairs, dtype=torch.float32, device="cuda")
    ctx.predict(mh, f, lat)
    torch.cuda.synchronize()
    rng = np.random.default_rng(3)
    p = np.concatenate([rng.integers(0, f.n_pairs, 2990), np.arange(5), f.n_pairs - 1 - np.arange(5)])
    ci, si = p % b.n_configs, p // b.n_configs
    o = orc.featurize(b, sa, cfg_idx=ci, spec_idx=si)
    pt = torch.from_numpy(p).cuda()
    g = (f.ints[:, pt].cpu().numpy(), f.flts[:, pt].cpu().numpy(), f.status[pt].cpu().numpy())
    assert_feature_parity(g, o, "cfg2 full-size sample")
    olat, _, _ = orc.predict(model, o)
    glat = lat[pt].cpu().numpy().astype(np.float64)
    assert (o.status == 0).all()
    np.testing.assert_allclose(glat, olat, rtol=LAT_RTOL_16, atol=0, err_msg="cfg2 full-size fp16 latency")


def _predict_both(sp, ctx, orc, batch, sa, precision, seed=5):
    model = models.random_mlp(batch.family, seed)
    f, _ = gpu_features(sp, ctx, batch, sa)
    mh = ctx.load_model(model, precision)
    lat = torch.empty(f.n_pairs, dtype=torch.float32, device="cuda")
    eff = torch.empty(f.n_pairs, dtype=torch.float32, device="cuda")
    ctx.predict(mh, f, lat, eff)
    torch.cuda.synchronize()
    o = orc.featurize(batch, sa)
    olat, oeff, _ = orc.predict(model, o)
    return lat.cpu().numpy(), eff.cpu().numpy(), olat, oeff


@pytest.mark.parametrize("fam", list(FAMILY_BATCHES))
def test_predict_fp32_parity(sp, ctx, orc, fam):
    b = FAMILY_BATCHES[fam]().subset(np.arange(300))
    sa = specs.paper_gpu_specs()
    lat, eff, olat, oeff = _predict_both(sp, ctx, orc, b, sa, "fp32")
    ok = ~np.isnan(olat)
    assert np.array_equal(np.isnan(lat), ~ok)
    np.testing.assert_allclose(lat[ok], olat[ok], rtol=LAT_RTOL_FP32)
    np.testing.assert_allclose(eff[ok], oeff[ok], rtol=LAT_RTOL_FP32)


@pytest.mark.parametrize("fam", list(FAMILY_BATCHES))
def test_predict_tcgen05_parity(sp, ctx, orc, fam):
    b = FAMILY_BATCHES[fam]().subset(np.arange(300))
    sa = specs.paper_gpu_specs()
    lat, eff, olat, oeff = _predict_both(sp, ctx, orc, b, sa, "fp16")
    ok = ~np.isnan(olat)
    assert np.array_equal(np.isnan(lat), ~ok)
    rel = np.abs(lat[ok] / olat[ok] - 1)
    print(f"fp16 {fam}: max rel {rel.max():.2e} p99 {np.quantile(rel, 0.99):.2e} mean {rel.mean():.2e}")
    np.testing.assert_allclose(lat[ok], olat[ok], rtol=LAT_RTOL_16)  # every element


def test_bf16_predictor_refused(sp, ctx):
    """bf16 operands miss north_star's 1e-2 (measured 3e-2 in r01): refused at
    load rather than served with a looser envelope."""
    with pytest.raises(sp.SynPerfError, match="SP_E_UNSUPPORTED"):
        ctx.load_model(models.random_mlp(gen.GEMM, 5), "bf16")


def test_fp16_range_checked_at_load(sp, ctx):
    """A BN variance of 1e-12 folds W2' = W2 * gamma / sqrt(var + eps) past
    fp16's 65504: the fp16 load refuses it (SP_E_DATA) instead of packing
    infinities; the fp32 path, which keeps BN unfolded, accepts it."""
    model = models.random_mlp(gen.GEMM, 5, bn_eps=1e-12)
    model["v1"] = np.full(256, 1e-12, np.float32)
    model["g1"] = np.full(256, 10.0, np.float32)
    with pytest.raises(sp.SynPerfError, match="SP_E_DATA"):
        ctx.load_model(model, "fp16")
    ctx.load_model(model, "fp32")


def test_fp16_activations_saturate(sp, ctx):
    """Layer-1 pre-activations far past 65504 (weights 4000 on every input):
    the epilogue's cvt.rn.satfinite clamps them, so no latency is NaN (cvt.rn
    would give inf activations, then inf - inf = NaN in the next layer; the
    sigmoid may still legitimately underflow the efficiency to 0 -> inf)."""
    b = gen.gen_gemm(300, 31)
    sa = specs.paper_gpu_specs()
    model = models.random_mlp(gen.GEMM, 6)
    model["w1"] = np.full_like(model["w1"], 4000.0)
    f, (gi, gf, gs) = gpu_features(sp, ctx, b, sa)
    mh = ctx.load_model(model, "fp16")
    lat = torch.empty(f.n_pairs, dtype=torch.float32, device="cuda")
    ctx.predict(mh, f, lat)
    torch.cuda.synchronize()
    ok = gs == 0
    assert not np.isnan(lat.cpu().numpy()[ok]).any()


@pytest.mark.parametrize("prec", ["fp32", "fp16"])
@pytest.mark.parametrize("fam", ["gemm", "attention"])
def test_predict_non_identity_batchnorm(sp, ctx, orc, fam, prec):
    """Eval BatchNorm far from the identity (gamma of both signs, shifts and means
    of the activations' size, variances over a decade and a half, eps 1e-3),
    folded into the next layer on the GPU (R18): the fold must reproduce the
    oracle's unfused Linear -> ReLU -> BN.  The statistics keep the logits in the
    seeded model's range (|z| <~ 4): a fp32 MLP's rounding grows with |z| (an
    fp32 emulation of this model measures 4.5e-6 against fp64, inside 1e-5)."""
    b = FAMILY_BATCHES[fam]().subset(np.arange(300))
    sa = specs.paper_gpu_specs()
    rng = np.random.default_rng(17)
    model = models.random_mlp(b.family, 17, bn_eps=1e-3)
    for li, w in zip((1, 2, 3), (256, 128, 64)):
        model[f"g{li}"] = (rng.uniform(0.5, 1.5, w) * rng.choice([-1, 1], w)).astype(np.float32)
        model[f"be{li}"] = rng.uniform(-0.5, 0.5, w).astype(np.float32)
        model[f"m{li}"] = rng.uniform(-0.5, 1.0, w).astype(np.float32)
        model[f"v{li}"] = np.exp(rng.uniform(np.log(0.2), np.log(3.0), w)).astype(np.float32)
    f, _ = gpu_features(sp, ctx, b, sa)
    mh = ctx.load_model(model, prec)
    lat = torch.empty(f.n_pairs, dtype=torch.float32, device="cuda")
    ctx.predict(mh, f, lat)
    torch.cuda.synchronize()
    o = orc.featurize(b, sa)
    olat, _, _ = orc.predict(model, o)
    ok = o.status == 0
    np.testing.assert_allclose(lat.cpu().numpy()[ok], olat[ok], rtol=LAT_RTOL_FP32 if prec == "fp32" else LAT_RTOL_16)


def test_predict_zero_output_layer_exact(sp, ctx, orc):
    """Zero final layer: e = 0.5 exactly, latency = 2 t_theory, both paths."""
    b = gen.gen_gemm(200, 9)
    sa = specs.paper_gpu_specs()
    f, (gi, gf, gs) = gpu_features(sp, ctx, b, sa)
    for prec in ("fp32", "fp16"):
        mh = ctx.load_model(models.zero_output_mlp(gen.GEMM, 1), prec)
        lat = torch.empty(f.n_pairs, dtype=torch.float32, device="cuda")
        ctx.predict(mh, f, lat)
        torch.cuda.synchronize()
        assert np.array_equal(lat.cpu().numpy(), 2.0 * gf[11]), prec


@pytest.mark.parametrize("fam", ["attention", "moe", "gemm"])
@pytest.mark.parametrize("chunks", [1, 3])
def test_predict_host_equals_device_path(sp, ctx, fam, chunks):
    """The public host-buffer call (pipelined H2D / kernels / D2H) returns
    exactly what the device-resident featurize + predict returns."""
    b = FAMILY_BATCHES[fam]()
    sa = specs.paper_gpu_specs()
    sh = ctx.load_gpu_specs(sa)
    m = ctx.load_model(models.random_mlp(b.family, 5), "fp16")
    f, _ = gpu_features(sp, ctx, b, sa, specs_handle=sh)
    lat = torch.empty(f.n_pairs, dtype=torch.float32, device="cuda")
    ctx.predict(m, f, lat)
    torch.cuda.synchronize()

    class Host:
        family = b.family

    h = Host()
    h.fields = torch.from_numpy(b.fields).pin_memory()
    h.ragged = None if b.ragged is None else torch.from_numpy(b.ragged).pin_memory()
    h.ragged_off = None if b.ragged_off is None else torch.from_numpy(b.ragged_off).pin_memory()
    got = ctx.predict_host(h, sh, m, chunks=chunks)
    assert np.array_equal(got, lat.cpu().numpy(), equal_nan=True)


@pytest.mark.parametrize("layout", ["reversed", "interior_jump"])
def test_predict_host_irregular_ragged_layout(sp, ctx, layout):
    """predict_host copies each slice's ragged range when the layout is config
    by config; layouts that break that (reversed chunks: caught on the host;
    an interior config pointing into another slice's range: caught on the
    device, the call redone with one whole copy) still give exactly the
    device path's latencies."""
    b = FAMILY_BATCHES["attention"]()
    off = b.ragged_off.copy()
    bs = b.field("BS").astype(np.int64)
    if layout == "reversed":
        chunks = [b.ragged[o:o + 2 * n] for o, n in zip(off, bs)][::-1]
        rag = np.concatenate(chunks).astype(np.int32)
        lens = (2 * bs)[::-1]
        starts = np.concatenate([[0], np.cumsum(lens)[:-1]])[::-1]
        off = starts.astype(np.int64)
    else:
        rag = b.ragged.copy()
        k_src = b.n_configs - 3  # a config in the last slice with the same batch size
        k = next(k for k in range(5, b.n_configs // 4) if bs[k] == bs[k_src])
        off[k] = off[k_src]
    b2 = gen.ConfigBatch(b.family, b.fields.copy(), rag, off)
    sa = specs.paper_gpu_specs()
    sh = ctx.load_gpu_specs(sa)
    m = ctx.load_model(models.random_mlp(b.family, 5), "fp16")
    f, _ = gpu_features(sp, ctx, b2, sa, specs_handle=sh)
    lat = torch.empty(f.n_pairs, dtype=torch.float32, device="cuda")
    ctx.predict(m, f, lat)
    torch.cuda.synchronize()

    class Host:
        family = b.family

    h = Host()
    h.fields = torch.from_numpy(b2.fields).pin_memory()
    h.ragged = torch.from_numpy(b2.ragged).pin_memory()
    h.ragged_off = torch.from_numpy(b2.ragged_off).pin_memory()
    got = ctx.predict_host(h, sh, m, chunks=4)
    assert np.array_equal(got, lat.cpu().numpy(), equal_nan=True)


@pytest.mark.parametrize("fam", ["attention", "moe"])
def test_predict_host_pageable_weights_subrange(sp, ctx, fam):
    """sp_predict_host from pageable numpy arrays, explicit slice weights, a
    spec sub-range: the device path's latencies for those specs, bit for bit."""
    b = FAMILY_BATCHES[fam]()
    sa = specs.paper_gpu_specs()
    sh = ctx.load_gpu_specs(sa)
    m = ctx.load_model(models.random_mlp(b.family, 5), "fp16")
    db = sp.DeviceBatch.from_host(b, ctx.torch_device)
    n = 5 * b.n_configs
    f = sp.Features.empty(b.family, n, ctx.torch_device)
    lat = torch.empty(n, dtype=torch.float32, device="cuda")
    ctx.featurize(db, sh, f, sp.cross(2, 7))
    ctx.predict(m, f, lat)
    torch.cuda.synchronize()
    got = ctx.predict_host(b, sh, m, spec_range=(2, 7), chunks=(1, 3, 3, 1))
    assert np.array_equal(got, lat.cpu().numpy(), equal_nan=True)
    got2 = ctx.predict_host(b, sh, m, spec_range=(2, 7), chunks=7)  # reuses the grown staging
    assert np.array_equal(got2, got, equal_nan=True)


def test_predict_host_argument_errors(sp, ctx):
    b = FAMILY_BATCHES["gemm"]()
    sa = specs.paper_gpu_specs()
    sh = ctx.load_gpu_specs(sa)
    m = ctx.load_model(models.random_mlp(b.family, 5), "fp16")
    with pytest.raises(sp.SynPerfError, match="SP_E_ARG"):
        ctx.predict_host(b, sh, m, spec_range=(3, 40))
    mm = ctx.load_model(models.random_mlp(gen.ATTENTION, 5), "fp16")
    with pytest.raises(sp.SynPerfError, match="SP_E_ARG"):  # family mismatch, from sp_featurize_predict
        ctx.predict_host(b, sh, mm)


@pytest.mark.parametrize("fam", ["attention", "gemm"])
def test_prepare_then_graph_capture(sp, ctx, fam):
    """After sp_prepare the hot calls neither allocate nor synchronize: a fresh
    context captures featurize_predict in a CUDA graph, and replays equal the
    eager result."""
    b = FAMILY_BATCHES[fam]()
    sa = specs.paper_gpu_specs()
    c2 = sp.Context(0)
    sh = c2.load_gpu_specs(sa)
    m = c2.load_model(models.random_mlp(b.family, 5), "fp16")
    db = sp.DeviceBatch.from_host(b, c2.torch_device)
    n = len(sa) * b.n_configs
    f = sp.Features.empty(b.family, n, c2.torch_device)
    lat = torch.empty(n, dtype=torch.float32, device="cuda")
    c2.prepare(b.family, b.n_configs, sh)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        c2.featurize_predict(db, sh, m, f, lat, stream=s)
    lat.zero_()
    g.replay()
    torch.cuda.synchronize()
    got = lat.cpu().numpy().copy()
    lat2 = torch.empty_like(lat)
    c2.featurize_predict(db, sh, m, f, lat2)
    torch.cuda.synchronize()
    assert np.array_equal(got, lat2.cpu().numpy(), equal_nan=True)


def test_featurize_deterministic(sp, ctx):
    b = FAMILY_BATCHES["attention"]()
    sa = specs.paper_gpu_specs()
    _, a = gpu_features(sp, ctx, b, sa)
    _, c = gpu_features(sp, ctx, b, sa)
    for x, y in zip(a, c):
        assert np.array_equal(x, y, equal_nan=True)


@pytest.mark.parametrize("fam", ["attention", "gemm"])
def test_predict_host_wide_spec_axis(sp, ctx, fam):
    """>= 64 specs: predict_host pipelines over spec slices (contiguous D2H
    runs of the spec-major output); identical to the device path."""
    b = FAMILY_BATCHES[fam]()
    sa = specs.hypothetical_sweep_specs(300)
    sh = ctx.load_gpu_specs(sa)
    m = ctx.load_model(models.random_mlp(b.family, 6), "fp16")
    f, _ = gpu_features(sp, ctx, b, sa, specs_handle=sh)
    lat = torch.empty(f.n_pairs, dtype=torch.float32, device="cuda")
    ctx.predict(m, f, lat)
    torch.cuda.synchronize()
    got = ctx.predict_host(b, sh, m)
    assert np.array_equal(got, lat.cpu().numpy(), equal_nan=True)


# ------------------------------------------------------------- clamped edge tiles (SP_FEAT_CLAMPED, NEXT-4)

@pytest.mark.parametrize("fam", ["gemm", "moe", "attention", "attention_gqa"])
def test_clamped_parity(sp, ctx, orc, fam):
    """Clamped edge tiles vs the oracle's CLAMPED flag: CROSS over Table VI and
    the odd SM counts, and a LIST with out-of-range indices."""
    b = FAMILY_BATCHES[fam]()
    for sa in (specs.paper_gpu_specs(), odd_specs()):
        sh = ctx.load_gpu_specs(sa)
        db = sp.DeviceBatch.from_host(b, ctx.torch_device)
        f = sp.Features.empty(b.family, len(sa) * b.n_configs, ctx.torch_device)
        ctx.featurize(db, sh, f, clamped=True)
        torch.cuda.synchronize()
        o = orc.featurize(b, sa, flags=orc.CLAMPED)
        assert (o.status == 0).mean() > 0.9
        assert_feature_parity(sp.features_to_host(f), o, fam + " clamped")
    rng = np.random.default_rng(8)
    ci, si = rng.integers(0, b.n_configs, 500), rng.integers(0, len(sa), 500)
    ci[0], si[1] = -1, len(sa)
    pr = sp.pair_list(torch.from_numpy(ci.astype(np.int64)).cuda(), torch.from_numpy(si.astype(np.int32)).cuda())
    f = sp.Features.empty(b.family, 500, ctx.torch_device)
    ctx.featurize(db, sh, f, pr, clamped=True)
    torch.cuda.synchronize()
    assert_feature_parity(sp.features_to_host(f), orc.featurize(b, sa, cfg_idx=ci, spec_idx=si, flags=orc.CLAMPED),
                          fam + " clamped list")


def test_clamped_edge_cases(sp, ctx, orc):
    """Single tile, exact multiples (clamped = padded when K is a multiple of BK),
    one row of tiles, huge M (many rows), and the golden MoE case; row-wise
    families and non-RR schedulers are refused."""
    cols = {k: [] for k in gen.FIELDS[gen.GEMM]}

    def add(**kw):
        d = dict(M=256, N=256, K=256, TM=128, TN=128, BK=64, STAGES=3, WARPS=8, REGS=168, SMEM=0, DTYPE=0)
        d.update(kw)
        for k in cols:
            cols[k].append(d[k])

    add(M=100, N=100, K=100)          # one clamped tile
    add()                             # exact multiples
    add(M=1, N=152064, K=4096)        # one row of 1188 tiles
    add(M=131072, N=130, K=300)       # 1024 rows, edge column of 2
    add(M=0)                          # dimension error
    b = gen.make_batch(gen.GEMM, cols)
    sa = np.concatenate([odd_specs(), specs.paper_gpu_specs()])
    sh = ctx.load_gpu_specs(sa)
    db = sp.DeviceBatch.from_host(b, ctx.torch_device)
    f = sp.Features.empty(b.family, len(sa) * b.n_configs, ctx.torch_device)
    ctx.featurize(db, sh, f, clamped=True)
    torch.cuda.synchronize()
    assert_feature_parity(sp.features_to_host(f), orc.featurize(b, sa, flags=orc.CLAMPED), "clamped edges")
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))["moe_clamped_tiny"]
    mb = gen.make_batch(gen.FUSED_MOE, {k: [v] for k, v in g["config"].items()}, g["hist"], [0])
    s3 = specs.spec_by_name("A100")
    s3["num_sms"] = g["n_sm"]
    f = sp.Features.empty(mb.family, 1, ctx.torch_device)
    ctx.featurize(sp.DeviceBatch.from_host(mb, ctx.torch_device), ctx.load_gpu_specs(s3), f, clamped=True)
    gi, _, gs = sp.features_to_host(f)
    assert gs[0] == 0 and (gi[6, 0], gi[10, 0], gi[3, 0], gi[9, 0]) == (g["max_T"], g["bytes_max"], g["tot_T"], g["bytes"])
    rms = FAMILY_BATCHES["rmsnorm"]()
    fr = sp.Features.empty(rms.family, len(sa) * rms.n_configs, ctx.torch_device)
    with pytest.raises(sp.SynPerfError):  # row-wise kernels have no edge tiles
        ctx.featurize(sp.DeviceBatch.from_host(rms, ctx.torch_device), sh, fr, clamped=True)
    f = sp.Features.empty(b.family, len(sa) * b.n_configs, ctx.torch_device)
    with pytest.raises(sp.SynPerfError):
        ctx.featurize(db, sh, f, clamped=True, scheduler="greedy")


# ------------------------------------------------------------- fused featurize -> predict (sp_featurize_predict)

@pytest.mark.parametrize("fam", ["gemm", "moe", "rmsnorm", "silu", "scaled_mm", "attention", "gemm_splitk"])
@pytest.mark.parametrize("prec", ["fp16", "fp32"])
def test_featurize_predict_equals_two_calls(sp, ctx, fam, prec):
    """The fused call writes the same records, bit for bit, and the same latencies
    and efficiencies as sp_featurize + sp_predict (full and partial spec ranges,
    odd SM counts; pair counts that are not multiples of the 128-row tile)."""
    b = FAMILY_BATCHES[fam]()
    b = b.subset(np.arange(min(333, b.n_configs)))
    m = ctx.load_model(models.random_mlp(b.family, 12), prec)
    db = sp.DeviceBatch.from_host(b, ctx.torch_device)
    for sa, (g0, g1) in ((specs.paper_gpu_specs(), (0, 11)), (specs.paper_gpu_specs(), (3, 9)), (odd_specs(), (0, 8))):
        sh = ctx.load_gpu_specs(sa)
        n = (g1 - g0) * b.n_configs
        outs = []
        for fused in (False, True):
            f = sp.Features.empty(b.family, n, ctx.torch_device)
            lat = torch.full((n,), -1.0, dtype=torch.float32, device="cuda")
            eff = torch.full((n,), -1.0, dtype=torch.float32, device="cuda")
            if fused:
                ctx.featurize_predict(db, sh, m, f, lat, eff, sp.cross(g0, g1))
            else:
                ctx.featurize(db, sh, f, sp.cross(g0, g1))
                ctx.predict(m, f, lat, eff)
            torch.cuda.synchronize()
            outs.append((sp.features_to_host(f), lat.cpu().numpy(), eff.cpu().numpy()))
        (gi0, gf0, gs0), l0, e0 = outs[0]
        (gi1, gf1, gs1), l1, e1 = outs[1]
        assert np.array_equal(gs0, gs1) and np.array_equal(gi0, gi1), fam
        assert np.array_equal(gf0.view(np.uint32), gf1.view(np.uint32)), fam
        assert np.array_equal(l0.view(np.uint32), l1.view(np.uint32)), fam
        assert np.array_equal(e0.view(np.uint32), e1.view(np.uint32)), fam


def test_featurize_predict_attention_planner_and_errors(sp, ctx, orc):
    """The fused attention path with split-KV planner configs (kv_chunk -1: the
    planner kernel's records are read back by the producers), domain errors
    (zero batch, GQA mismatch, causal kv < q) and both causal paths: records
    and latencies bit-identical to the two calls, and the oracle's ints."""
    b = gen.gen_attention(120, 120, 77, max_bs=6, qlen_max=3000, kvlen_max=6000, groups=(1, 3, 4, 5))
    ch = b.fields[gen.FIELDS[gen.ATTENTION].index("KV_CHUNK")]
    causal = b.fields[gen.FIELDS[gen.ATTENTION].index("CAUSAL")]
    ch[(np.arange(b.n_configs) % 4 == 1) & (causal == 0)] = -1
    nh = b.fields[gen.FIELDS[gen.ATTENTION].index("NH")]
    nh[7] += 1  # nh % nkv != 0 -> SP_PAIR_E_HEADS (unless nkv = 1)
    sa = specs.paper_gpu_specs()
    sh = ctx.load_gpu_specs(sa)
    m = ctx.load_model(models.random_mlp(b.family, 12), "fp16")
    db = sp.DeviceBatch.from_host(b, ctx.torch_device)
    n = len(sa) * b.n_configs
    outs = []
    for fused in (False, True):
        f = sp.Features.empty(b.family, n, ctx.torch_device)
        lat = torch.full((n,), -1.0, dtype=torch.float32, device="cuda")
        if fused:
            ctx.featurize_predict(db, sh, m, f, lat)
        else:
            ctx.featurize(db, sh, f)
            ctx.predict(m, f, lat)
        torch.cuda.synchronize()
        outs.append((sp.features_to_host(f), lat.cpu().numpy()))
    (gi0, gf0, gs0), l0 = outs[0]
    (gi1, gf1, gs1), l1 = outs[1]
    assert (ch == -1).sum() > 10
    assert np.array_equal(gs0, gs1) and np.array_equal(gi0, gi1)
    assert np.array_equal(gf0.view(np.uint32), gf1.view(np.uint32))
    assert np.array_equal(l0.view(np.uint32), l1.view(np.uint32))
    o = orc.featurize(b, sa)
    assert np.array_equal(gs1, o.status) and np.array_equal(gi1, o.ints)


@pytest.mark.parametrize("cfg", ["cfg3", "cfg5", "scaledmm", "splitk"])
def test_full_size_sampled_fused(sp, ctx, orc, cfg):
    """BASELINE configs 3 (1e6 fused-MoE configs x 11 GPUs) and 5 (1,000 serving
    GEMMs x 100,000 hypothetical specs = 1e8 pairs) at full size through
    sp_featurize_predict -- the launch configuration bench.py times for them --
    with 2,000 sampled pairs checked one by one against the oracle: records
    (ints bit-exact, floats 1e-5) and fp16 latencies (1e-2)."""
    if cfg == "cfg3":
        b, sa = gen.gen_moe(1_000_000, 1003), specs.paper_gpu_specs()
    elif cfg == "scaledmm":  # bench --workload scaledmm (fused)
        b, sa = gen.gen_scaled_mm(1_000_000, 1006), specs.paper_gpu_specs()
    elif cfg == "splitk":  # bench --workload splitk (the two calls behind the same entry point)
        b, sa = gen.gen_gemm_splitk(1_000_000, 1007), specs.paper_gpu_specs()
    else:
        b, sa = gen.gen_serving_gemms(1000, 1005), specs.hypothetical_sweep_specs(100_000)
    sh = ctx.load_gpu_specs(sa)
    model = models.random_mlp(b.family, 42)
    m = ctx.load_model(model, "fp16")
    n = len(sa) * b.n_configs
    f = sp.Features.empty(b.family, n, ctx.torch_device)
    lat = torch.empty(n, dtype=torch.float32, device="cuda")
    ctx.featurize_predict(sp.DeviceBatch.from_host(b, ctx.torch_device), sh, m, f, lat)
    torch.cuda.synchronize()
    rng = np.random.default_rng(4)
    p = rng.integers(0, n, 2000)
    ci, si = p % b.n_configs, p // b.n_configs
    o = orc.featurize(b, sa, cfg_idx=ci, spec_idx=si)
    pt = torch.from_numpy(p).cuda()
    g = (f.ints[:, pt].cpu().numpy(), f.flts[:, pt].cpu().numpy(), f.status[pt].cpu().numpy())
    assert_feature_parity(g, o, cfg + " full-size sample")
    olat, _, _ = orc.predict(model, o)
    gl = lat[pt].cpu().numpy()
    ok = ~np.isnan(olat)
    assert ok.mean() > (0.6 if cfg == "scaledmm" else 0.9) and np.array_equal(np.isnan(gl), ~ok)
    np.testing.assert_allclose(gl[ok], olat[ok], rtol=LAT_RTOL_16)
    del f, lat
    torch.cuda.empty_cache()


def test_clamped_attention_edge_cases(sp, ctx, orc):
    """Clamped attention: partial last q-blocks, causal + split-KV, the split-KV
    planner (-1), decode, GQA packing, kv shorter than BKV, and domain errors."""
    cols = {k: [] for k in gen.FIELDS[gen.ATTENTION]}
    rag, off = [], []

    def add(reqs, **kw):
        d = dict(NH=8, NKV=2, HD=128, BQ=64, BKV=64, KV_CHUNK=0, CAUSAL=1, WARPS=4, REGS=128, SMEM=0, DTYPE=0)
        d.update(kw)
        d["BS"] = len(reqs)
        for k in cols:
            cols[k].append(d[k])
        off.append(len(rag))
        for q, kv in reqs:
            rag.extend([q, kv])

    add([(100, 100)])                                   # partial q-blocks, causal
    add([(300, 5000), (77, 2000)], KV_CHUNK=512)        # causal + split-KV
    add([(1, 4000), (1, 300)], BQ=16, CAUSAL=0, KV_CHUNK=-1)   # planner
    add([(1, 20)] * 9, BQ=16, CAUSAL=0)                 # decode, kv < BKV
    add([(33, 40)], NH=32, NKV=2)                       # GQA group 16
    add([(5, 3)])                                       # causal with kv < q: status 5
    b = gen.make_batch(gen.ATTENTION, cols, rag, off)
    sa = np.concatenate([odd_specs(), specs.paper_gpu_specs()])
    sh = ctx.load_gpu_specs(sa)
    f = sp.Features.empty(b.family, len(sa) * b.n_configs, ctx.torch_device)
    ctx.featurize(sp.DeviceBatch.from_host(b, ctx.torch_device), sh, f, clamped=True)
    torch.cuda.synchronize()
    o = orc.featurize(b, sa, flags=orc.CLAMPED)
    assert (o.status == 0).sum() > 0 and (o.status == 5).any()
    assert_feature_parity(sp.features_to_host(f), o, "clamped attention edges")
