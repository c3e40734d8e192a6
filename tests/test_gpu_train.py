"""On-GPU estimator training (csrc/train.cu via the C-ABI) vs the fp64 training
oracle (oracle/train.py), element by element.

Inputs: seeded feature records (workloads/gen), featurised on both sides; the
measured latencies that define the efficiency targets come from the oracle's
t_theory and a seeded efficiency draw (never from the CUDA path).
Bars: the per-step loss within 1e-4 relative of fp64; parameters after a few
AdamW steps within 1e-5 absolute + 1e-4 relative for 99.9% of entries and
within 2 lr per step everywhere (an fp32 gradient of a near-zero fp64 gradient
may take the other sign, which moves that entry by up to 2 lr); running
statistics within 1e-4; determinism bitwise.
"""
import numpy as np
import pytest
import torch

from oracle import train as T
from workloads import gen, models, specs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_14910_b200 as sp

    return sp


@pytest.fixture(scope="module")
def ctx(sp):
    return sp.Context(0)


def setup(sp, ctx, orc, family=gen.ATTENTION, n=120, seed=21):
    """GPU features + oracle features of a small batch x 11 GPUs, valid pairs,
    oracle-derived measured latencies (efficiency ~ U(0.15, 0.9))."""
    if family == gen.ATTENTION:
        b = gen.gen_attention(n // 2, n // 2, seed, max_bs=4, qlen_max=3000, kvlen_max=5000)
    else:
        b = gen.gen_gemm(n, seed)
    sa = specs.paper_gpu_specs()
    sh = ctx.load_gpu_specs(sa)
    db = sp.DeviceBatch.from_host(b, ctx.torch_device)
    f = sp.Features.empty(b.family, len(sa) * b.n_configs, ctx.torch_device)
    ctx.featurize(db, sh, f)
    torch.cuda.synchronize()
    o = orc.featurize(b, sa)
    valid = np.nonzero(o.status == 0)[0]
    rng = np.random.default_rng(seed)
    eff = rng.uniform(0.15, 0.9, len(o.status))
    tt = o.flts[11]
    measured = np.where(o.status == 0, tt / eff, 1.0).astype(np.float32)
    return b, sa, f, o, valid, measured


def oracle_inputs(orc, model, o, measured, idx):
    x = np.stack([orc.mlp_input(model, o.ints[:, p], o.flts[:, p]) for p in idx])
    t = (np.float32(o.flts[11][idx]).astype(np.float32) / measured[idx]).astype(np.float64)
    return x, t


def dev(a, dt):
    return torch.from_numpy(np.ascontiguousarray(a).astype(dt)).cuda()


@pytest.mark.parametrize("loss", ["mape", "pinball"])
def test_train_step_gradients_match_oracle(sp, ctx, orc, loss):
    """One step from the same weights: every gradient within 1e-4 of its layer's
    gradient scale.  (The biases in front of BatchNorm have exactly-zero true
    gradients for units active on every row -- BN removes a constant shift --
    so their fp32 and fp64 values are both rounding noise; the layer scale
    bounds that noise.)"""
    b, sa, f, o, valid, measured = setup(sp, ctx, orc)
    model = models.random_mlp(b.family, 31)
    tr = ctx.trainer(model, loss=loss, max_batch=256, seed=77)
    p = T.init_params(model)
    cfg = dict(T.DEFAULTS, loss=loss, seed=77)
    idx = np.random.default_rng(5).choice(valid, 256, replace=False)
    x, t = oracle_inputs(orc, model, o, measured, idx)
    e, cache = T.forward_train(p, x, 0, cfg["seed"], cfg["drop"], cfg["eps"])
    go = T.backward(p, cache, t, loss, cfg["q"], cfg["drop"], cfg["eps"])
    lg = float(tr.step(f, dev(measured, np.float32), dev(idx, np.int64)).item())
    assert lg == pytest.approx(T.loss_value(e, t, loss, cfg["q"]), rel=1e-5)
    gg = tr.export_grads()
    for l in ("1", "2", "3", "4"):
        ks = [k for k in T.PARAM_ORDER if k[-1] == l]
        scale = max(np.abs(go[k]).max() for k in ks)
        for k in ks:
            err = np.abs(np.asarray(gg[k], np.float64).reshape(go[k].shape) - go[k]).max()
            assert err <= 1e-4 * scale, (k, err, scale)


@pytest.mark.parametrize("loss", ["mape", "pinball"])
def test_train_steps_match_oracle(sp, ctx, orc, loss):
    b, sa, f, o, valid, measured = setup(sp, ctx, orc)
    model = models.random_mlp(b.family, 31)
    tr = ctx.trainer(model, loss=loss, max_batch=256, seed=77)
    p = T.init_params(model)
    st = T.new_adam_state(p)
    cfg = dict(T.DEFAULTS, loss=loss, seed=77)
    rng = np.random.default_rng(5)
    m_dev = dev(measured, np.float32)
    for step, B in enumerate([256, 200, 37]):
        idx = rng.choice(valid, B, replace=False)
        x, t = oracle_inputs(orc, model, o, measured, idx)
        lo = T.train_step(p, st, x, t, step, cfg)
        lg = float(tr.step(f, m_dev, dev(idx, np.int64)).item())
        assert lg == pytest.approx(lo, rel=1e-4), (step, lg, lo)
    m = tr.export()
    for k in T.PARAM_ORDER:
        g = np.asarray(m[k], np.float64).reshape(-1)
        r = p[k].reshape(-1)
        err = np.abs(g - r)
        assert err.max() <= 2 * 1e-3 * 3 + 1e-5, (k, err.max())  # AdamW moves <= lr (1 + wd|p|) per step
        if k in ("b1", "b2", "b3"):
            continue  # noise-driven AdamW steps (see the gradient test); bounded above
        close = err <= 1e-5 + 1e-4 * np.abs(r)
        assert close.mean() >= 0.999, (k, close.mean(), err.max())
    # running statistics see the pre-BN biases, whose noise-driven steps (<= 2 lr each)
    # shift relu(z) by up to 2 lr per step; momentum 0.1 passes a tenth of that on
    for l in (1, 2, 3):
        np.testing.assert_allclose(m[f"m{l}"], p[f"m{l}"], rtol=1e-4, atol=0.1 * 2 * 1e-3 * 3)
        np.testing.assert_allclose(m[f"v{l}"], p[f"v{l}"], rtol=1e-3, atol=1e-4)


def test_eval_loss_chunks_match_oracle(sp, ctx, orc):
    """Eval mode (running statistics, no dropout) over more rows than max_batch."""
    b, sa, f, o, valid, measured = setup(sp, ctx, orc, family=gen.GEMM, n=100)
    model = models.random_mlp(b.family, 32)
    tr = ctx.trainer(model, max_batch=64)
    idx = valid[:300]
    x, t = oracle_inputs(orc, model, o, measured, idx)
    e = T.forward_eval(T.init_params(model), x, float(model["bn_eps"]))
    lg = float(tr.eval_loss(f, dev(measured, np.float32), dev(idx, np.int64)).item())
    assert lg == pytest.approx(T.loss_mape(e, t), rel=1e-4)


def test_fit_norm_matches_oracle(sp, ctx, orc):
    b, sa, f, o, valid, measured = setup(sp, ctx, orc)
    ident = dict(models.random_mlp(b.family, 1), mu=np.zeros(15, np.float32), sigma=np.ones(15, np.float32))
    lv = np.stack([orc.mlp_input(ident, o.ints[:, p], o.flts[:, p]) for p in valid])  # ln(1 + v), fp64
    mu_o, sg_o = T.fit_norm(np.expm1(lv))
    mu, sg = ctx.fit_norm(f, dev(valid, np.int64))
    np.testing.assert_allclose(mu, mu_o, rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(sg, sg_o, rtol=1e-5, atol=1e-6)


def test_train_deterministic_and_exports_a_predictor(sp, ctx, orc):
    """Same seed -> bitwise-identical parameters; the exported model loads into
    sp_predict (fp32) and matches the oracle's eval-mode forward of the same weights."""
    b, sa, f, o, valid, measured = setup(sp, ctx, orc, family=gen.GEMM, n=150)
    model = models.random_mlp(b.family, 33)
    m_dev = dev(measured, np.float32)
    outs = []
    for _ in range(2):
        tr = ctx.trainer(model, max_batch=128, seed=5)
        rng = np.random.default_rng(9)
        for _ in range(4):
            tr.step(f, m_dev, dev(rng.choice(valid, 128, replace=False), np.int64))
        outs.append(tr.export())
    for k in T.PARAM_ORDER + ["m1", "v1", "m3", "v3"]:
        assert np.array_equal(outs[0][k], outs[1][k]), k
    trained = outs[0]
    mh = ctx.load_model(trained, "fp32")
    lat = torch.empty(f.n_pairs, dtype=torch.float32, device="cuda")
    eff = torch.empty(f.n_pairs, dtype=torch.float32, device="cuda")
    ctx.predict(mh, f, lat, eff)
    torch.cuda.synchronize()
    idx = valid[:200]
    x = np.stack([orc.mlp_input(trained, o.ints[:, p], o.flts[:, p]) for p in idx])
    e_o = T.forward_eval(T.init_params(trained), x, float(trained["bn_eps"]))
    np.testing.assert_allclose(eff.cpu().numpy()[idx], e_o, rtol=1e-5)


def test_training_reduces_validation_mape(sp, ctx, orc):
    """A learnable synthetic target (efficiency = sigmoid of a fixed function of
    log t_theory, oracle-derived) is fitted: validation MAPE falls well below
    its initial value within a few epochs of early-stopped training."""
    b = gen.gen_gemm(3000, 41)
    sa = specs.paper_gpu_specs()
    sh = ctx.load_gpu_specs(sa)
    f = sp.Features.empty(b.family, len(sa) * b.n_configs, ctx.torch_device)
    ctx.featurize(sp.DeviceBatch.from_host(b, ctx.torch_device), sh, f)
    o = orc.featurize(b, sa)
    valid = np.nonzero(o.status == 0)[0]
    tt = o.flts[11]
    eff = 0.1 + 0.8 / (1.0 + np.exp(-(0.5 * np.log(np.maximum(tt, 1e-3)) - 2.0)))
    measured = np.where(o.status == 0, tt / eff, 1.0).astype(np.float32)
    rng = np.random.default_rng(3)
    perm = rng.permutation(valid)
    tr_idx, va_idx = dev(perm[:-2000], np.int64), dev(perm[-2000:], np.int64)
    model = models.random_mlp(b.family, 34)
    mu, sg = ctx.fit_norm(f, tr_idx)
    model["mu"], model["sigma"] = mu, sg
    tr = ctx.trainer(model, max_batch=256, seed=1)
    m_dev = dev(measured, np.float32)
    v0 = float(tr.eval_loss(f, m_dev, va_idx).item())
    res = tr.fit(f, m_dev, tr_idx, va_idx, max_epochs=8, patience=3)
    assert res["best_val_loss"] < 0.5 * v0 and res["best_val_loss"] < 0.1, (v0, res["val_history"])


def test_captured_step_graph_equals_eager_steps(sp, ctx, orc):
    """A CUDA graph of sp_train_step replayed three times (the batch buffer refilled
    in place) gives bitwise the same parameters as three eager steps: the step
    counter, dropout masks and bias corrections advance on the device."""
    b, sa, f, o, valid, measured = setup(sp, ctx, orc, family=gen.GEMM, n=150)
    model = models.random_mlp(b.family, 35)
    m_dev = dev(measured, np.float32)
    rng = np.random.default_rng(2)
    batches = [dev(rng.choice(valid, 128, replace=False), np.int64) for _ in range(3)]
    eager = ctx.trainer(model, max_batch=128, seed=9)
    for bi in batches:
        eager.step(f, m_dev, bi)
    tr = ctx.trainer(model, max_batch=128, seed=9)
    buf = torch.empty(128, dtype=torch.int64, device="cuda")
    g = tr.capture(f, m_dev, buf)
    for bi in batches:
        buf.copy_(bi)
        g.replay()
    torch.cuda.synchronize()
    a, c = eager.export(), tr.export()
    for k in T.PARAM_ORDER + ["m1", "v1", "m2", "v2", "m3", "v3"]:
        assert np.array_equal(a[k], c[k]), k


def test_training_argument_errors(sp, ctx, orc):
    """The C-ABI refuses bad training arguments with SP_E_ARG / SP_E_DATA and
    leaves the trainer usable."""
    b, sa, f, o, valid, measured = setup(sp, ctx, orc, family=gen.GEMM, n=60)
    model = models.random_mlp(b.family, 36)
    with pytest.raises(sp.SynPerfError):
        ctx.trainer(model, max_batch=1)                      # max_batch < 2
    with pytest.raises(sp.SynPerfError):
        ctx.trainer(model, loss="pinball", quantile=1.5)     # q outside (0, 1)
    with pytest.raises(sp.SynPerfError):
        ctx.trainer(dict(model, n_in=15))                    # Table IV width of another family
    tr = ctx.trainer(model, max_batch=64)
    m_dev = dev(measured, np.float32)
    with pytest.raises(sp.SynPerfError):
        tr.step(f, m_dev, dev(valid[:65], np.int64))         # B > max_batch
    with pytest.raises(sp.SynPerfError):
        tr.step(f, m_dev, dev(valid[:1], np.int64))          # B < 2
    other = sp.Features.empty(gen.ATTENTION, f.n_pairs, ctx.torch_device)
    with pytest.raises(sp.SynPerfError):
        tr.step(other, m_dev, dev(valid[:8], np.int64))      # family mismatch
    loss = float(tr.step(f, m_dev, dev(valid[:64], np.int64)).item())
    assert np.isfinite(loss)
