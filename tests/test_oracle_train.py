"""Pins of the training oracle (oracle/train.py; PAPER §V-C, §VII-A).

What pins it, independently of its own formulas:
  * SPEC's loss examples, typed in as printed;
  * central finite differences of the loss for every parameter tensor (the
    backward pass is the only hand-written chain rule here);
  * torch.nn fp64 (Linear, ReLU, BatchNorm1d in train mode, sigmoid) for the
    forward pass and the running statistics, and torch.optim.AdamW fp64 for
    the update (library routines);
  * the splitmix64 reference value (first output of seed 0) and the keep-rate
    of the dropout generator;
  * convergence: SPEC S:349-350's fixtures (sigmoid(3x) to < 2% MAPE; the
    pinball model to the P80 of U(0.5, 0.9) = 0.82).
"""
import numpy as np
import pytest
import torch

from oracle import train as T
from workloads import models


def small_model(n_in, seed):
    m = models.random_mlp(0, seed)
    rng = np.random.default_rng(seed)
    m["n_in"] = n_in
    m["w1"] = (rng.uniform(-1, 1, (256, n_in)) * np.sqrt(6.0 / n_in)).astype(np.float32)
    return T.init_params(m)


# ------------------------------------------------------------------ losses (SPEC)

def test_mape_examples():
    assert T.loss_mape(np.array([110.0, 180.0]), np.array([100.0, 200.0])) == pytest.approx(0.10)
    assert T.loss_mape(np.array([3.0]), np.array([3.0])) == 0.0
    assert T.loss_mape(np.array([0.5]), np.array([1.0])) == pytest.approx(0.5)


def test_pinball_examples():
    assert T.loss_pinball(np.array([0.7]), np.array([0.9]), 0.8) == pytest.approx(0.16)
    assert T.loss_pinball(np.array([0.7]), np.array([0.5]), 0.8) == pytest.approx(0.04)
    assert T.loss_pinball(np.array([0.4]), np.array([0.4]), 0.8) == 0.0


# ------------------------------------------------------------------ dropout generator

def test_splitmix64_reference_value():
    """splitmix64's first output for seed 0 is 0xE220A8397B1DCDAF (the published
    sequence); the keep-mask counter 1 (step 0, layer 0, row 0, col 1) hashes
    exactly that state."""
    assert int(T.splitmix64(np.uint64(0x9E3779B97F4A7C15))) == 0xE220A8397B1DCDAF


def test_dropout_keep_rate_and_independence():
    k = T.dropout_keep(7, 3, 1, 4096, 256, 0.1)
    n = k.size
    rate = k.mean()
    assert abs(rate - 0.9) < 4 * np.sqrt(0.09 / n)
    k2 = T.dropout_keep(7, 4, 1, 4096, 256, 0.1)
    k3 = T.dropout_keep(7, 3, 2, 4096, 256, 0.1)
    assert (k != k2).mean() == pytest.approx(0.18, abs=0.01)  # independent masks: 2 p (1 - p)
    assert (k != k3).mean() == pytest.approx(0.18, abs=0.01)
    assert np.array_equal(k, T.dropout_keep(7, 3, 1, 4096, 256, 0.1))
    assert T.dropout_keep(7, 3, 1, 8, 8, 0.0).all()


# ------------------------------------------------------------------ backward vs finite differences

@pytest.mark.parametrize("loss", ["mape", "pinball"])
def test_gradients_match_finite_differences(loss):
    rng = np.random.default_rng(3)
    n_in, B = 11, 24
    p = small_model(n_in, 5)
    x = rng.normal(size=(B, n_in))
    t = rng.uniform(0.2, 0.9, B)
    cfg = dict(T.DEFAULTS, loss=loss, seed=11)
    e, cache = T.forward_train(p, x, 2, cfg["seed"], cfg["drop"], cfg["eps"])
    g = T.backward(p, cache, t, loss, cfg["q"], cfg["drop"], cfg["eps"])

    def L():
        e2, _ = T.forward_train(p, x, 2, cfg["seed"], cfg["drop"], cfg["eps"])
        return T.loss_value(e2, t, loss, cfg["q"])

    h = 1e-6
    for k in T.PARAM_ORDER:
        flat = p[k].reshape(-1)
        idx = rng.choice(flat.size, min(6, flat.size), replace=False)
        for i in idx:
            old = flat[i]
            flat[i] = old + h
            lp = L()
            flat[i] = old - h
            lm = L()
            flat[i] = old
            fd = (lp - lm) / (2 * h)
            an = g[k].reshape(-1)[i]
            scale = max(abs(fd), abs(an), 1e-3 * np.abs(g[k]).max(), 1e-10)
            assert abs(fd - an) / scale < 1e-4, (k, i, fd, an)


# ------------------------------------------------------------------ forward / running stats vs torch.nn

def test_forward_and_running_stats_match_torch():
    rng = np.random.default_rng(4)
    n_in, B = 15, 64
    p = small_model(n_in, 6)
    x = rng.normal(size=(B, n_in))
    e, cache = T.forward_train(p, x, 0, 9, 0.1, 1e-5)
    layers = []
    fan = n_in
    for l, width in zip((1, 2, 3), T.HIDDEN):
        lin = torch.nn.Linear(fan, width).double()
        bn = torch.nn.BatchNorm1d(width, eps=1e-5, momentum=0.1).double()
        with torch.no_grad():
            lin.weight.copy_(torch.from_numpy(p[f"w{l}"]))
            lin.bias.copy_(torch.from_numpy(p[f"b{l}"]))
            bn.weight.copy_(torch.from_numpy(p[f"g{l}"]))
            bn.bias.copy_(torch.from_numpy(p[f"be{l}"]))
            bn.running_mean.copy_(torch.from_numpy(p[f"m{l}"]))
            bn.running_var.copy_(torch.from_numpy(p[f"v{l}"]))
        layers.append((lin, bn, torch.from_numpy(cache[f"keep{l}"].astype(np.float64))))
        fan = width
    h = torch.from_numpy(x)
    for lin, bn, keep in layers:
        bn.train()
        h = bn(torch.relu(lin(h))) * keep / (1.0 - float(np.float32(0.1)))
    et = torch.sigmoid(h @ torch.from_numpy(p["w4"]) + p["b4"][0]).detach().numpy()
    np.testing.assert_allclose(e, et, rtol=1e-12, atol=0)
    T.update_running(p, cache, 0.1, B)
    for l, (lin, bn, _) in zip((1, 2, 3), layers):
        np.testing.assert_allclose(p[f"m{l}"], bn.running_mean.numpy(), rtol=1e-12)
        np.testing.assert_allclose(p[f"v{l}"], bn.running_var.numpy(), rtol=1e-12)


def test_adamw_matches_torch():
    rng = np.random.default_rng(8)
    p = small_model(11, 7)
    st = T.new_adam_state(p)
    tp = {k: torch.nn.Parameter(torch.from_numpy(p[k].copy())) for k in T.PARAM_ORDER}
    opt = torch.optim.AdamW(list(tp.values()), lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01)
    for _ in range(3):
        g = {k: rng.normal(size=p[k].shape) * 10.0 ** rng.uniform(-6, 0) for k in T.PARAM_ORDER}
        T.adamw(p, g, st, 1e-3, 0.01)
        for k in T.PARAM_ORDER:
            tp[k].grad = torch.from_numpy(g[k])
        opt.step()
    for k in T.PARAM_ORDER:
        np.testing.assert_allclose(p[k], tp[k].detach().numpy(), rtol=1e-12, atol=1e-15)


def test_fit_norm_textbook():
    v = np.array([[0.0, 1.0], [np.e - 1, 3.0], [np.e ** 2 - 1, 7.0]])
    mu, sg = T.fit_norm(v)
    np.testing.assert_allclose(mu, [1.0, np.log([2, 4, 8]).mean()])
    np.testing.assert_allclose(sg, [np.std([0, 1, 2]), np.std(np.log([2, 4, 8]))])


# ------------------------------------------------------------------ convergence

def _fit(p, x, t, cfg, epochs, bs, seed):
    st = T.new_adam_state(p)
    rng = np.random.default_rng(seed)
    step = 0
    for _ in range(epochs):
        perm = rng.permutation(len(x))
        for i in range(0, len(x) - bs + 1, bs):
            b = perm[i:i + bs]
            T.train_step(p, st, x[b], t[b], step, cfg)
            step += 1


def test_converges_on_sigmoid_3x():
    """1-D target sigmoid(3x), 2000 samples -> validation MAPE < 2%."""
    rng = np.random.default_rng(12)
    x = rng.uniform(-1, 1, (2200, 1))
    t = 1.0 / (1.0 + np.exp(-3 * x[:, 0]))
    p = small_model(1, 13)
    cfg = dict(T.DEFAULTS, seed=5)
    _fit(p, x[:2000], t[:2000], cfg, 60, 128, 1)
    assert T.loss_mape(T.forward_eval(p, x[2000:], 1e-5), t[2000:]) < 0.02


def test_pinball_converges_to_p80():
    """constant features, t = 0.5 + U(0, 0.4) -> prediction -> P80 = 0.82."""
    rng = np.random.default_rng(14)
    x = np.ones((2048, 3))
    t = 0.5 + rng.uniform(0, 0.4, 2048)
    p = small_model(3, 15)
    cfg = dict(T.DEFAULTS, loss="pinball", q=0.8, seed=6, lr=3e-3)
    _fit(p, x, t, cfg, 150, 256, 2)
    pred = T.forward_eval(p, x[:4], 1e-5)
    assert pred == pytest.approx(0.82, abs=0.02)
