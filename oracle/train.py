"""Oracle of the estimator's training step (PAPER §V-C, §VII-A P:670;
SURVEY §8(f) NEXT-4 "on-GPU batched MLP training (AdamW + MAPE/pinball)").

TEST INFRASTRUCTURE ONLY (see oracle/oracle.py's header): tests/ are the only
callers; the product package never imports this module.

Plain numpy, fp64, one array operation per line of the algorithm, in the
paper's order (readings T1..T9):
  forward (train mode), per hidden layer l = 1..3 ("ReLU activations
  followed by Batch Normalization and Dropout (rate 0.1)"):
      z = h W^T + b ; a = relu(z)
      mu = mean_B(a) ; var = mean_B((a - mu)^2)          (T2: batch statistics, biased)
      a_hat = (a - mu) / sqrt(var + eps) ; y = gamma a_hat + beta
      h = y * keep / (1 - p)                             (T3: inverted dropout, keep mask below)
  output: z4 = h3 . w4 + b4 ; e = sigmoid(z4)            (P:489 sigmoid = efficiency)
  loss (T4): MAPE  mean_B |e - t| / max(t, 1e-6)
             pinball(q) mean_B max(q (t - e), (q - 1)(t - e))  (P:670 quantile loss)
  backward: the chain rule of the lines above, written out by hand
  AdamW (T5): m = b1 m + (1-b1) g ; v = b2 v + (1-b2) g^2
      theta -= lr * (wd * theta + (m / (1-b1^t)) / (sqrt(v / (1-b2^t)) + eps_adam))
  running statistics (T6): rm = (1-mom) rm + mom mu ; rv = (1-mom) rv + mom var B/(B-1)
The dropout keep mask is a counter-based generator (T3) that the CUDA path
implements independently: splitmix64's finaliser of seed + ctr * 0x9E3779B97F4A7C15,
ctr = (((step * 4 + layer) * 2^20 + row) * 2^8 + col), keep iff bits 63..40 >= round(p * 2^24).
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
HIDDEN = (256, 128, 64)
PARAM_ORDER = ["w1", "b1", "g1", "be1", "w2", "b2", "g2", "be2", "w3", "b3", "g3", "be3", "w4", "b4"]


def splitmix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser (uint64 arithmetic, wrapping)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def dropout_keep(seed: int, step: int, layer: int, rows: int, cols: int, p: float) -> np.ndarray:
    """T3 keep mask [rows, cols] of hidden layer `layer` (0..2) at training step `step`."""
    r = np.arange(rows, dtype=np.uint64)[:, None]
    c = np.arange(cols, dtype=np.uint64)[None, :]
    base = (np.uint64(step) * np.uint64(4) + np.uint64(layer)) << np.uint64(20)
    ctr = ((base + r) << np.uint64(8)) + c
    with np.errstate(over="ignore"):
        z = splitmix64(np.uint64(seed) + ctr * GOLDEN)
    thr = int(round(float(np.float32(p)) * (1 << 24)))
    return (z >> np.uint64(40)) >= np.uint64(thr)


def loss_mape(e: np.ndarray, t: np.ndarray) -> float:
    """MAPE (T4): mean |e - t| / t with t clamped below at 1e-6."""
    tc = np.maximum(t, 1e-6)
    return float(np.mean(np.abs(e - t) / tc))


def loss_pinball(e: np.ndarray, t: np.ndarray, q: float) -> float:
    """Quantile (pinball) loss: mean max(q (t - e), (q - 1)(t - e))."""
    d = t - e
    return float(np.mean(np.maximum(q * d, (q - 1.0) * d)))


def _dloss_de(e, t, loss, q):
    """dL/de of T4 (subgradient 0 at e == t)."""
    B = e.shape[0]
    if loss == "mape":
        return np.sign(e - t) / np.maximum(t, 1e-6) / B
    return (np.where(e > t, 1.0 - q, 0.0) - np.where(t > e, q, 0.0)) / B


def init_params(model: dict) -> dict:
    """fp64 copies of the trainable parameters and the running statistics of a
    workloads/models.py model dict."""
    p = {k: np.asarray(model[k], dtype=np.float64).copy() for k in PARAM_ORDER[:-1]}
    p["b4"] = np.array([float(model["b4"])])
    for l in (1, 2, 3):
        p[f"m{l}"] = np.asarray(model[f"m{l}"], dtype=np.float64).copy()
        p[f"v{l}"] = np.asarray(model[f"v{l}"], dtype=np.float64).copy()
    return p


def forward_train(p: dict, x: np.ndarray, step: int, seed: int, drop: float, eps: float):
    """Train-mode forward; returns (e, cache)."""
    cache = {"h0": x}
    h = x
    for l, width in zip((1, 2, 3), HIDDEN):
        z = h @ p[f"w{l}"].T + p[f"b{l}"]
        a = np.maximum(z, 0.0)
        mu = a.mean(axis=0)
        var = ((a - mu) ** 2).mean(axis=0)
        a_hat = (a - mu) / np.sqrt(var + eps)
        y = p[f"g{l}"] * a_hat + p[f"be{l}"]
        keep = dropout_keep(seed, step, l - 1, x.shape[0], width, drop)
        h = y * keep / (1.0 - float(np.float32(drop)))
        cache.update({f"z{l}": z, f"mu{l}": mu, f"var{l}": var, f"ahat{l}": a_hat, f"keep{l}": keep,
                      f"h{l}": h})
    z4 = h @ p["w4"] + p["b4"][0]
    e = 1.0 / (1.0 + np.exp(-z4))
    cache["e"] = e
    return e, cache


def forward_eval(p: dict, x: np.ndarray, eps: float) -> np.ndarray:
    """Eval-mode forward (running statistics, no dropout): the predictor's O10-O11."""
    h = x
    for l in (1, 2, 3):
        a = np.maximum(h @ p[f"w{l}"].T + p[f"b{l}"], 0.0)
        h = p[f"g{l}"] * (a - p[f"m{l}"]) / np.sqrt(p[f"v{l}"] + eps) + p[f"be{l}"]
    return 1.0 / (1.0 + np.exp(-(h @ p["w4"] + p["b4"][0])))


def backward(p: dict, cache: dict, t: np.ndarray, loss: str, q: float, drop: float, eps: float) -> dict:
    """Gradients of the batch loss w.r.t. every trainable parameter."""
    g = {}
    e = cache["e"]
    dz4 = _dloss_de(e, t, loss, q) * e * (1.0 - e)
    g["w4"] = cache["h3"].T @ dz4
    g["b4"] = np.array([dz4.sum()])
    dh = np.outer(dz4, p["w4"])
    scale = 1.0 / (1.0 - float(np.float32(drop)))
    for l in (3, 2, 1):
        dy = dh * cache[f"keep{l}"] * scale
        a_hat = cache[f"ahat{l}"]
        g[f"g{l}"] = (dy * a_hat).sum(axis=0)
        g[f"be{l}"] = dy.sum(axis=0)
        dahat = dy * p[f"g{l}"]
        inv_std = 1.0 / np.sqrt(cache[f"var{l}"] + eps)
        da = inv_std * (dahat - dahat.mean(axis=0) - a_hat * (dahat * a_hat).mean(axis=0))
        dz = da * (cache[f"z{l}"] > 0)
        g[f"w{l}"] = dz.T @ cache[f"h{l - 1}"]
        g[f"b{l}"] = dz.sum(axis=0)
        dh = dz @ p[f"w{l}"]
    return g


def loss_value(e, t, loss, q):
    return loss_mape(e, t) if loss == "mape" else loss_pinball(e, t, q)


def new_adam_state(p: dict) -> dict:
    return {"t": 0, "m": {k: np.zeros_like(p[k]) for k in PARAM_ORDER},
            "v": {k: np.zeros_like(p[k]) for k in PARAM_ORDER}}


def adamw(p: dict, g: dict, st: dict, lr, wd, b1=0.9, b2=0.999, eps=1e-8):
    """AdamW (T5): decoupled weight decay on every parameter, bias-corrected moments."""
    st["t"] += 1
    t = st["t"]
    for k in PARAM_ORDER:
        st["m"][k] = b1 * st["m"][k] + (1.0 - b1) * g[k]
        st["v"][k] = b2 * st["v"][k] + (1.0 - b2) * g[k] * g[k]
        m_hat = st["m"][k] / (1.0 - b1 ** t)
        v_hat = st["v"][k] / (1.0 - b2 ** t)
        p[k] = p[k] - lr * (wd * p[k] + m_hat / (np.sqrt(v_hat) + eps))


def update_running(p: dict, cache: dict, momentum: float, B: int):
    """T6: PyTorch BatchNorm1d running statistics (unbiased variance)."""
    for l in (1, 2, 3):
        p[f"m{l}"] = (1.0 - momentum) * p[f"m{l}"] + momentum * cache[f"mu{l}"]
        p[f"v{l}"] = (1.0 - momentum) * p[f"v{l}"] + momentum * cache[f"var{l}"] * B / (B - 1)


def train_step(p, st, x, t, step, cfg) -> float:
    """One minibatch step; returns the (pre-update) batch loss.  cfg: dict with
    loss, q, lr, wd, b1, b2, adam_eps, drop, bn_momentum, eps, seed."""
    e, cache = forward_train(p, x, step, cfg["seed"], cfg["drop"], cfg["eps"])
    L = loss_value(e, t, cfg["loss"], cfg["q"])
    g = backward(p, cache, t, cfg["loss"], cfg["q"], cfg["drop"], cfg["eps"])
    update_running(p, cache, cfg["bn_momentum"], x.shape[0])
    adamw(p, g, st, cfg["lr"], cfg["wd"], cfg["b1"], cfg["b2"], cfg["adam_eps"])
    return L


def fit_norm(v: np.ndarray):
    """T7 (R17's statistics): per feature mean and population standard deviation
    of ln(1 + v) over the rows of v [n, n_in]."""
    lv = np.log1p(np.asarray(v, dtype=np.float64))
    mu = lv.mean(axis=0)
    return mu, np.sqrt(((lv - mu) ** 2).mean(axis=0))


DEFAULTS = dict(loss="mape", q=0.8, lr=1e-3, wd=0.01, b1=0.9, b2=0.999, adam_eps=1e-8, drop=0.1,
                bn_momentum=0.1, eps=1e-5, seed=0)
