"""Seeded synthetic weights for the per-family MLP estimator (input-only).

The paper trains one MLP per kernel category with 3 hidden layers of
256, 128 and 64 units, ReLU -> BatchNorm -> Dropout(0.1), sigmoid output
(P:489).  Its trained weights are not available, so the hot path is exercised
with seeded weights of exactly that architecture (SURVEY §8(c) "Realism ...
parity unpinned").  This module only draws numbers; the arithmetic that uses
them lives in the CUDA path and, independently, in oracle/.

A model is a dict of float32 numpy arrays with the field names of
`sp_mlp_desc` in include/synperf.h:
  mu, sigma [n_in]                       log1p z-score stats (R17)
  w1 [256, n_in], b1 [256], g1/be1/m1/v1 [256]   Linear + BN(eval) layer 1
  w2 [128, 256],  b2 [128], g2/be2/m2/v2 [128]
  w3 [64, 128],   b3 [64],  g3/be3/m3/v3 [64]
  w4 [64], b4 (scalar), bn_eps (scalar)
"""
from __future__ import annotations

import numpy as np

HIDDEN = (256, 128, 64)
N_IN = {0: 11, 1: 15, 2: 11, 3: 15, 4: 15, 5: 11, 6: 11}  # family -> Table IV width (4*pipes + 7)


def _he_uniform(rng, fan_out, fan_in):
    lim = np.sqrt(6.0 / fan_in)
    return rng.uniform(-lim, lim, (fan_out, fan_in)).astype(np.float32)


def random_mlp(family: int, seed: int, bn_eps: float = 1e-5) -> dict:
    """He-uniform weights, small biases, synthetic BN running statistics."""
    rng = np.random.default_rng(seed)
    n_in = N_IN[family]
    m = {"family": family, "n_in": n_in, "bn_eps": np.float32(bn_eps)}
    m["mu"] = rng.uniform(5.0, 25.0, n_in).astype(np.float32)
    m["sigma"] = rng.uniform(2.0, 8.0, n_in).astype(np.float32)
    fan_in = n_in
    for li, width in enumerate(HIDDEN, start=1):
        m[f"w{li}"] = _he_uniform(rng, width, fan_in)
        m[f"b{li}"] = rng.uniform(-0.1, 0.1, width).astype(np.float32)
        m[f"g{li}"] = rng.uniform(0.8, 1.2, width).astype(np.float32)
        m[f"be{li}"] = rng.uniform(-0.1, 0.1, width).astype(np.float32)
        m[f"m{li}"] = rng.uniform(0.2, 0.8, width).astype(np.float32)
        m[f"v{li}"] = rng.uniform(0.3, 1.0, width).astype(np.float32)
        fan_in = width
    m["w4"] = (_he_uniform(rng, 1, 64)[0] * 0.5).astype(np.float32)
    m["b4"] = np.float32(rng.uniform(-0.5, 0.5))
    return m


def zero_output_mlp(family: int, seed: int) -> dict:
    """Final layer zeroed: sigmoid(0) = 0.5, so latency = 2 * t_theory."""
    m = random_mlp(family, seed)
    m["w4"] = np.zeros(64, np.float32)
    m["b4"] = np.float32(0.0)
    return m


def identity_bn_mlp(family: int, seed: int) -> dict:
    """BN made the identity (gamma=1, beta=0, mean=0, var=1-eps): the network
    reduces to a plain Linear/ReLU MLP (a textbook routine to compare against)."""
    m = random_mlp(family, seed)
    eps = float(m["bn_eps"])
    for li, width in enumerate(HIDDEN, start=1):
        m[f"g{li}"] = np.ones(width, np.float32)
        m[f"be{li}"] = np.zeros(width, np.float32)
        m[f"m{li}"] = np.zeros(width, np.float32)
        m[f"v{li}"] = np.full(width, 1.0 - eps, np.float32)
    return m
