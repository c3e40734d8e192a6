"""Pins of the E2E composition oracle (oracle/e2e.py) against what SPEC/PAPER
fix: worked examples (tests/golden/e2e_examples.json, cited per case), closed-
form invocation counts, additivity and permutation invariance,
and the interpolation identities of the comm estimator."""
import json
import os

import numpy as np
import pytest

from oracle import e2e as E
from workloads import gen, specs

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "e2e_examples.json")))


def toy(tp=1, pp=1):
    return E.ServingModel(**GOLD["toy_model"], tp=tp, pp=pp)


def split(reqs):
    return [i for i, _ in reqs], [o for _, o in reqs]


def count(trace):
    comp = sum(1 for s in trace for inv in s if inv.family >= 0)
    comm = sum(1 for s in trace for inv in s if inv.family < 0)
    return comp, comm


@pytest.mark.parametrize("case", ["toy_prefill_tp1", "toy_prefill_tp2", "toy_pp2"])
def test_spec_invocation_counts(case):
    g = GOLD[case]
    tr = E.generate_trace(toy(g["tp"], g.get("pp", 1)), *split(g["requests"]))
    assert len(tr) == g.get("n_steps", 1)
    assert count(tr) == (g["n_compute"], g["n_comm"])


def test_template_order():
    """S:556 template, one layer: RMSNorm, QKV, Attention, O, AR, RMSNorm, GateUp, SiLU, Down, AR."""
    tr = E.generate_trace(toy(2), [10], [1])
    names = [inv.name for inv in tr[0][:10]]
    assert names == ["input_norm", "qkv", "attention", "o_proj", "allreduce", "post_attn_norm",
                     "gate_up", "silu_mul", "down", "allreduce"]
    assert [inv.name for inv in tr[0][-2:]] == ["final_norm", "lm_head"]


def test_decode_growth():
    g = GOLD["decode_growth"]
    tr = E.generate_trace(toy(), *split(g["requests"]))
    assert len(tr) == len(g["steps"])
    for step, want in zip(tr, g["steps"]):
        attn = [inv for inv in step if inv.kind == "attention"]
        assert len(attn) == toy().n_layers
        assert [list(r) for r in attn[0].requests] == want["attn"]
        assert attn[0].cols["CAUSAL"] == [1 if want["prefill"] else 0]
        gem = {inv.name: inv for inv in step if inv.kind == "gemm"}
        assert gem["qkv"].cols["M"] == [want["M"]]
        assert gem["lm_head"].cols["M"] == [want["lm_M"]]
        rms = [inv for inv in step if inv.kind == "rmsnorm"]
        assert all(inv.cols["SEQ"] == [want["M"]] for inv in rms)


@pytest.mark.parametrize("tp", [1, 2])
def test_llama3_gemm_shapes(tp):
    g = GOLD["llama3_8b_gemms"][f"tp{tp}"]
    m = E.ServingModel(**gen.serving_model("llama3-8b", tp=tp))
    tr = E.generate_trace(m, [7, 9], [1, 1])
    gem = {inv.name: inv for inv in tr[0] if inv.kind == "gemm"}
    for name, (n, k) in g.items():
        assert (gem[name].cols["N"][0], gem[name].cols["K"][0]) == (n, k), name
    attn = next(inv for inv in tr[0] if inv.kind == "attention")
    assert attn.cols["NH"] == [32 // tp] and attn.cols["NKV"] == [8 // tp]


def test_comm_interpolation():
    g = GOLD["comm_interp"]
    for nbytes, want in g["queries"]:
        assert E.predict_comm(g["bytes"], g["us"], nbytes) == pytest.approx(want, rel=1e-12)
    assert E.predict_comm(g["bytes"], g["us"], 1 << 40) == 30.0  # clamped flat above (E7)


def test_comm_interpolation_is_linear_in_log_bytes():
    """Closed form: between two points the latency is affine in ln(bytes)."""
    xs, ys = [1e3, 1e5, 1e7], [5.0, 9.0, 40.0]
    for x in (2e3, 3.3e4, 9.9e4, 1e6, 5e6):
        i = 0 if x < 1e5 else 1
        t = np.log(x / xs[i]) / np.log(xs[i + 1] / xs[i])
        assert E.predict_comm(xs, ys, x) == pytest.approx(ys[i] + t * (ys[i + 1] - ys[i]), rel=1e-12)


def const_kernel(v):
    return lambda inv: np.full(3, float(v))


def test_additivity_spec_example():
    g = GOLD["additivity"]
    trace = [[E.Invocation("gemm", 0, name=str(i)) for i in range(3)]]
    lats = iter(g["lat"])
    steps, total, cats = E.predict_e2e(trace, 1, lambda inv: np.array([next(lats)]), None)
    assert total[0] == g["total"] and cats.sum() == g["total"]


def test_counting_closed_form():
    """Every compute kernel 1 us, every collective 0: a trace's total is
    S_r * (8L + 2), S_r = max output_len (E2), for any tp."""
    reqs = [(40, 5), (13, 2), (77, 4)]
    for tp in (1, 2):
        m = toy(tp)
        tr = E.generate_trace(m, *split(reqs))
        steps, total, cats = E.predict_e2e(tr, 3, const_kernel(1.0), lambda inv: np.zeros(3))
        assert np.all(total == 5 * (8 * m.n_layers + 2))
        assert np.all(cats[:, E.CAT_GEMM] == 5 * (4 * m.n_layers + 1))
        assert np.all(cats[:, E.CAT_ATTENTION] == 5 * m.n_layers)
        assert np.all(cats[:, E.CAT_RMSNORM] == 5 * (2 * m.n_layers + 1))
        assert np.all(cats[:, E.CAT_SILU] == 5 * m.n_layers)
        assert np.all(cats[:, E.CAT_COMM] == 0)


def test_tp1_has_zero_comm():
    tr = E.generate_trace(toy(1), [30, 20], [3, 2])
    assert count(tr)[1] == 0


def test_comm_bytes_and_count():
    """TP=2: 2 AllReduce per layer of M*hidden*2 bytes; sum of comm = 2L * table(M*h*2)."""
    sa = specs.paper_gpu_specs()
    comm = specs.synthetic_comm_tables(sa, 2)
    m = toy(2)
    tr = E.generate_trace(m, [100, 28], [1, 1])
    _, _, cats = E.predict_e2e(tr, len(sa), lambda inv: np.zeros(len(sa)),
                               E.comm_latency_fn(comm))
    nb = 128 * m.hidden * 2
    for g in range(len(sa)):
        want = 2 * m.n_layers * E.predict_comm(comm["bytes"], comm["allreduce_us"][g], nb)
        assert cats[g, E.CAT_COMM] == pytest.approx(want, rel=1e-12)


def test_permutation_invariance():
    """permuting trace order leaves the total unchanged."""
    rng = np.random.default_rng(0)
    tr = E.generate_trace(toy(2), [30, 20, 5], [4, 2, 3])
    lat = {id(inv): rng.uniform(1, 100, 2) for s in tr for inv in s}
    f = lambda inv: lat[id(inv)]  # noqa: E731
    _, t0, _ = E.predict_e2e(tr, 2, f, f)
    flat = [inv for s in tr for inv in s]
    perm = [flat[i] for i in rng.permutation(len(flat))]
    _, t1, _ = E.predict_e2e([perm], 2, f, f)
    np.testing.assert_allclose(t0, t1, rtol=1e-12)


def test_divisibility_errors():
    with pytest.raises(ValueError):
        E.generate_trace(toy(3), [10], [1])
    with pytest.raises(ValueError):
        E.generate_trace(toy(1, 3), [10], [1])
    with pytest.raises(ValueError):
        E.generate_trace(toy(), [10, 0], [1, 1])


def test_tile_rule_boundaries():
    """Reading E4 boundaries (M = 64 | 65, 256 | 257)."""
    t = {M: E.gemm_invocation("x", M, 4096, 4096).cols for M in (1, 64, 65, 256, 257, 10000)}
    assert (t[64]["TM"], t[64]["TN"], t[64]["WARPS"], t[64]["REGS"]) == ([64], [128], [4], [128])
    assert (t[65]["TM"], t[65]["TN"], t[65]["WARPS"], t[65]["REGS"]) == ([128], [128], [8], [168])
    assert (t[257]["TM"], t[257]["TN"], t[257]["STAGES"], t[257]["REGS"]) == ([128], [256], [3], [232])


def test_real_estimator_runs_small(orc):
    """The literal composition with the fp64 oracle estimators: positive, and
    the prefill step (all tokens) costs more than any single decode step."""
    from workloads import models

    sa = specs.paper_gpu_specs()[:3]
    mdl = {f: models.random_mlp(f, 10 + f) for f in (0, 1, 3, 4)}
    tr = E.generate_trace(toy(), [300, 200], [3, 2])
    steps, total, cats = E.predict_e2e(tr, len(sa), E.kernel_latency_fn(sa, mdl, orc), None)
    assert np.all(steps > 0)
    assert np.all(steps[:, 0] > steps[:, 1:].max(axis=1))
    np.testing.assert_allclose(cats.sum(axis=1), total, rtol=1e-12)
