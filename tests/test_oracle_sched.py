"""Pins of the oracle's GREEDY / MINHEAP schedulers:
SPEC S:186-193 worked examples, hand-simulated attention cases
(tests/golden/scheduler_examples.json), and invariants -- uniform tasks give
the cyclic partition under every scheduler; totals never depend on the
scheduler; enough resident slots make GREEDY cyclic."""
import json
import os

import numpy as np
import pytest

from workloads import gen, specs

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "scheduler_examples.json")))


@pytest.fixture(scope="module")
def modes(orc):
    return {"rr": 0, "greedy": orc.SCHED_GREEDY, "minheap": orc.SCHED_MINHEAP}


@pytest.mark.parametrize("case", ["minheap_spec_1", "minheap_spec_2", "minheap_spec_3"])
def test_minheap_spec_examples(orc, case):
    g = GOLD[case]
    w, sm = orc.schedule_minheap(g["costs"], g["n_sm"], g["occ"])
    assert w.tolist() == g["worker_of"]
    if "loads" in g:
        loads = np.bincount(w, weights=g["costs"], minlength=len(g["loads"]))
        assert loads.tolist() == g["loads"]
    if "sm_of" in g:
        assert sm.tolist() == g["sm_of"]


@pytest.mark.parametrize("case", ["greedy_spec_rr4", "greedy_spec_rr3", "greedy_spec_one", "greedy_retire"])
def test_greedy_examples(orc, case):
    g = GOLD[case]
    assert orc.schedule_greedy(g["costs"], g["n_sm"], g["occ"]).tolist() == g["sm_of"]


def test_greedy_is_cyclic_while_slots_last(orc):
    rng = np.random.default_rng(3)
    c = rng.integers(1, 100, 50)
    assert orc.schedule_greedy(c, 7, 8).tolist() == (np.arange(50) % 7).tolist()  # 7*8 >= 50


def tiny_spec(n_sm: int, occ: int) -> np.ndarray:
    s = specs.spec_by_name("A100")
    s["num_sms"] = n_sm
    s["max_ctas_per_sm"] = occ  # every other occupancy quota is larger for this config
    return s


@pytest.mark.parametrize("k", range(5))
def test_attention_hand_cases(orc, modes, k):
    g = GOLD["attention_greedy"]
    case = g["cases"][k]
    cols = {n: [v] for n, v in g["config"].items()}
    b = gen.make_batch(gen.ATTENTION, cols, ragged=np.array(g["requests"]).ravel(), ragged_off=[0])
    o = orc.featurize(b, tiny_spec(g["n_sm"], case["occ"]), flags=modes[case["mode"]])
    assert o.status[0] == 0
    assert o.ints[1, 0] == case["occ"]
    assert o.ints[6, 0] == max(case["sm_units"]) * g["ops_per_unit"]  # max-SM Tensor ops
    assert o.ints[3, 0] == g["total_units"] * g["ops_per_unit"]
    assert sum(case["sm_units"]) == g["total_units"]


@pytest.mark.parametrize("fam", [gen.GEMM, gen.FUSED_MOE, gen.RMSNORM, gen.SILU_MUL])
def test_uniform_tasks_schedule_independent(orc, modes, fam):
    """Uniform tasks (R2): GREEDY's retirement order and MINHEAP's cyclic
    workers both reproduce cyclic dealing, so every feature is identical."""
    if fam == gen.GEMM:
        b = gen.gen_gemm(40, 5, m_range=(2, 4000), n_range=(384, 4000), k_range=(256, 2000))
    elif fam == gen.FUSED_MOE:
        b = gen.gen_moe(30, 6)
        b = b.subset(np.nonzero(b.field("M") < 600)[0][:10])  # keep the literal task lists small
    else:
        b = gen.gen_rowwise(fam, 30, 7 + fam)
        b.fields[0] = np.minimum(b.fields[0], 3000)
    sa = specs.paper_gpu_specs()[[1, 4, 10]]
    base = orc.featurize(b, sa)
    for m in ("greedy", "minheap"):
        o = orc.featurize(b, sa, flags=modes[m])
        assert np.array_equal(o.status, base.status)
        assert np.array_equal(o.ints, base.ints), m
        np.testing.assert_array_equal(o.flts, base.flts)


def test_totals_schedule_independent_attention(orc, modes):
    b = gen.gen_attention(6, 6, 21, max_bs=3, qlen_max=900, kvlen_max=1500)
    sa = specs.paper_gpu_specs()[[0, 5]]
    base = orc.featurize(b, sa)
    for m in ("greedy", "minheap"):
        o = orc.featurize(b, sa, flags=modes[m])
        ok = base.status == 0
        for k in (0, 1, 2, 3, 4, 5, 9):  # T, occ, waves, totals
            assert np.array_equal(o.ints[k, ok], base.ints[k, ok]), (m, k)
        mean = base.ints[3, ok] / np.array([sa["num_sms"][i // b.n_configs] for i in np.nonzero(ok)[0]])
        assert np.all(o.ints[6, ok] >= mean - 1e-9)  # max >= mean
