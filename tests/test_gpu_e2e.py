"""E2E serving composition on the GPU (sp_e2e_*, through the C-ABI) vs the
literal CPU oracle (oracle/e2e.py).

Bar: the expanded config batches are bit-exact with the oracle's trace
(every invocation's config fields and (qlen, kvlen) list); step and trace
latencies within 1e-5 relative with the fp32 MLP and 1e-2 with the fp16
tcgen05 MLP (north_star's predictor bars: the composition itself is an fp64
sum of the per-kernel predictions).
"""
import numpy as np
import pytest
import torch

from oracle import e2e as E
from workloads import gen, models, specs

pytestmark = pytest.mark.gpu

FAMS = (gen.GEMM, gen.ATTENTION, gen.RMSNORM, gen.SILU_MUL)
RTOL = {"fp32": 1e-5, "fp16": 1e-2}
TOY = dict(n_layers=2, hidden=1024, n_heads=8, n_kv_heads=2, head_dim=128, intermediate=4096,
           vocab=32000)


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_14910_b200 as sp

    return sp


@pytest.fixture(scope="module")
def ctx(sp):
    return sp.Context(0)


def mlps(seed=40):
    return {f: models.random_mlp(f, seed + f) for f in FAMS}


def host_batch(ctx, plan, fam):
    """Copy a plan batch to the host as a gen.ConfigBatch."""
    b = plan.batch(fam).c_struct()
    n = int(b.n_configs)
    nf = int(b.n_fields)
    fields = torch.empty((nf, n), dtype=torch.int32)
    _copy(fields, b.fields, nf * n * 4)
    rag = off = None
    if fam == gen.ATTENTION:
        rag = torch.empty(int(b.n_ragged), dtype=torch.int32)
        off = torch.empty(n, dtype=torch.int64)
        _copy(rag, b.ragged, rag.numel() * 4)
        _copy(off, b.ragged_off, n * 8)
        rag, off = rag.numpy(), off.numpy()
    return gen.ConfigBatch(fam, fields.numpy(), rag, off)


def _copy(dst_host: torch.Tensor, src_ptr: int, nbytes: int):
    """D2H copy of plan-owned device memory (test-side inspection only)."""
    from cuda.bindings import runtime as rt

    torch.cuda.synchronize()
    if nbytes == 0:
        return
    (err,) = rt.cudaMemcpy(dst_host.data_ptr(), src_ptr, nbytes, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
    assert err == rt.cudaError_t.cudaSuccess, err


def oracle_cols(inv):
    return {k: v[0] for k, v in inv.cols.items()}


def assert_plan_matches_oracle(ctx, plan, model, traces):
    """Every invocation of every step of the oracle's literal trace is found,
    field for field, at the slot include/synperf.h documents."""
    inf = plan.info()
    B, NS = inf["max_batch"], inf["n_slots"]
    att = host_batch(ctx, plan, gen.ATTENTION)
    gem = host_batch(ctx, plan, gen.GEMM)
    rms = host_batch(ctx, plan, gen.RMSNORM)
    sil = host_batch(ctx, plan, gen.SILU_MUL)
    m = E.ServingModel(**model)
    s = 0
    kinds = {"qkv": 0, "o_proj": 1, "gate_up": 2, "down": 3}
    for r in range(traces.n_traces):
        tr = E.generate_trace(m, *traces.trace(r))
        for k, invs in enumerate(tr):
            a = next(inv for inv in invs if inv.kind == "attention")
            names = gen.FIELDS[gen.ATTENTION]
            got = {n: int(att.fields[i, s]) for i, n in enumerate(names)}
            assert got == oracle_cols(a), f"attention config of step {s} (trace {r}, k {k})"
            o = int(att.ragged_off[s])
            bs = got["BS"]
            pairs = att.ragged[o:o + 2 * bs].reshape(-1, 2).tolist()
            assert pairs == [list(p) for p in a.requests], f"requests of step {s}"
            M = sum(q for q, _ in a.requests)
            slot = B + r if k == 0 else M - 1
            for inv in invs:
                if inv.kind == "gemm":
                    col = 4 * NS + inv.cols["M"][0] - 1 if inv.name == "lm_head" else kinds[inv.name] * NS + slot
                    got = {n: int(gem.fields[i, col]) for i, n in enumerate(gen.FIELDS[gen.GEMM])}
                    assert got == oracle_cols(inv), f"{inv.name} of step {s}"
                elif inv.kind in ("rmsnorm", "silu_mul"):
                    bt = rms if inv.kind == "rmsnorm" else sil
                    got = {n: int(bt.fields[i, slot]) for i, n in enumerate(gen.FIELDS[bt.family])}
                    assert got == oracle_cols(inv), f"{inv.kind} of step {s}"
            s += 1
    assert s == inf["n_steps"]


def small_traces():
    return gen.make_traces([
        [(300, 4), (120, 1), (77, 3)],
        [(5, 1)],
        [(1000, 2), (1, 6)],
        [(17, 3)] * 40,  # > 32 requests: two ballot passes
    ])


@pytest.mark.parametrize("tp,pp", [(1, 1), (2, 1), (1, 2)])
def test_plan_bit_exact(ctx, tp, pp):
    model = dict(TOY, tp=tp, pp=pp)
    tr = small_traces()
    plan = ctx.e2e_plan(model, tr)
    torch.cuda.synchronize()
    assert_plan_matches_oracle(ctx, plan, model, tr)


def test_plan_bit_exact_serving_sample(ctx):
    tr = gen.gen_serving_traces(6, 77, batches=(8, 12, 16, 48, 64, 3), out_max=60)
    model = gen.serving_model("llama3-8b")
    plan = ctx.e2e_plan(model, tr)
    assert_plan_matches_oracle(ctx, plan, model, tr)


def run_both(sp, ctx, model, traces, precision, spec_arr, comm=None):
    mdl = mlps()
    sh = ctx.load_gpu_specs(spec_arr)
    gm = {f: ctx.load_model(mdl[f], precision) for f in FAMS}
    cm = ctx.load_comm_model(comm) if comm is not None else None
    plan = ctx.e2e_plan(model, traces)
    res = ctx.predict_e2e(plan, sh, gm, cm)
    torch.cuda.synchronize()
    return plan, res, mdl


@pytest.mark.parametrize("precision", ["fp32", "fp16"])
@pytest.mark.parametrize("tp,pp", [(1, 1), (2, 1), (2, 2)])
def test_compose_parity_small(sp, ctx, orc, precision, tp, pp):
    model = dict(TOY, tp=tp, pp=pp)
    sa = specs.paper_gpu_specs()
    comm = specs.synthetic_comm_tables(sa, tp) if (tp > 1 or pp > 1) else None
    tr = small_traces()
    plan, res, mdl = run_both(sp, ctx, model, tr, precision, sa, comm)
    m = E.ServingModel(**model)
    kf = E.kernel_latency_fn(sa, mdl, orc)
    cf = E.comm_latency_fn(comm)
    step = res.step_us.cpu().numpy()
    tot = res.trace_us.cpu().numpy()
    cat = res.trace_cat.cpu().numpy()
    s0 = 0
    for r in range(tr.n_traces):
        o_steps, o_tot, o_cat = E.predict_e2e(E.generate_trace(m, *tr.trace(r)), len(sa), kf, cf)
        ns = o_steps.shape[1]
        np.testing.assert_allclose(step[:, s0:s0 + ns], o_steps, rtol=RTOL[precision], atol=0)
        np.testing.assert_allclose(tot[:, r], o_tot, rtol=RTOL[precision], atol=0)
        np.testing.assert_allclose(cat[:, r, :], o_cat, rtol=RTOL[precision], atol=1e-9)
        s0 += ns
    np.testing.assert_allclose(cat.sum(axis=2), tot, rtol=1e-12)  # additivity


@pytest.mark.parametrize("name", ["llama3-8b", "qwen2.5-14b"])
def test_compose_full_size_sampled(sp, ctx, orc, name):
    """BASELINE config 4 at full size (256 traces, launch config of bench.py)
    for both serving models -- Qwen2.5-14B's 40/8 heads give GQA group 5,
    which does not divide BQ, so its causal prefill runs the general q_last
    path: sampled steps recomputed literally by the oracle; the per-trace
    totals equal the sum of the step latencies (a property at any size)."""
    tr = gen.gen_serving_traces(256, 1004)
    model = gen.serving_model(name)
    sa = specs.paper_gpu_specs()
    plan, res, mdl = run_both(sp, ctx, model, tr, "fp16", sa)
    inf = plan.info()
    step = res.step_us.cpu().numpy()
    tot = res.trace_us.cpu().numpy()
    np.testing.assert_allclose(tot, _seg_sum(step, tr), rtol=1e-5)
    m = E.ServingModel(**model)
    kf = E.kernel_latency_fn(sa, mdl, orc)
    rng = np.random.default_rng(5)
    step_off = np.concatenate([[0], np.cumsum([int(tr.trace(r)[1].max()) for r in range(tr.n_traces)])])
    assert step_off[-1] == inf["n_steps"]
    for r in rng.choice(tr.n_traces, 4, replace=False):
        ins, outs = tr.trace(r)
        steps = E.steps_of_trace(ins, outs)
        for k in sorted(set([0, 1, len(steps) - 1, int(rng.integers(0, len(steps)))])):
            pf, req = steps[k]
            o_steps, _, _ = E.predict_e2e([E.forward_pass(m, req, pf)], len(sa), kf, None)
            np.testing.assert_allclose(step[:, step_off[r] + k], o_steps[:, 0], rtol=1e-2, atol=0)


def _seg_sum(step, tr):
    out = np.zeros((step.shape[0], tr.n_traces))
    s0 = 0
    for r in range(tr.n_traces):
        ns = int(tr.trace(r)[1].max())
        out[:, r] = step[:, s0:s0 + ns].astype(np.float64).sum(axis=1)
        s0 += ns
    return out


def test_update_reuses_plan(sp, ctx):
    model = dict(TOY)
    a, b = small_traces(), gen.make_traces([[(10, 2)], [(3, 3), (4, 1)]])
    plan = ctx.e2e_plan(model, a)
    plan.update(b)
    torch.cuda.synchronize()
    assert_plan_matches_oracle(ctx, plan, model, b)
    plan.update(a)
    assert_plan_matches_oracle(ctx, plan, model, a)


def test_host_api_matches_device_api(sp, ctx):
    model = dict(TOY, tp=2)
    sa = specs.paper_gpu_specs()
    comm = specs.synthetic_comm_tables(sa, 2)
    tr = small_traces()
    plan, res, mdl = run_both(sp, ctx, model, tr, "fp16", sa, comm)
    sh = ctx.load_gpu_specs(sa)
    gm = {f: ctx.load_model(mdl[f], "fp16") for f in FAMS}
    tot, cat = ctx.predict_e2e_host(model, tr, sh, gm, ctx.load_comm_model(comm))
    np.testing.assert_array_equal(tot, res.trace_us.cpu().numpy())
    np.testing.assert_array_equal(cat, res.trace_cat.cpu().numpy())


def test_errors(sp, ctx):
    with pytest.raises(sp.SynPerfError, match="SP_E_DATA"):
        ctx.e2e_plan(dict(TOY), gen.make_traces([[(10, 1)], []]))
    with pytest.raises(sp.SynPerfError, match="SP_E_DATA"):
        ctx.e2e_plan(dict(TOY), gen.make_traces([[(10, 0)]]))
    with pytest.raises(sp.SynPerfError, match="SP_E_ARG"):
        ctx.e2e_plan(dict(TOY, tp=3), gen.make_traces([[(10, 1)]]))
    with pytest.raises(sp.SynPerfError, match="SP_E_ARG"):
        ctx.e2e_plan(dict(TOY, pp=3), gen.make_traces([[(10, 1)]]))
    sa = specs.paper_gpu_specs()
    with pytest.raises(sp.SynPerfError, match="SP_E_ARG"):  # tp > 1 without a comm model
        run_both(sp, ctx, dict(TOY, tp=2), small_traces(), "fp16", sa, None)
    bad = specs.synthetic_comm_tables(sa, 2)
    bad["allreduce_us"][0, 3] = bad["allreduce_us"][0, 2] - 1.0  # decreasing
    with pytest.raises(sp.SynPerfError, match="SP_E_DATA"):
        ctx.load_comm_model(bad)
