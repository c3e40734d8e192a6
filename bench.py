#!/usr/bin/env python
"""Benchmark of the B200 SynPerf hot path: predictions/sec over (kernel config x
GPU spec) pairs.  One step = feature stage (sp_featurize) + predictor stage
(sp_predict) over one batch of synthetic pairs [+ the NCCL all-gather of
predictions when N > 1], through the C-ABI.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg2]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...
    python bench.py --impl reference ...   # the fp64 CPU oracle arm

Rank 0 prints ONE JSON line (contract in the task statement / DESIGN.md §7).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import gen, models, specs  # noqa: E402

BASELINE_METRIC = "predictions/sec (kernel-config×GPU pairs) at 1/2/4/8 B200; % HBM / tensor peak"
UNIT = "pairs/s"
MLP_FLOP_PER_PAIR = {11: 87_680, 15: 89_728}  # 2*(n_in*256 + 256*128 + 128*64 + 64), SURVEY §8(a) a11
RECORD_BYTES = 11 * 8 + 12 * 4 + 1  # a9: 137 B/pair written


# ----------------------------------------------------------------- workloads

WORKLOADS = {
    "cfg1": "1,000 GEMM configs x 1 GPU spec (A100, Table VI)",
    "cfg2": "FlashAttention prefill/decode sweep, 1e6 configs x the paper's 11 GPU specs",
    "cfg3": "fused MoE Triton config space, 1e6 configs x 11 GPU specs",
    "cfg4": "E2E serving iterations: Llama-3-8B + Qwen2.5-14B over 256 static-batch request traces "
            "(arxiv/splitwise-like), per-kernel predictions composed per step, x 11 GPU specs",
    "cfg5": "1,000 serving GEMMs x 100,000 hypothetical GPU specs (1e8 pairs), sharded by spec",
    "scaledmm": "FP8 Scaled MM (block-wise quantisation) space of P:480, 1e6 configs x 11 GPU specs "
                "(not a BASELINE config: NEXT-4 variant)",
    "splitk": "split-K GEMM space (long K, few output tiles; reading R25), 1e6 configs x 11 GPU specs "
              "(not a BASELINE config: NEXT-4 variant)",
}
FUSABLE = (gen.GEMM, gen.FUSED_MOE, gen.RMSNORM, gen.SILU_MUL, gen.SCALED_MM)
E2E_MODELS = ("llama3-8b", "qwen2.5-14b")
E2E_FAMILIES = (gen.GEMM, gen.ATTENTION, gen.RMSNORM, gen.SILU_MUL)


def build_workload(name: str, rank: int, world: int, scale: float = 1.0, scaling: str | None = None):
    """Returns (batch, spec_array, (g0, g1), scaling).  Strong scaling (the
    default): the same global workload on every rank, which
    run_gpu shards with dist.Sharder (see SHARDING); weak: rank r's own
    full-size workload (seeded by r) over all specs."""
    weak = scaling == "weak"
    r = rank if weak else 0
    scaling = "weak" if weak else "strong"
    if name == "cfg1":
        return gen.gen_gemm(1000, 1001 + 7919 * r), specs.spec_by_name("A100"), (0, 1), scaling
    if name == "cfg2":
        n = int(500_000 * scale)
        b = gen.gen_attention(n, n, 1002 + 7919 * r)
        sa = specs.paper_gpu_specs()
        return b, sa, (0, len(sa)), scaling
    if name == "cfg3":
        b = gen.gen_moe(int(1_000_000 * scale), 1003 + 7919 * r)
        sa = specs.paper_gpu_specs()
        return b, sa, (0, len(sa)), scaling
    if name == "scaledmm":
        b = gen.gen_scaled_mm(int(1_000_000 * scale), 1006 + 7919 * r)
        sa = specs.paper_gpu_specs()
        return b, sa, (0, len(sa)), scaling
    if name == "splitk":
        b = gen.gen_gemm_splitk(int(1_000_000 * scale), 1007 + 7919 * r)
        sa = specs.paper_gpu_specs()
        return b, sa, (0, len(sa)), scaling
    if name == "cfg5":
        b = gen.gen_serving_gemms(1000, 1005)
        sa = specs.hypothetical_sweep_specs(int(100_000 * scale))
        return b, sa, (0, len(sa)), "strong"  # the 10^8-pair sweep is one workload, sharded by spec
    raise SystemExit(f"unknown workload {name}")


# How the bench shards each workload across ranks (dist.Sharder): the config
# axis after a seeded shuffle (cost balance: attention configs range over five
# orders of magnitude of tasks; at N = 1 the shuffle is the cfg2 order the
# tests use, gen.shuffle(b, 7)), or the spec axis for the 10^5-spec sweep.
SHARDING = {"cfg5": ("spec", None)}
DEFAULT_SHARDING = ("config", 7)


def sharder_for(name: str, b, sa, rank: int, world: int, scaling: str, chunks: int):
    from paper_2601_14910_b200.dist import Sharder

    axis, seed = SHARDING.get(name, DEFAULT_SHARDING)
    if scaling == "weak":  # the rank's own workload, unsharded
        return Sharder(b.n_configs, len(sa), 1, 0, axis, seed, chunks)
    return Sharder(b.n_configs, len(sa), world, rank, axis, seed, chunks)


def local_workload(name: str, scale: float = 1.0):
    """The single-GPU bench workload as run_gpu computes it (the shard of rank 0
    of 1: the global batch in the sharder's order) -- for the tools."""
    b, sa, rng, scaling = build_workload(name, 0, 1, scale)
    sh = sharder_for(name, b, sa, 0, 1, scaling, 1)
    cfg = sh.configs
    if len(cfg) != b.n_configs or not np.array_equal(cfg, np.arange(len(cfg))):
        b = b.subset(cfg)
    return b, sa, rng, scaling


# -------------------------------------------------------------------- clocks

class ClockSampler:
    """Polls NVML during the timed region: SM clock, max clock, throttle reasons."""

    REASONS = {
        "hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
        "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
        "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
        "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
        "hw_power_brake_slowdown": "nvmlClocksEventReasonHwPowerBrakeSlowdown",
    }

    def __init__(self, index: int, period: float = 0.01):
        self.index, self.period = index, period
        self.samples, self.reasons, self.ok = [], set(), False
        self._stop = threading.Event()
        try:
            import pynvml

            self.nv = pynvml
            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # no NVML: report nulls
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, attr in self.REASONS.items():
                    if r & getattr(nv, attr, 0):
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": len(self.samples)}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------- reference (oracle)

def oracle_rate(batch, spec_arr, spec_range, model, target_s: float, seed: int = 0, keep: dict | None = None):
    """Times the fp64 oracle (as it stands) on a bounded random sample of the
    workload's pairs: featurize + predict.  Returns (pairs/s, n_sample, secs,
    threads, single-core pairs/s).  keep: receives the main sample's local pair
    indices and the oracle's features and latencies (the bench's parity check)."""
    from oracle import oracle as O

    O.build()
    rng = np.random.default_rng(seed)
    g0, g1 = spec_range
    total = (g1 - g0) * batch.n_configs

    def run(n, threads=0, store=False):
        p = rng.integers(0, total, n)
        ci, si = p % batch.n_configs, g0 + p // batch.n_configs
        t = time.perf_counter()
        f = O.featurize(batch, spec_arr, cfg_idx=ci, spec_idx=si, nthreads=threads)
        lat, _, _ = O.predict(model, f, nthreads=threads)
        dt = time.perf_counter() - t
        if store and keep is not None:
            keep.update(pairs=p, feats=f, latency=lat)
        return dt

    threads = O.num_threads()
    n = 256
    dt = run(n)
    while dt < 0.5 and n < 10_000_000:
        n *= 4
        dt = run(n)
    n = max(256, int(n * target_s / max(dt, 1e-6)))
    dt = run(n, store=True)
    # one core (SURVEY §8(d) asks for both): a sample sized for ~1/5 of the time budget
    n1 = max(64, int(n / max(threads, 1) * 0.2))
    dt1 = run(n1, 1)
    run(64, threads)  # restore the OpenMP team size
    return n / dt, n, dt, threads, n1 / dt1


def oracle_e2e_rate(traces, sa, mlps, target_s: float, seed: int = 0, keep: list | None = None):
    """Times the literal E2E oracle (oracle/e2e.py) on random serving steps:
    every invocation of the sampled steps featurised + predicted on every spec
    and summed.  Returns (step-spec predictions/s, pairs/s, n_steps, secs, threads).
    keep: receives (model, trace, step, oracle step latency per spec) per sample."""
    from oracle import e2e as E
    from oracle import oracle as O

    O.build()
    rng = np.random.default_rng(seed)
    kf = E.kernel_latency_fn(sa, mlps, O)
    steps = []
    t0 = time.perf_counter()
    n_pairs = 0
    while time.perf_counter() - t0 < target_s or not steps:
        name = E2E_MODELS[len(steps) % len(E2E_MODELS)]
        m = E.ServingModel(**gen.serving_model(name))
        r = int(rng.integers(0, traces.n_traces))
        ins, outs = traces.trace(r)
        st = E.steps_of_trace(ins, outs)
        k = int(rng.integers(0, len(st)))
        pf, req = st[k]
        invs = E.forward_pass(m, req, pf)
        o_steps, _, _ = E.predict_e2e([invs], len(sa), kf, None)
        if keep is not None:
            keep.append((name, r, k, o_steps[:, 0]))
        n_pairs += len(invs) * len(sa)
        steps.append((name, r))
    dt = time.perf_counter() - t0
    return len(steps) * len(sa) / dt, n_pairs / dt, len(steps), dt, O.num_threads()


def run_reference(args, rank, world):
    if rank != 0:
        return
    if args.workload == "cfg4":
        return run_reference_e2e(args)
    b, sa, rng_, _ = build_workload(args.workload, 0, 1, args.scale)
    model = models.random_mlp(b.family, 42)
    budget = 150.0 / max(1, args.steps + args.warmup)
    per_step = min(10.0, budget)
    from oracle import oracle as O

    O.build()
    # size one step's sample from a calibration run
    _, n_cal, dt_cal, threads, _ = oracle_rate(b, sa, rng_, model, target_s=min(2.0, per_step), seed=1)
    n_step = max(256, int(n_cal * per_step / max(dt_cal, 1e-6)))
    rng = np.random.default_rng(11)
    g0, g1 = rng_
    total = (g1 - g0) * b.n_configs
    times = []
    for s in range(args.warmup + args.steps):
        p = rng.integers(0, total, n_step)
        ci, si = p % b.n_configs, g0 + p // b.n_configs
        t = time.perf_counter()
        f = O.featurize(b, sa, cfg_idx=ci, spec_idx=si)
        O.predict(model, f)
        if s >= args.warmup:
            times.append(time.perf_counter() - t)
    tot = float(np.sum(times))
    value = n_step * args.steps / tot
    sample = (f"{n_step} random pairs per step of workload {args.workload} "
              f"({total} pairs), featurize + predict, fp64")
    line = {
        "impl": "reference", "metric": BASELINE_METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "description": WORKLOADS[args.workload],
                   "pairs_per_step": n_step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_reference_e2e(args):
    traces = gen.gen_serving_traces(256, 1004)
    sa = specs.paper_gpu_specs()
    mlps = {f: models.random_mlp(f, 42 + f) for f in E2E_FAMILIES}
    per_step = min(10.0, 150.0 / max(1, args.steps + args.warmup))
    times, rates = [], []
    for s in range(args.warmup + args.steps):
        sps, pps, n, dt, threads = oracle_e2e_rate(traces, sa, mlps, per_step, seed=100 + s)
        if s >= args.warmup:
            times.append(dt)
            rates.append((sps, pps, n))
    tot = float(np.sum(times))
    value = float(np.sum([r[1] * t for r, t in zip(rates, times)]) / tot)
    steps_ps = float(np.sum([r[0] * t for r, t in zip(rates, times)]) / tot)
    sample = (f"random serving steps of the cfg4 traces (Llama-3-8B / Qwen2.5-14B), every invocation "
              f"featurised + predicted literally on 11 specs, ~{per_step:.0f} s per step, fp64")
    line = {
        "impl": "reference", "metric": BASELINE_METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg4", "description": WORKLOADS["cfg4"]},
        "step_predictions_per_s": steps_ps,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm

def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def device_of(local_rank: int, args) -> int:
    """The rank's GPU: LOCAL_RANK, or all ranks on GPU 0 for the gloo functional check."""
    return local_rank if args.dist_backend == "nccl" else 0


def run_gpu(args, rank, world, local_rank):
    import torch

    import paper_2601_14910_b200 as sp
    from paper_2601_14910_b200.dist import ShardedPredictor

    local_rank = device_of(local_rank, args)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:  # functional check of the N > 1 path on a single GPU (timings meaningless)
            dist.init_process_group("gloo")
    ctx = sp.Context(local_rank)
    b, sa, (g0, g1), scaling = build_workload(args.workload, rank, world, args.scale, args.scaling)
    # the all-gather of chunk k overlaps chunk k+1's compute; each extra chunk costs a launch tail
    # (measured at N = 1: 4 chunks +16% on cfg2, +7% on cfg3), so N > 1 defaults to 2
    chunks = args.chunks if args.chunks > 0 else (1 if world == 1 else 2)
    sharder = sharder_for(args.workload, b, sa, rank, world, scaling, chunks)
    specs_h = ctx.load_gpu_specs(sa)
    model_d = models.random_mlp(b.family, 42)
    precision = args.precision
    model = ctx.load_model(model_d, precision)
    n_in = int(model_d["n_in"])
    # this rank's shard: configs sharder.configs x specs sharder.spec_range, uploaded once
    pred = ShardedPredictor(ctx, b, sa, model, sharder, specs=specs_h)
    g0, g1 = sharder.spec_range
    n_pairs = sharder.local_pairs
    stream = torch.cuda.current_stream()
    gather = world > 1 and not args.no_gather
    gathered_weak = None
    if gather and scaling == "weak":  # every rank's own full workload: one all-gather of it
        gathered_weak = torch.empty(world * sharder.padded_pairs, dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    if args.scheduler != "rr" or (args.fused == "off" and b.family in FUSABLE) or precision == "fp32":
        # variants outside the fused pass: sp_featurize_sched + sp_predict (unsharded, rank-local)
        feats_v = sp.Features.empty(b.family, n_pairs, dev)
        lat_v = torch.empty(max(n_pairs, 1), dtype=torch.float32, device=dev)

        def compute():
            ctx.featurize(pred.db, specs_h, feats_v, sp.cross(g0, g1), stream, scheduler=args.scheduler)
            ctx.predict(model, feats_v, lat_v, None, stream)
    else:
        feats_v = lat_v = None

        def compute():
            if scaling == "strong" and gather:
                pred.run()  # chunk by chunk, the all-gather of chunk k overlapping chunk k+1
            else:
                pred.run(gather=False)
                if gathered_weak is not None:
                    dist.all_gather_into_tensor(gathered_weak, pred.local)

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        compute()
        if ev is not None:
            ev[1].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ctx.profile_read(reset=True)
    ctx.set_profiling(True)  # per-kernel CUDA events on the launch stream (sp_set_profiling)
    with ClockSampler(local_rank) as clk:
        for s in range(args.steps):
            flush.zero_()  # L2 flush between timed steps, outside the events
            step(evs[s])
        torch.cuda.synchronize()
    ctx.set_profiling(False)
    kst = ctx.profile_read(reset=True)  # {kernel: (launches, device ms)} of the timed region
    if dist is not None:
        dist.barrier()
    t_step = np.array([e[0].elapsed_time(e[1]) for e in evs])
    tot_ms = float(t_step.sum())
    if dist is not None:
        t = torch.tensor([tot_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    pairs_all = n_pairs * world if scaling == "weak" else len(sa) * b.n_configs
    value = pairs_all * args.steps / (tot_ms * 1e-3)

    # the last step's records and latencies in this rank's local order (one chunk: all of them)
    one_pass = feats_v is not None or len(sharder.chunk_bounds()) == 1
    feats = feats_v if feats_v is not None else pred.feats
    lat = lat_v if lat_v is not None else pred.last
    if one_pass:  # sanity: no NaN outside error pairs
        st = feats.status[:n_pairs]
        bad = int(((st == 0) & torch.isnan(lat[:n_pairs])).sum().item())
        if bad:
            raise SystemExit(f"{bad} valid pairs produced NaN latency")

    # ---- e2e through the public API with host buffers (this rank's shard)
    local_b = b if (sharder.axis == "spec" or np.array_equal(sharder.configs, np.arange(b.n_configs))) \
        else b.subset(sharder.configs)
    e2e = run_e2e(args, ctx, specs_h, model, local_b, (g0, g1), dev, dist, world, scaling, len(sa),
                  pairs_all)

    # ---- roofline of the dominant kernel
    peaks = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json")) or {}
    prof = load_json(os.path.join(ROOT, "profiles", "ncu_traffic.json")) or {}
    n_chunks = 1 if feats_v is not None else len(sharder.chunk_bounds())
    roof = roofline(args, local_b, n_pairs / n_chunks, n_in, precision, kst, peaks, prof, tot_ms)
    if b.family == gen.ATTENTION and roof["kernel"] == "attn_schedule_cross" and one_pass:
        roof["algorithmic"] = attention_work(local_b, sa, (g0, g1), feats, roof["avg_launch_ms"])
    stage = {}
    for k, (n, t) in kst.items():
        key = "predict" if k.startswith("predict") else "featurize"
        stage[key] = stage.get(key, 0.0) + t / args.steps
    stage["other (copies, all-gather wait)"] = max(0.0, tot_ms / args.steps - sum(stage.values()))

    line = {
        "metric": BASELINE_METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
        "dtype": {"bf16": "bf16", "fp16": "f16", "fp32": "f32"}[precision],
        "data": "synthetic (seeded generators, workloads/; seeded random MLP weights)",
        "config": {
            "workload": args.workload, "description": WORKLOADS[args.workload],
            "pairs_per_gpu": n_pairs, "configs_per_gpu": b.n_configs, "specs": g1 - g0,
            "family": gen.FAMILY_NAMES[b.family], "mlp_precision": precision,
            "scheduler": args.scheduler,
            "parallelism": f"dp{world}" + ("+allgather" if gather else ""),
            "sharding": {"axis": sharder.axis, "seeded_shuffle": sharder.axis == "config" and
                         SHARDING.get(args.workload, DEFAULT_SHARDING)[1] is not None,
                         "allgather_chunks": n_chunks if gather else 0,
                         "pairs_this_rank": n_pairs, "pairs_total": pairs_all},
            "l2": "flushed between timed steps (256 MiB write, outside the events)",
        },
        "stage_ms": stage,
        "roofline": roof,
        "kernels": {k: {"launches": n, "avg_ms": t / max(n, 1)} for k, (n, t) in sorted(kst.items())},
        "e2e": e2e,
        "gpu_launches": int(sum(n for n, _ in kst.values())),
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        keep = {}
        v, n, dt, thr, v1 = oracle_rate(b, sa, (g0, g1), model_d, target_s=args.cpu_seconds, keep=keep)
        line["cpu_baseline"] = {
            "value": v, "unit": UNIT, "cores": thr, "kind": "oracle",
            "sample": f"{n} random pairs of this workload, fp64 oracle featurize+predict, {dt:.1f} s",
            "single_core_value": v1}
        if one_pass:
            line["parity"] = parity_stats(keep, feats, lat, precision, sharder)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def parity_stats(keep, feats, lat, precision, sharder):
    """north_star's bar on this run's own output: the GPU records and latencies
    of the last timed step at the cpu_baseline sample's pairs, against the
    oracle's values for the same pairs (computed by the timed oracle run).
    The sample's pairs are global (g * C + c); the run's buffers are in the
    shard's local order [g][position of c in sharder.configs] (N = 1)."""
    import torch

    p = keep["pairs"]
    o = keep["feats"]
    C = sharder.n_configs
    inv = np.empty(C, dtype=np.int64)
    inv[sharder.configs] = np.arange(C)
    local = (p // C) * C + inv[p % C]
    idx = torch.from_numpy(local).to(feats.status.device)
    gs = feats.status[idx].cpu().numpy()
    gi = feats.ints[:, idx].cpu().numpy()
    gf = feats.flts[:, idx].cpu().numpy().astype(np.float64)
    gl = lat[idx].cpu().numpy().astype(np.float64)
    ok = o.status == 0
    with np.errstate(divide="ignore", invalid="ignore"):
        rf = np.abs(gf[:, ok] / o.flts[:, ok] - 1.0)
        rf = np.where(o.flts[:, ok] == 0, np.abs(gf[:, ok]), rf)
        rl = np.abs(gl[ok] / keep["latency"][ok] - 1.0)
    bar = 1e-5 if precision == "fp32" else 1e-2
    max_f = float(rf.max()) if rf.size else 0.0
    max_l = float(rl.max()) if rl.size else 0.0
    res = {"pairs": int(len(p)), "valid_pairs": int(ok.sum()),
           "status_mismatches": int((gs != o.status).sum()),
           "int_mismatches": int((gi != o.ints).any(axis=0).sum()),
           "max_rel_float": max_f, "max_rel_latency": max_l,
           "float_bar": 1e-5, "latency_bar": bar,
           "sample": "the cpu_baseline sample's pairs; GPU output of the last timed step"}
    res["pass"] = bool(res["status_mismatches"] == 0 and res["int_mismatches"] == 0 and max_f <= 1e-5
                       and max_l <= bar)
    return res


def run_gpu_e2e(args, rank, world, local_rank):
    """cfg4: one step = for each serving model, re-expand the plan on the GPU
    (sp_e2e_plan_expand), featurise + predict the four families' batches x 11
    specs, and compose per-step / per-trace latencies (sp_e2e_compose) [+ the
    all-gather of per-trace totals when N > 1].  Weak scaling: every rank has
    its own 256 traces."""
    import torch

    import paper_2601_14910_b200 as sp

    local_rank = device_of(local_rank, args)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:  # functional check of the N > 1 path on a single GPU (timings meaningless)
            dist.init_process_group("gloo")
    ctx = sp.Context(local_rank)
    n_tr = max(1, int(256 * args.scale))
    traces = gen.gen_serving_traces(n_tr, 1004 + 7919 * rank)
    sa = specs.paper_gpu_specs()
    G = len(sa)
    specs_h = ctx.load_gpu_specs(sa)
    mlps = {f: models.random_mlp(f, 42 + f) for f in E2E_FAMILIES}
    mdl = {f: ctx.load_model(mlps[f], args.precision) for f in E2E_FAMILIES}
    stream = torch.cuda.current_stream()
    plans = [ctx.e2e_plan(gen.serving_model(n), traces, stream) for n in E2E_MODELS]
    infos = [p.info() for p in plans]
    pairs_per_step = sum(G * p["n_configs"][f] for p in infos for f in E2E_FAMILIES)
    step_preds = sum(G * p["n_steps"] for p in infos)
    invocations = 0
    for name, p in zip(E2E_MODELS, plans):
        L = gen.serving_model(name)["n_layers"]
        invocations += G * p.info()["n_steps"] * (8 * L + 2)
    tot_all = torch.empty((len(plans), G, n_tr), dtype=torch.float64, device=dev)
    gathered = torch.empty(world * tot_all.numel(), dtype=torch.float64, device=dev) if dist else None
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    results = [None] * len(plans)

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        for i, p in enumerate(plans):
            p.expand(stream)
            r = ctx.predict_e2e(p, specs_h, mdl, None, (0, G), step_latencies=True, stream=stream)
            results[i] = r
            tot_all[i].copy_(r.trace_us)
        if gathered is not None:
            dist.all_gather_into_tensor(gathered, tot_all.view(-1))
        if ev is not None:
            ev[1].record(stream)
        return r

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if torch.isnan(tot_all).any():
        raise SystemExit("NaN trace latency")
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ctx.profile_read(reset=True)
    ctx.set_profiling(True)
    with ClockSampler(local_rank) as clk:
        for s in range(args.steps):
            flush.zero_()
            step(evs[s])
        torch.cuda.synchronize()
    ctx.set_profiling(False)
    kst = ctx.profile_read(reset=True)
    # the last timed step's composed step latencies (the parity check below; host API calls reuse buffers)
    steps_gpu = {name: results[i].step_us.cpu().numpy() for i, name in enumerate(E2E_MODELS)}
    if dist is not None:
        dist.barrier()
    t_step = np.array([e[0].elapsed_time(e[1]) for e in evs])
    tot_ms = float(t_step.sum())
    if dist is not None:
        t = torch.tensor([tot_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    value = pairs_per_step * world * args.steps / (tot_ms * 1e-3)

    # ---- e2e through the public host API: host traces in, host per-trace latencies out
    for _ in range(2):
        for n in E2E_MODELS:
            ctx.predict_e2e_host(gen.serving_model(n), traces, specs_h, mdl)
    e_steps = max(1, min(args.steps, args.e2e_steps))
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e_steps):
        for n in E2E_MODELS:
            ctx.predict_e2e_host(gen.serving_model(n), traces, specs_h, mdl)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    if dist is not None:
        tt = torch.tensor([el], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        el = float(tt.item())
    h2d = len(E2E_MODELS) * (traces.req_off.nbytes + traces.input_len.nbytes + traces.output_len.nbytes)
    d2h = len(E2E_MODELS) * G * n_tr * 8 * (1 + 5)
    e2e = {"value": pairs_per_step * world * e_steps / el, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(d2h), "steps": e_steps,
           "api": "Context.predict_e2e_host (host request traces -> H2D -> GPU expansion -> "
                  "sp_featurize/sp_predict x 4 families -> sp_e2e_compose -> D2H per-trace latencies)"}

    peaks = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json")) or {}
    prof = load_json(os.path.join(ROOT, "profiles", "ncu_traffic.json")) or {}
    roof = roofline_e2e(infos, G, kst, peaks, prof, tot_ms, args)
    line = {
        "metric": BASELINE_METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": {"bf16": "bf16", "fp16": "f16", "fp32": "f32"}[args.precision],
        "data": "synthetic (seeded request traces and MLP weights, workloads/)",
        "config": {
            "workload": "cfg4", "description": WORKLOADS["cfg4"], "traces_per_gpu": n_tr,
            "requests_per_gpu": int(traces.req_off[-1]), "models": list(E2E_MODELS), "specs": G,
            "serving_steps_per_gpu": int(sum(p["n_steps"] for p in infos)),
            "pairs_per_gpu": pairs_per_step, "mlp_precision": args.precision,
            "parallelism": f"dp{world}" + ("+allgather" if gathered is not None else ""),
            "l2": "flushed between timed steps (256 MiB write, outside the events)",
        },
        "step_predictions_per_s": step_preds * world * args.steps / (tot_ms * 1e-3),
        "invocations_per_s": invocations * world * args.steps / (tot_ms * 1e-3),
        "roofline": roof,
        "kernels": {k: {"launches": n, "avg_ms": t / max(n, 1)} for k, (n, t) in sorted(kst.items())},
        "e2e": e2e,
        "gpu_launches": int(sum(n for n, _ in kst.values())),
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        keep = []
        sps, pps, n, dt, thr = oracle_e2e_rate(traces, sa, mlps, args.cpu_seconds, keep=keep)
        line["cpu_baseline"] = {
            "value": pps, "unit": UNIT, "cores": thr, "kind": "oracle",
            "step_predictions_per_s": sps,
            "sample": f"{n} random serving steps, every invocation featurised + predicted literally "
                      f"on 11 specs (fp64 oracle), {dt:.1f} s"}
        # parity: the GPU's composed step latencies of the last timed step at the sampled steps
        step_off = np.concatenate([[0], np.cumsum([int(traces.trace(r)[1].max()) for r in range(n_tr)])])
        rel = [np.abs(steps_gpu[name][:, step_off[r] + k].astype(np.float64) / o - 1.0).max()
               for name, r, k, o in keep]
        bar = 1e-5 if args.precision == "fp32" else 1e-2
        line["parity"] = {"steps": len(keep), "step_spec_values": len(keep) * G,
                          "max_rel_step_latency": float(max(rel)), "latency_bar": bar,
                          "pass": bool(max(rel) <= bar),
                          "sample": "the cpu_baseline sample's serving steps (literal oracle: every "
                                    "invocation of the step featurised + predicted); GPU step latencies "
                                    "of the last timed step"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def roofline_e2e(infos, G, kst, peaks, prof, tot_ms, args):
    """Dominant kernel of a cfg4 step; its algorithmic work summed over the
    step's launches (different batch sizes per family) / its summed device time."""
    kernel, (launches, total) = max(kst.items(), key=lambda kv: kv[1][1])
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    long_region = tot_ms > 1000.0
    wp = prof.get("cfg4", {}) or {}
    steps = args.steps
    if kernel.startswith("predict"):
        flop = steps * sum(G * p["n_configs"][f] * MLP_FLOP_PER_PAIR[models.N_IN[f]]
                           for p in infos for f in E2E_FAMILIES)
        achieved = flop / (total * 1e-3) / 1e12
        key = "bf16_tflops_sustained" if long_region else "bf16_tflops"
        peak, bound, unit, src = peaks.get(key), "tensor", "TFLOP/s", f"MEASURED_PEAKS.json {key}"
        per_unit = "MLP FLOP/pair (87,680 F=11; 89,728 F=15) x pairs of all launches"
    elif kernel == "attn_schedule_cross":
        instr = wp.get("attn_schedule_cross_inst_executed")  # per step (ncu, all launches of one step)
        achieved = None if instr is None else instr * steps / (total * 1e-3) / 1e9
        peak = 4 * 148 * sm_mhz * 1e6 / 1e9
        bound, unit, src = "alu", "Ginstr/s", "4 warp-instr/clk/SM x 148 x sm_max_mhz (DESIGN.md §6)"
        per_unit = "warp instructions per step (ncu smsp__inst_executed.sum summed over the step's launches)"
    else:
        nbytes = steps * sum(G * p["n_configs"][f] for p in infos for f in E2E_FAMILIES) * RECORD_BYTES
        achieved = nbytes / (total * 1e-3) / 1e9
        peak, bound, unit, src = peaks.get("hbm_gbs"), "hbm", "GB/s", "MEASURED_PEAKS.json hbm_gbs"
        per_unit = f"{RECORD_BYTES} B/pair written"
    return {"kernel": kernel, "bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
            "frac": (achieved / peak) if (achieved is not None and peak) else None,
            "traffic": wp.get(f"{kernel}_dram_bytes"), "avg_launch_ms": total / max(launches, 1),
            "launches": launches, "per_unit": per_unit, "peak_source": src}


def run_e2e(args, ctx, specs_h, model, b, spec_range, dev, dist, world, scaling, n_specs, pairs_all):
    """Same metric through Context.predict_host with pinned host buffers: every
    step copies the configs H2D and the fp32 latencies D2H."""
    import torch

    fields = torch.from_numpy(b.fields).pin_memory()
    ragged = torch.from_numpy(b.ragged).pin_memory() if b.ragged is not None else None
    roff = torch.from_numpy(b.ragged_off).pin_memory() if b.ragged_off is not None else None

    class HostBatch:
        family = b.family

    hb = HostBatch()
    hb.fields, hb.ragged, hb.ragged_off = fields, ragged, roff
    g0, g1 = spec_range
    n_pairs = (g1 - g0) * b.n_configs
    out = torch.empty(n_pairs, dtype=torch.float32).pin_memory()
    h2d = fields.numel() * 4 + (ragged.numel() * 4 if ragged is not None else 0) + \
        (roff.numel() * 8 if roff is not None else 0)
    d2h = n_pairs * 4
    for _ in range(max(1, min(args.warmup, 2))):
        ctx.predict_host(hb, specs_h, model, spec_range, out=out)
    steps = max(1, min(args.steps, args.e2e_steps))
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(steps):
        ctx.predict_host(hb, specs_h, model, spec_range, out=out)
    torch.cuda.synchronize()
    el = time.perf_counter() - t
    if dist is not None:
        tt = torch.tensor([el], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        el = float(tt.item())
    return {"value": pairs_all * steps / el, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": steps,
            "api": "sp_predict_host via Context.predict_host (pinned host configs -> pipelined H2D -> "
                   "sp_featurize_predict -> D2H latencies, all inside libsynperf)"}


def attention_work(b, sa, spec_range, feats, ms):
    """Algorithmic work of one attn_schedule_cross launch, counted from its own
    output: head-0 tasks (a config's task count T / nkv, the record's first
    slot) x the distinct SM counts of the spec range (the kernel
    accumulates one residue table per distinct N), and the (pair, task) units
    the records describe (sum of T over all pairs)."""
    import torch

    g0, g1 = spec_range
    C = b.n_configs
    T0 = feats.ints[0, :C].clamp(min=0)  # spec g0's records: pair p = c
    nkv = torch.from_numpy(b.field("NKV").astype(np.int64)).to(T0.device)
    head0 = int((T0 // nkv).sum().item())
    distinct = int(len(np.unique(sa["num_sms"][g0:g1])))
    pair_tasks = int(feats.ints[0, :(g1 - g0) * C].clamp(min=0).sum().item())
    units = head0 * distinct
    return {"units_per_launch": units, "unit": "head-0 task x distinct SM count",
            "units_per_s": units / (ms * 1e-3), "head0_tasks": head0, "distinct_sm_counts": distinct,
            "pair_tasks_per_launch": pair_tasks, "pair_tasks_per_s": pair_tasks / (ms * 1e-3)}


def roofline(args, b, n_pairs, n_in, precision, kst, peaks, prof, tot_ms):
    """Roofline object for the dominant kernel of the step: the kernel with
    the largest device time in the timed region (per-kernel CUDA events, sp_set_profiling);
    achieved = its algorithmic work per launch / its measured average launch time."""
    hbm = peaks.get("hbm_gbs")
    long_region = tot_ms > 1000.0
    bf16_peak = peaks.get("bf16_tflops_sustained" if long_region else "bf16_tflops")
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    kernel, (launches, total) = max(kst.items(), key=lambda kv: kv[1][1])
    ms = total / max(launches, 1)
    per_launch_pairs = n_pairs  # one launch covers the step's pairs (featurize / predict)
    wp = prof.get(args.workload, {}) or {}
    if kernel.startswith("predict"):
        flop = MLP_FLOP_PER_PAIR[n_in] * per_launch_pairs
        achieved = flop / (ms * 1e-3) / 1e12
        if precision != "fp32":  # fp16 and bf16 share the dense tensor rate (guide: ratio 1)
            peak, bound, src = bf16_peak, "tensor", ("MEASURED_PEAKS.json " +
                                                     ("bf16_tflops_sustained" if long_region else "bf16_tflops"))
        else:
            # fp32 FFMA peak from unit counts: 148 SMs x 128 lanes x 2 FLOP x max SM clock
            peak, bound, src = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12, "alu", \
                "148 SMs x 128 FP32 lanes x 2 FLOP x sm_max_mhz (DESIGN.md §6)"
        unit, per_unit = "TFLOP/s", f"{MLP_FLOP_PER_PAIR[n_in]} FLOP/pair x {per_launch_pairs} pairs"
        traffic = wp.get(f"{kernel}_{precision}_dram_bytes")
    elif kernel == "attn_schedule_cross":
        # integer-issue roofline: warp instructions per launch (ncu capture of this workload)
        instr = wp.get("attn_schedule_cross_inst_executed")
        achieved = None if instr is None else instr / (ms * 1e-3) / 1e9
        peak = 4 * 148 * sm_mhz * 1e6 / 1e9
        bound, unit, src = "alu", "Ginstr/s", "4 warp-instr/clk/SM x 148 x sm_max_mhz (DESIGN.md §6)"
        per_unit = "warp instructions per launch (ncu smsp__inst_executed.sum, profiles/ncu_traffic.json)"
        traffic = wp.get("attn_schedule_cross_dram_bytes")
    else:  # record-writing kernels: HBM
        nbytes = n_pairs * RECORD_BYTES + b.fields.nbytes + \
            (b.ragged.nbytes if b.ragged is not None else 0)
        achieved = nbytes / (ms * 1e-3) / 1e9
        peak, bound, unit, src = hbm, "hbm", "GB/s", "MEASURED_PEAKS.json hbm_gbs"
        per_unit = f"{RECORD_BYTES} B/pair written + config bytes read"
        traffic = wp.get(f"{kernel}_dram_bytes")
    return {"kernel": kernel, "bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
            "frac": (achieved / peak) if (achieved is not None and peak) else None,
            "traffic": traffic, "avg_launch_ms": ms, "launches": launches, "per_unit": per_unit,
            "peak_source": src}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--scale", type=float, default=1.0, help="workload size multiplier (testing)")
    ap.add_argument("--precision", default="fp16", choices=["fp16", "fp32"])
    ap.add_argument("--scheduler", default="rr", choices=["rr", "greedy", "minheap"],
                    help="Scheduling Simulator variant (sp_featurize_sched; default cyclic RR)")
    ap.add_argument("--fused", default="auto", choices=["auto", "on", "off"],
                    help="sp_featurize_predict for the uniform families (auto) or never (off)")
    ap.add_argument("--no-gather", action="store_true")
    ap.add_argument("--scaling", default=None, choices=["strong", "weak"],
                    help="strong (default): one global workload sharded across ranks; weak: every rank "
                         "its own full-size workload (cfg5 is always strong)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: every rank on GPU 0 over gloo -- a functional check of the N>1 path on a "
                         "one-GPU box, not a measurement")
    ap.add_argument("--chunks", type=int, default=0,
                    help="all-gather chunks overlapped with compute (0: 1 at N=1, 2 at N>1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--e2e-steps", type=int, default=5)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.workload == "cfg4":
        run_gpu_e2e(args, rank, world, local_rank)
        return
    run_gpu(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
