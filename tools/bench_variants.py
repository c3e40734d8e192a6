"""Throughput of the §8(f) variants on one B200 (one JSON line each):
  * sp_featurize_sched GREEDY / MINHEAP on a slice of BASELINE config 2
    (attention x 11 GPUs; sequential scheduler simulation, warp per pair);
  * sp_featurize_ex SP_FEAT_CLAMPED (clamped edge tiles) vs the padded path,
    GEMM, fused MoE and attention x 11 GPUs;
  * sp_perf_gap (P80 gap diagnosis) over BASELINE config 3 (fused MoE x 11,
    the paper applies it to its fused-MoE dataset);
  * sp_train_step (on-GPU estimator training, NEXT-4) on config-3 features at
    minibatch 256 (the SPEC default) and 4096: steps/s, samples/s, per-kernel
    device times (sp_set_profiling) and FLOP rate (6 x forward MACs per sample).
Device-timed with CUDA events, median of --reps after warm-up.

    python tools/bench_variants.py [--reps 5] [--scale 0.02]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_14910_b200 as sp  # noqa: E402
from workloads import models  # noqa: E402


def timed(fn, reps):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--scale", type=float, default=0.02, help="fraction of config 2 for the scheduler variants")
    args = ap.parse_args()
    ctx = sp.Context(0)
    # ---- scheduler variants on a config-2 slice
    b, sa, (g0, g1), _ = bench.local_workload("cfg2", args.scale)
    sh = ctx.load_gpu_specs(sa)
    db = sp.DeviceBatch.from_host(b, "cuda:0")
    n = (g1 - g0) * b.n_configs
    f = sp.Features.empty(b.family, n, "cuda:0")
    for mode in ("rr", "greedy", "minheap"):
        ms = timed(lambda: ctx.featurize(db, sh, f, sp.cross(g0, g1), scheduler=mode), args.reps)
        print(json.dumps({"variant": f"featurize_{mode}", "workload": f"cfg2 x{args.scale}", "pairs": n,
                          "ms": ms, "pairs_per_s": n / (ms * 1e-3)}), flush=True)
    # ---- clamped edge tiles (SP_FEAT_CLAMPED): GEMM (config-1 shapes) and fused MoE (config 3), x 11 GPUs
    from workloads import gen, specs as wspecs
    for name, bb in (("gemm 1e5 x 11", gen.gen_gemm(100_000, 1001)), ("cfg3 x0.1", bench.local_workload("cfg3", 0.1)[0]),
                     ("cfg2 x0.02", bench.local_workload("cfg2", 0.02)[0])):
        sa2 = wspecs.paper_gpu_specs()
        sh2 = ctx.load_gpu_specs(sa2)
        db2 = sp.DeviceBatch.from_host(bb, "cuda:0")
        n2 = len(sa2) * bb.n_configs
        f2 = sp.Features.empty(bb.family, n2, "cuda:0")
        for clamped in (False, True):
            ms = timed(lambda: ctx.featurize(db2, sh2, f2, clamped=clamped), args.reps)
            print(json.dumps({"variant": "featurize_clamped" if clamped else "featurize_padded", "workload": name,
                              "pairs": n2, "ms": ms, "pairs_per_s": n2 / (ms * 1e-3)}), flush=True)
    # ---- gap diagnosis over config 3
    b, sa, (g0, g1), _ = bench.local_workload("cfg3", 1.0)
    sh = ctx.load_gpu_specs(sa)
    db = sp.DeviceBatch.from_host(b, "cuda:0")
    n = (g1 - g0) * b.n_configs
    f = sp.Features.empty(b.family, n, "cuda:0")
    ctx.featurize(db, sh, f)
    m = ctx.load_model(models.random_mlp(b.family, 80), "fp16")
    lat = torch.empty(n, dtype=torch.float32, device="cuda:0")
    eff = torch.empty(n, dtype=torch.float32, device="cuda:0")
    ctx.predict(m, f, lat, eff)
    meas = lat * torch.empty_like(lat).uniform_(1.0, 3.0)  # synthetic "measured" latencies
    pr = sp.cross(g0, g1)
    ms = timed(lambda: ctx.perf_gap(f, eff, meas, pr, n_configs=b.n_configs), args.reps)
    _, counts, _ = ctx.perf_gap(f, eff, meas, pr, n_configs=b.n_configs)
    c = counts.cpu().numpy()
    nbytes = n * (4 + 1 + 4 + 4 + 4)  # t_theory, status, y_p80, measured read; gap written
    print(json.dumps({"variant": "perf_gap", "workload": "cfg3", "pairs": n, "ms": ms,
                      "pairs_per_s": n / (ms * 1e-3), "achieved_gbs": nbytes / (ms * 1e-3) / 1e9,
                      "underperforming": int(c[:, 1].sum()), "valid": int(c[:, 0].sum())}), flush=True)
    # ---- estimator training on the same features
    valid = torch.nonzero(torch.from_numpy(sp.features_to_host(f)[2] == 0)).view(-1).cuda()
    n_in = 11
    flop = 6 * (n_in * 256 + 256 * 128 + 128 * 64 + 64)  # fwd 2 x MACs, bwd 2 x that (dX + dW)
    for B in (256, 4096):
        tr = ctx.trainer(models.random_mlp(b.family, 81), max_batch=B, seed=3)
        g = torch.Generator(device="cuda:0")
        g.manual_seed(0)
        batches = [valid[torch.randint(0, valid.numel(), (B,), generator=g, device="cuda:0")] for _ in range(50)]

        def run():
            for bi in batches:
                tr.step(f, meas, bi)

        ctx.set_profiling(True)
        ctx.profile_read(reset=True)
        ms = timed(run, args.reps) / len(batches)
        kst = ctx.profile_read(reset=True)
        ctx.set_profiling(False)
        ms_np = timed(run, args.reps) / len(batches)  # without the per-launch events
        buf = torch.empty(B, dtype=torch.int64, device="cuda:0")
        graph = tr.capture(f, meas, buf)

        def run_graph():
            for bi in batches:
                buf.copy_(bi)
                graph.replay()

        ms_graph = timed(run_graph, args.reps) / len(batches)
        print(json.dumps({"variant": "train_step", "workload": "cfg3 features", "batch": B,
                          "ms_per_step": ms_np, "steps_per_s": 1e3 / ms_np, "samples_per_s": B * 1e3 / ms_np,
                          "graph_ms_per_step": ms_graph, "graph_samples_per_s": B * 1e3 / ms_graph,
                          "tflops": flop * B / (ms_np * 1e-3) / 1e12,
                          "launches_per_step": sum(v[0] for v in kst.values()) / ((args.reps + 2) * len(batches)),
                          "kernels_ms_per_step": {k: v[1] / ((args.reps + 2) * len(batches)) for k, v in kst.items()}}),
              flush=True)


if __name__ == "__main__":
    main()
