"""Quick A/B timing of the two stages on a BASELINE workload (no oracle, no e2e).

    SYNPERF_LIB=variants/lib_x.so python tools/time_stages.py [--workload cfg2] [--reps 10]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_14910_b200 as sp  # noqa: E402
from workloads import models  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--precision", default="fp16")
    ap.add_argument("--fused", action="store_true", help="also time sp_featurize_predict (the bench step)")
    args = ap.parse_args()
    ctx = sp.Context(0)
    b, sa, (g0, g1), _ = bench.local_workload(args.workload, args.scale)
    sh = ctx.load_gpu_specs(sa)
    md = models.random_mlp(b.family, 42)
    m = ctx.load_model(md, args.precision)
    db = sp.DeviceBatch.from_host(b, "cuda:0")
    n = (g1 - g0) * b.n_configs
    f = sp.Features.empty(b.family, n, "cuda:0")
    lat = torch.empty(n, dtype=torch.float32, device="cuda:0")
    pr = sp.cross(g0, g1)
    for _ in range(3):
        ctx.featurize(db, sh, f, pr)
        ctx.predict(m, f, lat)
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.reps)]
    for e in ev:
        e[0].record()
        ctx.featurize(db, sh, f, pr)
        e[1].record()
        ctx.predict(m, f, lat)
        e[2].record()
    torch.cuda.synchronize()
    tf = sorted(e[0].elapsed_time(e[1]) for e in ev)
    tp = sorted(e[1].elapsed_time(e[2]) for e in ev)
    fused = ""
    if args.fused:
        for _ in range(3):
            ctx.featurize_predict(db, sh, m, f, lat, pairs=pr)
        ef = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.reps)]
        for e in ef:
            e[0].record()
            ctx.featurize_predict(db, sh, m, f, lat, pairs=pr)
            e[1].record()
        torch.cuda.synchronize()
        tz = sorted(e[0].elapsed_time(e[1]) for e in ef)
        fused = f"  fused {tz[len(tz)//2]:.3f} ms (min {tz[0]:.3f})"
    print(f"{os.environ.get('SYNPERF_LIB', 'default')}: featurize {tf[len(tf)//2]:.3f} ms (min {tf[0]:.3f})  "
          f"predict {tp[len(tp)//2]:.3f} ms (min {tp[0]:.3f}){fused}  pairs {n}")


if __name__ == "__main__":
    main()
