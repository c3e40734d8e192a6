"""Host-buffer API (Context.predict_host) throughput vs the number of pipeline
slices, for a bench workload (pinned host configs -> H2D -> fused/two-call
kernels -> D2H).

    python tools/e2e_chunks.py [--workload cfg2] [--chunks 1 2 4 8]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_14910_b200 as sp  # noqa: E402
from workloads import models  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--chunks", nargs="+", default=["1", "2", "4", "8"],
                    help="slice counts, or comma-separated slice weights (e.g. 1,3,3,1)")
    ap.add_argument("--reps", type=int, default=4)
    args = ap.parse_args()
    ctx = sp.Context(0)
    b, sa, (g0, g1), _ = bench.local_workload(args.workload, 1.0)
    sh = ctx.load_gpu_specs(sa)
    m = ctx.load_model(models.random_mlp(b.family, 42), "fp16")

    class HB:
        family = b.family

    hb = HB()
    hb.fields = torch.from_numpy(b.fields).pin_memory()
    hb.ragged = None if b.ragged is None else torch.from_numpy(b.ragged).pin_memory()
    hb.ragged_off = None if b.ragged_off is None else torch.from_numpy(b.ragged_off).pin_memory()
    n = (g1 - g0) * b.n_configs
    out = torch.empty(n, dtype=torch.float32).pin_memory()
    for spec_ in args.chunks:
        ch = [float(x) for x in spec_.split(",")] if "," in spec_ else int(spec_)
        for _ in range(2):
            ctx.predict_host(hb, sh, m, (g0, g1), out=out, chunks=ch)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(args.reps):
            ctx.predict_host(hb, sh, m, (g0, g1), out=out, chunks=ch)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t) / args.reps * 1e3
        print(json.dumps({"workload": args.workload, "chunks": spec_, "ms": ms, "pairs_per_s": n / ms * 1e3}), flush=True)


if __name__ == "__main__":
    main()
