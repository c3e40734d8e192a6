"""Probe: does featurize of spec chunk g+1 overlap the tcgen05 predictor of chunk g
when they run on two streams?  (HBM-bound record writer vs TMEM/tensor-bound
persistent predictor; co-residency needs the featurize CTA to fit beside the
predictor's 80 x 672 registers and 218 KB of shared memory.)

    python tools/overlap_probe.py [--workload cfg3] [--reps 10]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--chunk-specs", type=int, default=1)
    args = ap.parse_args()
    ctx = sp.Context(0)
    b, sa, (g0, g1), _ = bench.local_workload(args.workload, 1.0)
    sh = ctx.load_gpu_specs(sa)
    db = sp.DeviceBatch.from_host(b, "cuda:0")
    C = b.n_configs
    n = (g1 - g0) * C
    f = sp.Features.empty(b.family, n, "cuda:0")
    m = ctx.load_model(models.random_mlp(b.family, 3), "fp16")
    lat = torch.empty(n, dtype=torch.float32, device="cuda:0")
    lo, hi = torch.cuda.Stream(priority=0), torch.cuda.Stream(priority=-1)  # predictor: high priority
    ks = args.chunk_specs
    chunks = [(g, min(g + ks, g1)) for g in range(g0, g1, ks)]

    def seq():
        ctx.featurize(db, sh, f, sp.cross(g0, g1))
        ctx.predict(m, f, lat)

    def piped():
        cur = torch.cuda.current_stream()
        lo.wait_stream(cur)
        hi.wait_stream(cur)
        evs = []
        for (a, z) in chunks:
            off, cnt = (a - g0) * C, (z - a) * C
            with torch.cuda.stream(lo):
                ctx.featurize(db, sh, f.view(off, cnt), sp.cross(a, z), stream=lo)
                e = torch.cuda.Event()
                e.record(lo)
            evs.append((e, off, cnt))
        for e, off, cnt in evs:
            hi.wait_event(e)
            with torch.cuda.stream(hi):
                ctx.predict(m, f.view(off, cnt), lat[off:off + cnt], stream=hi)
        cur.wait_stream(hi)
        cur.wait_stream(lo)

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.reps):
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            z.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(z))
        return float(np.median(ts))

    t_seq = timed(seq)
    ref = lat.clone()
    t_pip = timed(piped)
    same = bool(torch.equal(ref, lat))
    print(json.dumps({"workload": args.workload, "pairs": n, "seq_ms": t_seq, "piped_ms": t_pip,
                      "chunks": len(chunks), "identical": same}), flush=True)


if __name__ == "__main__":
    main()
