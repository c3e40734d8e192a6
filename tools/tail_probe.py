"""Does the attention schedule kernel pay a load-imbalance tail?  Times
sp_featurize on cfg2 in the bench's (shuffled) config order and with the
configs sorted by descending estimated cost (head-0 q-blocks x kv-heads x
kv units, from the host arrays).

    python tools/tail_probe.py [--reps 10]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402  (SYNPERF_LIB selects the library)

import bench  # noqa: E402
import paper_2601_14910_b200 as sp  # noqa: E402
from workloads import gen  # noqa: E402


def est_cost(b):
    bs = b.field("BS").astype(np.int64)
    nh, nkv, bq = b.field("NH").astype(np.int64), b.field("NKV").astype(np.int64), b.field("BQ").astype(np.int64)
    g = np.maximum(nh // np.maximum(nkv, 1), 1)
    off = b.ragged_off
    q = b.ragged[0::2].astype(np.int64)
    req_cfg = np.repeat(np.arange(b.n_configs), bs)
    rows = q * g[req_cfg]
    nqb = (rows + bq[req_cfg] - 1) // bq[req_cfg]
    L = np.bincount(req_cfg, weights=nqb, minlength=b.n_configs)
    return L * nkv


def time_featurize(ctx, b, sa, reps):
    sh = ctx.load_gpu_specs(sa)
    db = sp.DeviceBatch.from_host(b, "cuda:0")
    f = sp.Features.empty(b.family, len(sa) * b.n_configs, "cuda:0")
    for _ in range(3):
        ctx.featurize(db, sh, f)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.featurize(db, sh, f)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    ctx = sp.Context(0)
    b, sa, _, _ = bench.local_workload("cfg2")
    cost = est_cost(b)
    t0 = time_featurize(ctx, b, sa, args.reps)
    order = np.argsort(-cost, kind="stable")
    t1 = time_featurize(ctx, b.subset(order), sa, args.reps)
    t2 = time_featurize(ctx, b.subset(order[::-1].copy()), sa, args.reps)
    # log2-cost buckets, heaviest bucket first, bench order inside a bucket
    bucket = np.floor(np.log2(np.maximum(cost, 1))).astype(np.int64)
    t3 = time_featurize(ctx, b.subset(np.argsort(-bucket, kind="stable")), sa, args.reps)
    # only the configs with cost >= 2^14 first (bench order otherwise)
    heavy = cost >= 2 ** 14
    t4 = time_featurize(ctx, b.subset(np.concatenate([np.nonzero(heavy)[0], np.nonzero(~heavy)[0]])), sa, args.reps)
    print(f"featurize cfg2: bench order {t0:.3f} ms, heaviest first {t1:.3f} ms, lightest first {t2:.3f} ms, "
          f"log2 buckets {t3:.3f} ms, heavy (>= 2^14) first {t4:.3f} ms; "
          f"max est cost {cost.max():.0f}, mean {cost.mean():.1f}")


if __name__ == "__main__":
    main()
