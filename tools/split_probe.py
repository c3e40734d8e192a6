"""Where the attention schedule time goes on cfg2: sp_featurize on the prefill
(causal) and decode (non-causal) halves separately, and the whole batch.

    python tools/split_probe.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import paper_2601_14910_b200 as sp  # noqa: E402
import bench  # noqa: E402
from tail_probe import time_featurize  # noqa: E402


def main():
    ctx = sp.Context(0)
    b, sa, _, _ = bench.local_workload("cfg2")
    causal = b.field("CAUSAL") != 0
    chunk = b.field("KV_CHUNK")
    out = {"all": time_featurize(ctx, b, sa, 10)}
    out["prefill"] = time_featurize(ctx, b.subset(np.nonzero(causal)[0]), sa, 10)
    out["decode"] = time_featurize(ctx, b.subset(np.nonzero(~causal)[0]), sa, 10)
    out["decode_unsplit"] = time_featurize(ctx, b.subset(np.nonzero(~causal & (chunk == 0))[0]), sa, 10)
    out["decode_split"] = time_featurize(ctx, b.subset(np.nonzero(~causal & (chunk != 0))[0]), sa, 10)
    print({k: round(v, 3) for k, v in out.items()}, "configs", int(causal.sum()), int((~causal).sum()))


if __name__ == "__main__":
    main()
