"""sp_featurize on a subset of cfg2 (for ncu captures): --part prefill|decode_split|decode_unsplit|all
    python tools/subset_featurize.py --part decode_split
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import paper_2601_14910_b200 as sp  # noqa: E402
import bench  # noqa: E402
from tail_probe import time_featurize  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--part", default="decode_split")
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
ctx = sp.Context(0)
b, sa, _, _ = bench.local_workload("cfg2")
causal = b.field("CAUSAL") != 0
chunk = b.field("KV_CHUNK")
sel = {"prefill": causal, "decode_split": ~causal & (chunk != 0), "decode_unsplit": ~causal & (chunk == 0),
       "all": np.ones_like(causal)}[args.part]
print(args.part, time_featurize(ctx, b.subset(np.nonzero(sel)[0]), sa, args.reps))
