"""Small invocations of every hot kernel for compute-sanitizer (memcheck,
racecheck, synccheck): attention (CROSS, LIST, clamped, GREEDY), the fp16
tcgen05 predictor, the fused uniform pass (GEMM, MoE with histograms), the
host-buffer call, split-K, the E2E plan + compose, perf-gap and one training
step.  Prints OK when every call returned (errors are reported by the tool).

    compute-sanitizer --tool memcheck python tools/sanitize.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_14910_b200 as sp  # noqa: E402
from workloads import gen, models, specs  # noqa: E402


def main():
    ctx = sp.Context(0)
    sa = specs.paper_gpu_specs()
    sh = ctx.load_gpu_specs(sa)
    dev = "cuda:0"
    att = gen.gen_attention(40, 40, 3, max_bs=4, qlen_max=3000, kvlen_max=5000)
    for b in (att, gen.gen_gemm(300, 4), gen.gen_moe(300, 5), gen.gen_rowwise(gen.RMSNORM, 200, 6),
              gen.gen_gemm_splitk(200, 7), gen.gen_scaled_mm(200, 8)):
        m = ctx.load_model(models.random_mlp(b.family, 1), "fp16")
        db = sp.DeviceBatch.from_host(b, dev)
        n = len(sa) * b.n_configs
        f = sp.Features.empty(b.family, n, dev)
        lat = torch.empty(n, dtype=torch.float32, device=dev)
        ctx.featurize(db, sh, f)
        ctx.predict(m, f, lat)
        ctx.featurize_predict(db, sh, m, f, lat)
        ctx.predict_host(b, sh, m, chunks=3)
        torch.cuda.synchronize()
    # pair list, clamped, GREEDY on attention
    db = sp.DeviceBatch.from_host(att, dev)
    ci = torch.arange(att.n_configs, dtype=torch.int64, device=dev)
    si = (ci % len(sa)).to(torch.int32)
    f = sp.Features.empty(att.family, att.n_configs, dev)
    ctx.featurize(db, sh, f, sp.pair_list(ci, si))
    fc = sp.Features.empty(att.family, len(sa) * att.n_configs, dev)
    ctx.featurize(db, sh, fc, clamped=True)
    ctx.featurize(db, sh, fc, scheduler="greedy")
    torch.cuda.synchronize()
    print("OK")


if __name__ == "__main__":
    main()
