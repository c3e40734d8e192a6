import time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench, paper_2601_14910_b200 as sp
from workloads import models
ctx = sp.Context(0)
for w in ("cfg3", "cfg2"):
    b, sa, (g0, g1), _ = bench.local_workload(w, 1.0)
    sh = ctx.load_gpu_specs(sa)
    m = ctx.load_model(models.random_mlp(b.family, 42), "fp16")
    class H: pass
    h = H(); h.family = b.family
    h.fields = torch.from_numpy(b.fields).pin_memory()
    h.ragged = torch.from_numpy(b.ragged).pin_memory() if b.ragged is not None else None
    h.ragged_off = torch.from_numpy(b.ragged_off).pin_memory() if b.ragged_off is not None else None
    n = (g1 - g0) * b.n_configs
    out = torch.empty(n, dtype=torch.float32).pin_memory()
    for ch in (1, 4, 8):
        for _ in range(2): ctx.predict_host(h, sh, m, (g0, g1), out=out, chunks=ch)
        torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(3): ctx.predict_host(h, sh, m, (g0, g1), out=out, chunks=ch)
        torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 3
        print(w, "chunks", ch, "ms", dt * 1e3, "pairs/s %.3g" % (n / dt), flush=True)
    # raw H2D bandwidth
    nb = h.fields.numel() * 4 + (h.ragged.numel() * 4 if h.ragged is not None else 0)
    d = torch.empty(h.fields.shape, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(5): d.copy_(h.fields, non_blocking=True)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 5
    print(w, "H2D fields GB/s", h.fields.numel() * 4 / dt / 1e9, "config bytes", nb, flush=True)
    import cProfile, pstats
    pr = cProfile.Profile(); pr.enable()
    ctx.predict_host(h, sh, m, (g0, g1), out=out, chunks=4); torch.cuda.synchronize()
    pr.disable(); pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
