"""Phase timeline of the tcgen05 predictor (debug build with -DSP_PRED_TRACE).

    SYNPERF_LIB=variants/lib_trace.so python tools/pred_trace.py
Prints the median cycles between the stamps of CTA 0's two epilogue slots and
its MMA issuer (see PTRACE in predict_tcgen05.cu).
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_14910_b200 as sp  # noqa: E402
from paper_2601_14910_b200 import _abi  # noqa: E402
from workloads import models  # noqa: E402

ctx = sp.Context(0)
b, sa, (g0, g1), _ = bench.local_workload("cfg2", 0.25)
sh = ctx.load_gpu_specs(sa)
m = ctx.load_model(models.random_mlp(b.family, 42), "fp16")
db = sp.DeviceBatch.from_host(b, "cuda:0")
n = (g1 - g0) * b.n_configs
f = sp.Features.empty(b.family, n, "cuda:0")
lat = torch.empty(n, dtype=torch.float32, device="cuda:0")
ctx.featurize(db, sh, f)
for _ in range(3):
    ctx.predict(m, f, lat)
torch.cuda.synchronize()
allbuf = np.zeros(3 * 64 * 16 + 16 * 64 * 16, np.int64)
_abi.lib.sp_debug_pred_trace.argtypes = [C.c_void_p]
print("rc", _abi.lib.sp_debug_pred_trace(allbuf.ctypes.data))
buf = allbuf[:3 * 64 * 16].reshape(3, 64, 16)
wbuf = allbuf[3 * 64 * 16:].reshape(16, 64, 16)
names = ["start", "-", "D1 ready", "A2 arrived", "D2 ready", "A3 arrived", "D3 ready", "end"]
t = buf[2, 2:60, 1].astype(np.float64)
print("period (L1s0 issue to next):", np.median(np.diff(t)))
# a window of iterations, all roles on a common clock
ev = []
for it in (9, 10, 11):
    for role, nm in ((0, "s0"), (1, "s1")):
        for i, name in enumerate(names):
            if name != "-":
                ev.append((buf[role, it, i], f"{nm} {name} [{it}]"))
    mma = ["iter", "L1s0 issued", "L1s1 issued", "L2s0 issued", "L2s1 issued", "L3s0 issued", "L3s1 issued", "-",
           "X(s0) full", "X(s1) full"]
    for i, name in enumerate(mma):
        if buf[2, it, i] and name != "-" and "full" not in name:
            ev.append((buf[2, it, i], f"    MMA {name} [{it}]"))
ev.sort()
t0 = ev[0][0]
it = 10
print("timeline (cycles):")
for t, name in ev:
    print(f"  {t - t0:7d}  {name}")
print("per-warp (rows: warp = slot*8 + half*4 + quadrant), cycles from t0:")
print("      " + " ".join(f"{n[:10]:>10}" for n in names))
for w in range(16):
    print(f"w{w:2d}   " + " ".join(f"{wbuf[w, it, i] - t0:10d}" for i in range(8)))
out = os.environ.get("PRED_TRACE_OUT")
if out:  # raw stamps for offline analysis
    np.savez(out, buf=buf, wbuf=wbuf)
