"""ctypes wrapper of the fp64 CPU oracle (oracle/synperf_oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs are the only permitted callers.  The
product package (paper_2601_14910_b200/) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "synperf_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

CLAMPED = 1
# scheduler modes (flags bits 4..5): cyclic RR is 0
SCHED_GREEDY = 1 << 4   # hardware RR with greedy retirement
SCHED_MINHEAP = 2 << 4  # persistent kernel, software MinHeap

N_INTS, N_FLTS = 11, 12
INT_NAMES = ["n_tasks", "occupancy", "waves", "tot_T", "tot_F", "tot_X", "max_T", "max_F",
             "max_X", "bytes", "bytes_max"]
FLT_NAMES = ["cg_T", "cg_F", "cg_X", "cs_T", "cs_F", "cs_X", "glob_gpu", "l2_gpu", "glob_sm",
             "l2_sm", "smem_sm", "t_theory_us"]


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, -O2, no fast-math, OpenMP)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fopenmp", "-shared", "-fPIC",
                               "-o", LIB, SRC, "-lm"])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        L.orc_featurize.restype = C.c_int
        L.orc_featurize.argtypes = [C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                    C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_int]
        L.orc_predict.restype = C.c_int
        L.orc_predict.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        L.orc_task_list.restype = C.c_int64
        L.orc_task_list.argtypes = [C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                    C.c_int, C.c_int64, C.c_void_p, C.c_int64]
        L.orc_schedule_rr.restype = None
        L.orc_schedule_rr.argtypes = [C.c_int64, C.c_int64, C.c_void_p]
        L.orc_schedule_greedy.restype = None
        L.orc_schedule_greedy.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p]
        L.orc_schedule_minheap.restype = None
        L.orc_schedule_minheap.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                                           C.c_void_p]
        L.orc_mlp_input.restype = C.c_int
        L.orc_mlp_input.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_count.restype = C.c_int
        L.orc_count.argtypes = [C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                                C.c_void_p]
        L.orc_num_threads.restype = C.c_int
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


@dataclass
class OracleFeatures:
    ints: np.ndarray  # int64 [11, n_pairs]
    flts: np.ndarray  # float64 [12, n_pairs]
    status: np.ndarray  # uint8 [n_pairs]


def cross_pairs(n_configs: int, spec_range) -> tuple[np.ndarray, np.ndarray]:
    """Spec-major cross product: pair p = (g - g0) * C + c."""
    g0, g1 = spec_range
    g = np.repeat(np.arange(g0, g1, dtype=np.int64), n_configs)
    c = np.tile(np.arange(n_configs, dtype=np.int64), g1 - g0)
    return c, g


def featurize(batch, specs: np.ndarray, cfg_idx=None, spec_idx=None, flags: int = 0,
              nthreads: int = 0) -> OracleFeatures:
    """Oracle O1..O7 for the pairs (cfg_idx[p], spec_idx[p]); default: full
    spec-major cross product of all specs x all configs."""
    if cfg_idx is None:
        cfg_idx, spec_idx = cross_pairs(batch.n_configs, (0, len(specs)))
    cfg_idx = np.ascontiguousarray(cfg_idx, dtype=np.int64)
    spec_idx = np.ascontiguousarray(spec_idx, dtype=np.int64)
    n = len(cfg_idx)
    fields = np.ascontiguousarray(batch.fields, dtype=np.int32)
    ragged = None if batch.ragged is None else np.ascontiguousarray(batch.ragged, dtype=np.int32)
    roff = None if batch.ragged_off is None else np.ascontiguousarray(batch.ragged_off, np.int64)
    specs = np.ascontiguousarray(specs)
    ints = np.zeros((N_INTS, n), np.int64)
    flts = np.zeros((N_FLTS, n), np.float64)
    status = np.zeros(n, np.uint8)
    rc = lib().orc_featurize(batch.family, batch.n_configs, _ptr(fields), fields.shape[1],
                             _ptr(ragged), _ptr(roff), _ptr(specs), len(specs), n, _ptr(cfg_idx),
                             _ptr(spec_idx), flags, _ptr(ints), _ptr(flts), _ptr(status),
                             nthreads)
    if rc != 0:
        raise ValueError(f"oracle rejected family {batch.family}")
    return OracleFeatures(ints, flts, status)


def task_list(batch, c: int = 0, flags: int = 0, cap: int = 1 << 20) -> np.ndarray:
    """Per-task demands [T, 4] = (Tensor ops, FMA ops, XU ops, load bytes) in task order."""
    fields = np.ascontiguousarray(batch.fields, dtype=np.int32)
    rag = None
    if batch.ragged_off is not None and batch.ragged_off[c] >= 0:
        rag = np.ascontiguousarray(batch.ragged[batch.ragged_off[c]:], dtype=np.int32)
    out = np.zeros((cap, 4), np.int64)
    n = lib().orc_task_list(batch.family, _ptr(fields), fields.shape[1], c, _ptr(rag), flags,
                            0, _ptr(out), cap)
    if n < 0:
        raise ValueError(f"config rejected with status {-n}")
    return out[:n].copy()


def count(batch, c: int = 0) -> tuple[int, int, int]:
    """(status, T, U) of config c: its task count and, for attention, the
    per-kv-head sum of kv_eff/BKV, as the oracle's domain check counts them
    (no 32-bit limit; saturated counts read as 2^63 - 1)."""
    fields = np.ascontiguousarray(batch.fields, dtype=np.int32)
    rag = None
    if batch.ragged_off is not None and batch.ragged_off[c] >= 0:
        rag = np.ascontiguousarray(batch.ragged[batch.ragged_off[c]:], dtype=np.int32)
    T = C.c_int64(0)
    U = C.c_int64(0)
    st = lib().orc_count(batch.family, _ptr(fields), fields.shape[1], c, _ptr(rag), C.byref(T), C.byref(U))
    return int(st), int(T.value), int(U.value)


def schedule_rr(n_tasks: int, n_sm: int) -> np.ndarray:
    out = np.zeros(n_tasks, np.int64)
    lib().orc_schedule_rr(n_tasks, n_sm, _ptr(out))
    return out


def schedule_greedy(costs, n_sm: int, occ: int) -> np.ndarray:
    """sm_of[t] under the GREEDY scheduler for explicit integer task costs."""
    c = np.ascontiguousarray(costs, dtype=np.int64)
    out = np.zeros(len(c), np.int64)
    lib().orc_schedule_greedy(_ptr(c), len(c), n_sm, occ, _ptr(out))
    return out


def schedule_minheap(costs, n_sm: int, occ: int) -> tuple[np.ndarray, np.ndarray]:
    """(worker_of[t], sm_of[t]) under the MINHEAP scheduler for explicit costs."""
    c = np.ascontiguousarray(costs, dtype=np.int64)
    w = np.zeros(len(c), np.int64)
    out = np.zeros(len(c), np.int64)
    lib().orc_schedule_minheap(_ptr(c), len(c), n_sm, occ, _ptr(w), _ptr(out))
    return w, out


class _Mlp(C.Structure):
    _fields_ = [("family", C.c_int32), ("n_in", C.c_int32), ("precision", C.c_int32),
                ("pad_", C.c_int32)] + [
        (k, C.c_void_p) for k in ["mu", "sigma", "w1", "b1", "g1", "be1", "m1", "v1",
                                  "w2", "b2", "g2", "be2", "m2", "v2",
                                  "w3", "b3", "g3", "be3", "m3", "v3", "w4"]
    ] + [("b4", C.c_float), ("bn_eps", C.c_float)]


def _mlp_struct(model: dict):
    keep = {}
    st = _Mlp()
    st.family = int(model["family"])
    st.n_in = int(model["n_in"])
    for k in ["mu", "sigma", "w1", "b1", "g1", "be1", "m1", "v1", "w2", "b2", "g2", "be2",
              "m2", "v2", "w3", "b3", "g3", "be3", "m3", "v3", "w4"]:
        a = np.ascontiguousarray(model[k], dtype=np.float32)
        keep[k] = a
        setattr(st, k, a.ctypes.data)
    st.b4 = float(model["b4"])
    st.bn_eps = float(model["bn_eps"])
    return st, keep


def predict(model: dict, feats: OracleFeatures, nthreads: int = 0):
    """Oracle O8..O11: returns (latency_us, efficiency, logit), fp64."""
    st, keep = _mlp_struct(model)
    n = feats.status.shape[0]
    lat = np.zeros(n, np.float64)
    eff = np.zeros(n, np.float64)
    z = np.zeros(n, np.float64)
    ints = np.ascontiguousarray(feats.ints)
    flts = np.ascontiguousarray(feats.flts)
    stt = np.ascontiguousarray(feats.status)
    lib().orc_predict(C.byref(st), n, _ptr(ints), _ptr(flts), _ptr(stt), _ptr(lat), _ptr(eff),
                      _ptr(z), nthreads)
    del keep
    return lat, eff, z


def mlp_input(model: dict, ints_col: np.ndarray, flts_col: np.ndarray) -> np.ndarray:
    """Normalised MLP input vector (O8+O9) of one pair."""
    st, keep = _mlp_struct(model)
    pi = np.ascontiguousarray(ints_col, dtype=np.int64)
    pf = np.ascontiguousarray(flts_col, dtype=np.float64)
    out = np.zeros(16, np.float64)
    n = lib().orc_mlp_input(C.byref(st), _ptr(pi), _ptr(pf), _ptr(out))
    del keep
    return out[:n]


def _round16(a: np.ndarray, kind: str) -> np.ndarray:
    """Round fp64 values to bf16 or fp16, round-to-nearest-even, back to fp64."""
    if kind == "fp16":
        return np.asarray(a, np.float64).astype(np.float16).astype(np.float64)
    u = np.asarray(a, np.float64).astype(np.float32).view(np.uint32)  # fp64 -> fp32 (RNE), then fp32 -> bf16 (RNE)
    r = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000)
    return r.view(np.float32).astype(np.float64)


def predict_emulated(model: dict, feats: OracleFeatures, kind: str = "bf16", idx=None):
    """O12 --emulate-bf16: the O10-O11 MLP with every weight matrix
    and each layer's input rounded to 16 bits (bf16 or fp16, RNE), accumulation
    and BatchNorm in fp64.  Isolates operand rounding from accumulation order when
    diagnosing the 16-bit GPU predictor.  Returns latency_us for pairs idx
    (default all); NaN for pairs with status != 0."""
    idx = np.arange(feats.status.shape[0]) if idx is None else np.asarray(idx)
    x = np.stack([mlp_input(model, feats.ints[:, p], feats.flts[:, p]) for p in idx])
    eps = float(model.get("bn_eps", 1e-5))
    h = _round16(x, kind)
    for l in (1, 2, 3):
        a = h @ _round16(np.asarray(model[f"w{l}"], np.float64), kind).T + np.asarray(model[f"b{l}"], np.float64)
        r = np.maximum(a, 0.0)
        y = (np.asarray(model[f"g{l}"], np.float64) * (r - np.asarray(model[f"m{l}"], np.float64))
             / np.sqrt(np.asarray(model[f"v{l}"], np.float64) + eps) + np.asarray(model[f"be{l}"], np.float64))
        h = _round16(y, kind) if l < 3 else y  # layer 3 feeds the fp32 output layer
    z = h @ np.asarray(model["w4"], np.float64) + float(model["b4"])
    e = 1.0 / (1.0 + np.exp(-z))
    lat = feats.flts[11][idx] / e
    return np.where(feats.status[idx] == 0, lat, np.nan)


def num_threads() -> int:
    return int(lib().orc_num_threads())
