"""Thin Python binding over the C-ABI (include/synperf.h).

Argument marshalling only: torch supplies device memory and streams; every
step of the prediction path runs in libsynperf.so's CUDA kernels.  Names
follow the C entry points (sp_featurize -> Context.featurize, ...).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from ._abi import lib

N_INTS, N_FLTS = 11, 12
INT_NAMES = ["n_tasks", "occupancy", "waves", "tot_T", "tot_F", "tot_X", "max_T", "max_F",
             "max_X", "bytes", "bytes_max"]
FLT_NAMES = ["cg_T", "cg_F", "cg_X", "cs_T", "cs_F", "cs_X", "glob_gpu", "l2_gpu", "glob_sm",
             "l2_sm", "smem_sm", "t_theory_us"]


class SynPerfError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_abi.STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _stream_ptr(stream) -> int | None:
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) or None


@dataclass
class DeviceBatch:
    """Device-resident configs of one family (the C sp_config_batch)."""

    family: int
    fields: torch.Tensor  # int32 [n_fields, n_configs]
    ragged: torch.Tensor | None
    ragged_off: torch.Tensor | None

    @property
    def n_configs(self) -> int:
        return int(self.fields.shape[1])

    @staticmethod
    def from_host(batch, device, non_blocking: bool = False) -> "DeviceBatch":
        """From any object with .family, .fields (int32 [F, C]), .ragged, .ragged_off."""
        dev = torch.device(device)

        def up(a, dt):
            if a is None:
                return None
            t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
            return t.to(device=dev, dtype=dt, non_blocking=non_blocking).contiguous()

        return DeviceBatch(int(batch.family), up(batch.fields, torch.int32),
                           up(batch.ragged, torch.int32), up(batch.ragged_off, torch.int64))

    def slice(self, c0: int, c1: int) -> "DeviceBatch":
        """Configs [c0, c1) as a view (field rows keep their stride; the ragged
        data is shared, its offsets are absolute)."""
        return DeviceBatch(self.family, self.fields[:, c0:c1], self.ragged,
                           None if self.ragged_off is None else self.ragged_off[c0:c1])

    def c_struct(self) -> _abi.sp_config_batch:
        s = _abi.sp_config_batch()
        s.family = self.family
        s.n_fields = int(self.fields.shape[0])
        s.n_configs = self.n_configs
        s.field_ld = int(self.fields.stride(0)) if self.n_configs > 0 else 0
        s.fields = self.fields.data_ptr() if self.n_configs > 0 else None
        if self.ragged is not None and self.ragged.numel() > 0:
            s.ragged = self.ragged.data_ptr()
            s.n_ragged = self.ragged.numel()
        if self.ragged_off is not None and self.ragged_off.numel() > 0:
            s.ragged_off = self.ragged_off.data_ptr()
        return s


@dataclass
class Features:
    """Caller-owned device feature record (the C sp_features), SoA."""

    family: int
    ints: torch.Tensor  # int64 [11, ld]
    flts: torch.Tensor  # fp32 [12, ld]
    status: torch.Tensor  # uint8 [n_pairs]
    n_pairs: int

    @staticmethod
    def empty(family: int, n_pairs: int, device) -> "Features":
        dev = torch.device(device)
        return Features(family, torch.empty((N_INTS, max(n_pairs, 1)), dtype=torch.int64, device=dev),
                        torch.empty((N_FLTS, max(n_pairs, 1)), dtype=torch.float32, device=dev),
                        torch.empty(max(n_pairs, 1), dtype=torch.uint8, device=dev), n_pairs)

    def view(self, start: int, n: int) -> "Features":
        """Sub-range [start, start+n) sharing storage (the C struct uses ld = full width)."""
        return Features(self.family, self.ints[:, start:], self.flts[:, start:],
                        self.status[start:], n)

    def c_struct(self) -> _abi.sp_features:
        s = _abi.sp_features()
        s.family = self.family
        s.n_pairs = self.n_pairs
        s.ld = int(self.ints.stride(0))
        assert int(self.flts.stride(0)) == s.ld, "ints and flts must share a leading dimension"
        s.ints = self.ints.data_ptr()
        s.flts = self.flts.data_ptr()
        s.status = self.status.data_ptr()
        return s


def cross(spec_begin: int, spec_end: int) -> _abi.sp_pairing:
    p = _abi.sp_pairing()
    p.kind = _abi.SP_PAIRS_CROSS
    p.spec_begin, p.spec_end = int(spec_begin), int(spec_end)
    return p


def pair_list(cfg_idx: torch.Tensor, spec_idx: torch.Tensor) -> _abi.sp_pairing:
    assert cfg_idx.dtype == torch.int64 and spec_idx.dtype == torch.int32
    assert cfg_idx.is_contiguous() and spec_idx.is_contiguous()
    p = _abi.sp_pairing()
    p.kind = _abi.SP_PAIRS_LIST
    p.n_pairs = int(cfg_idx.numel())
    p.cfg_idx = cfg_idx.data_ptr() if p.n_pairs else None
    p.spec_idx = spec_idx.data_ptr() if p.n_pairs else None
    return p


class Specs:
    def __init__(self, ctx: "Context", handle: int, n: int):
        self._ctx, self._h, self.n = ctx, handle, n

    @property
    def handle(self):
        return self._h

    def __len__(self):
        return self.n

    def __del__(self):
        if getattr(self, "_h", None):
            lib.sp_free_specs(self._h)
            self._h = None


class Model:
    def __init__(self, ctx: "Context", handle: int, family: int, precision: int):
        self._ctx, self._h, self.family, self.precision = ctx, handle, family, precision

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None):
            lib.sp_free_model(self._h)
            self._h = None


class Trainer:
    """sp_trainer: on-GPU training of one per-category estimator (PAPER §V-C
    P:486-491).  Argument marshalling only; the step runs in
    csrc/train.cu."""

    PARAM_ORDER = ["w1", "b1", "g1", "be1", "w2", "b2", "g2", "be2", "w3", "b3", "g3", "be3", "w4", "b4"]

    def __init__(self, ctx: "Context", init: dict, loss: str = "mape", quantile: float = 0.8,
                 lr: float = 1e-3, weight_decay: float = 0.01, betas=(0.9, 0.999), adam_eps: float = 1e-8,
                 dropout: float = 0.1, bn_momentum: float = 0.1, max_batch: int = 256, seed: int = 0):
        self._ctx, self.family, self.n_in = ctx, int(init["family"]), int(init["n_in"])
        self.bn_eps = float(init.get("bn_eps", 1e-5))
        self.mu = np.asarray(init["mu"], np.float32).copy()
        self.sigma = np.asarray(init["sigma"], np.float32).copy()
        d, keep = ctx._mlp_desc(init, "fp32")
        c = _abi.sp_train_config()
        c.loss = _abi.LOSSES[loss]
        c.quantile, c.lr, c.weight_decay = quantile, lr, weight_decay
        c.beta1, c.beta2, c.adam_eps = betas[0], betas[1], adam_eps
        c.dropout, c.bn_momentum, c.max_batch, c.seed = dropout, bn_momentum, int(max_batch), int(seed)
        h = C.c_void_p()
        ctx._check(lib.sp_train_create(ctx._h, C.byref(d), C.byref(c), C.byref(h)))
        del keep
        self._h = h.value
        self.max_batch = int(max_batch)
        self.loss_dev = torch.zeros(1, dtype=torch.float32, device=ctx.torch_device)

    def __del__(self):
        if getattr(self, "_h", None):
            lib.sp_train_destroy(self._h)
            self._h = None

    def step(self, feats: "Features", measured_us: torch.Tensor, batch_idx: torch.Tensor, stream=None) -> torch.Tensor:
        """sp_train_step over pairs batch_idx (int64, device); returns the device loss scalar."""
        fs = feats.c_struct()
        self._ctx._check(lib.sp_train_step(self._h, C.byref(fs), measured_us.data_ptr(), batch_idx.data_ptr(),
                                           int(batch_idx.numel()), self.loss_dev.data_ptr(), _stream_ptr(stream)))
        return self.loss_dev

    def capture(self, feats: "Features", measured_us: torch.Tensor, batch_idx: torch.Tensor) -> "torch.cuda.CUDAGraph":
        """CUDA graph of one sp_train_step over the fixed device buffer batch_idx
        (refill it in place between replays).  The step counter, dropout masks and
        AdamW bias corrections live on the device, so each replay is the next
        step.  Capture launches nothing; kernel accounting must be off."""
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fs = feats.c_struct()
            self._ctx._check(lib.sp_train_step(self._h, C.byref(fs), measured_us.data_ptr(), batch_idx.data_ptr(),
                                               int(batch_idx.numel()), self.loss_dev.data_ptr(),
                                               _stream_ptr(torch.cuda.current_stream())))
        return g

    def eval_loss(self, feats: "Features", measured_us: torch.Tensor, idx: torch.Tensor, stream=None) -> torch.Tensor:
        out = torch.empty(1, dtype=torch.float32, device=self._ctx.torch_device)
        fs = feats.c_struct()
        self._ctx._check(lib.sp_train_eval(self._h, C.byref(fs), measured_us.data_ptr(), idx.data_ptr(),
                                           int(idx.numel()), out.data_ptr(), _stream_ptr(stream)))
        return out

    def export(self, stream=None) -> dict:
        """Current weights + running statistics as a model dict (sp_load_model's layout)."""
        n = int(lib.sp_train_export_count(self._h))
        buf = np.empty(n, np.float32)
        self._ctx._check(lib.sp_train_export(self._h, buf.ctypes.data, _stream_ptr(stream)))
        m = {"family": self.family, "n_in": self.n_in, "bn_eps": np.float32(self.bn_eps),
             "mu": self.mu.copy(), "sigma": self.sigma.copy()}
        m.update(self._split(buf))
        o = n - 2 * (256 + 128 + 64)  # running statistics follow the P parameters
        m["b4"] = np.float32(m["b4"][0])
        for l, width in zip((1, 2, 3), (256, 128, 64)):
            m[f"m{l}"] = buf[o:o + width].copy()
            m[f"v{l}"] = buf[o + width:o + 2 * width].copy()
            o += 2 * width
        return m

    def _split(self, buf: np.ndarray) -> dict:
        shapes = {"w1": (256, self.n_in), "w2": (128, 256), "w3": (64, 128), "w4": (64,), "b4": (1,)}
        out, o = {}, 0
        for k in self.PARAM_ORDER:
            shp = shapes[k] if k in shapes else ({"1": 256, "2": 128, "3": 64}[k[-1]],)
            cnt = int(np.prod(shp))
            out[k] = buf[o:o + cnt].reshape(shp).copy()
            o += cnt
        return out

    def export_grads(self, stream=None) -> dict:
        """Gradients of the last step, per parameter (sp_train_export_grads)."""
        n = int(lib.sp_train_export_count(self._h)) - 2 * (256 + 128 + 64)
        buf = np.empty(n, np.float32)
        self._ctx._check(lib.sp_train_export_grads(self._h, buf.ctypes.data, _stream_ptr(stream)))
        return self._split(buf)

    def fit(self, feats: "Features", measured_us: torch.Tensor, train_idx: torch.Tensor, val_idx: torch.Tensor,
            max_epochs: int = 100, patience: int = 20, batch: int | None = None, seed: int = 0) -> dict:
        """Early-stopped training loop ("Early stopping ... monitoring validation loss"):
        shuffled minibatches (seeded permutation of train_idx on the device), one eval
        loss per epoch, best-validation snapshot returned with the loss history."""
        bs = batch or self.max_batch
        g = torch.Generator(device=self._ctx.torch_device)
        g.manual_seed(seed)
        best, best_m, bad, hist = float("inf"), None, 0, []
        n = int(train_idx.numel())
        for _ in range(max_epochs):
            perm = train_idx[torch.randperm(n, generator=g, device=train_idx.device)]
            for i in range(0, n - bs + 1, bs):
                self.step(feats, measured_us, perm[i:i + bs])
            v = float(self.eval_loss(feats, measured_us, val_idx).item())
            hist.append(v)
            if v < best:
                best, best_m, bad = v, self.export(), 0
            else:
                bad += 1
                if bad > patience:
                    break
        return {"model": best_m, "best_val_loss": best, "val_history": hist}


class CommModel:
    """sp_comm_model: per-spec All-Reduce / Send-Recv calibration tables."""

    def __init__(self, ctx: "Context", handle: int, n_specs: int):
        self._ctx, self._h, self.n_specs = ctx, handle, n_specs

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None):
            lib.sp_free_comm_model(self._h)
            self._h = None


class PlanBatch:
    """A config batch owned by an E2EPlan (device pointers into the plan)."""

    def __init__(self, s: _abi.sp_config_batch):
        self._s = s
        self.family = int(s.family)

    @property
    def n_configs(self) -> int:
        return int(self._s.n_configs)

    def c_struct(self) -> _abi.sp_config_batch:
        return self._s


class E2EPlan:
    """sp_e2e_plan: the Workload Generator's invocation plan of a set of request
    traces for one serving model, expanded on the GPU."""

    FAMILIES = (_abi.SP_GEMM, _abi.SP_ATTENTION, _abi.SP_RMSNORM, _abi.SP_SILU_MUL)

    def __init__(self, ctx: "Context", handle: int, model: dict):
        self._ctx, self._h, self.model = ctx, handle, dict(model)

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None):
            lib.sp_free_e2e_plan(self._h)
            self._h = None

    def info(self) -> dict:
        inf = _abi.sp_e2e_info()
        self._ctx._check(lib.sp_e2e_plan_info(self._h, C.byref(inf)))
        return {"n_traces": inf.n_traces, "max_batch": inf.max_batch, "n_requests": inf.n_requests,
                "n_steps": inf.n_steps, "n_ragged": inf.n_ragged, "n_slots": inf.n_slots,
                "n_configs": {f: int(inf.n_configs[f]) for f in range(5)}}

    def batch(self, family: int) -> PlanBatch:
        s = _abi.sp_config_batch()
        self._ctx._check(lib.sp_e2e_plan_batch(self._h, int(family), C.byref(s)))
        return PlanBatch(s)

    def expand(self, stream=None) -> "E2EPlan":
        """Re-run the expansion kernels on the resident requests (sp_e2e_plan_expand)."""
        self._ctx._check(lib.sp_e2e_plan_expand(self._h, _stream_ptr(stream)))
        return self

    def update(self, traces, stream=None) -> "E2EPlan":
        off, ins, outs = _trace_arrays(traces)
        self._ctx._check(lib.sp_e2e_plan_update(self._h, len(off) - 1, off.ctypes.data, ins.ctypes.data,
                                                outs.ctypes.data, _stream_ptr(stream)))
        return self


def _trace_arrays(traces):
    off = np.ascontiguousarray(traces.req_off, dtype=np.int64)
    ins = np.ascontiguousarray(traces.input_len, dtype=np.int32)
    outs = np.ascontiguousarray(traces.output_len, dtype=np.int32)
    return off, ins, outs


@dataclass
class E2EResult:
    """Device outputs of Context.predict_e2e for specs [g0, g1)."""

    step_us: torch.Tensor | None   # fp32 [G, n_steps]
    trace_us: torch.Tensor         # fp64 [G, n_traces]
    trace_cat: torch.Tensor        # fp64 [G, n_traces, 5] (gemm, attention, rmsnorm, silu_mul, comm)
    latency: dict                  # family -> fp32 [G * n_configs] per-kernel predictions
    n_pairs: int                   # (config, spec) pairs featurised and predicted


class Context:
    """sp_ctx on one CUDA device."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        st = lib.sp_create(int(device), C.byref(h))
        if st != _abi.SP_OK:
            raise SynPerfError(st, lib.sp_last_error(None).decode())
        self._h = h.value
        self.device = int(device)
        self.torch_device = torch.device("cuda", self.device)

    def __del__(self):
        if getattr(self, "_h", None):
            lib.sp_destroy(self._h)
            self._h = None

    @property
    def num_sms(self) -> int:
        return int(lib.sp_device_sms(self._h))

    def last_error(self) -> str:
        return lib.sp_last_error(self._h).decode()

    def _check(self, st):
        if st != _abi.SP_OK:
            raise SynPerfError(st, self.last_error())

    # -- kernel accounting (measurement)
    def set_profiling(self, enable: bool) -> None:
        """Bracket every kernel launch of this context with CUDA events (sp_set_profiling)."""
        self._check(lib.sp_set_profiling(self._h, 1 if enable else 0))

    def profile_read(self, reset: bool = True) -> dict:
        """{kernel: (launches, device ms summed)} since the last reset (sp_profile_read)."""
        buf = (_abi.sp_kernel_stat * 32)()
        n = lib.sp_profile_read(self._h, buf, 32, 1 if reset else 0)
        if n < 0:
            raise SynPerfError(_abi.SP_E_INTERNAL, self.last_error())
        return {buf[i].kernel.decode(): (int(buf[i].launches), float(buf[i].total_ms)) for i in range(min(n, 32))}

    # -- a1
    def load_gpu_specs(self, specs: np.ndarray, strict: bool = False) -> Specs:
        arr = np.ascontiguousarray(specs)
        assert arr.dtype.itemsize == C.sizeof(_abi.sp_gpu_spec)
        h = C.c_void_p()
        self._check(lib.sp_load_gpu_specs(self._h, arr.ctypes.data, len(arr),
                                          _abi.SP_STRICT if strict else 0, C.byref(h)))
        return Specs(self, h.value, len(arr))

    # -- estimator
    def _mlp_desc(self, model: dict, precision: str):
        d = _abi.sp_mlp_desc()
        d.family = int(model["family"])
        d.n_in = int(model["n_in"])
        d.precision = _abi.PRECISIONS[precision]
        keep = []
        for k in _abi.MLP_ARRAYS:
            a = np.ascontiguousarray(model[k], dtype=np.float32)
            keep.append(a)
            setattr(d, k, a.ctypes.data)
        d.b4 = float(model["b4"])
        d.bn_eps = float(model.get("bn_eps", 1e-5))
        return d, keep

    def trainer(self, init: dict, **cfg) -> Trainer:
        """sp_train_create: on-GPU estimator training from the initial weights `init`."""
        return Trainer(self, init, **cfg)

    def fit_norm(self, feats: "Features", idx: torch.Tensor, stream=None):
        """sp_fit_norm: (mu, sigma) fp32 [n_in] of ln(1+v) over pairs idx (R17, T7)."""
        n_in = 11 if feats.family in (_abi.SP_GEMM, _abi.SP_FUSED_MOE, _abi.SP_SCALED_MM,
                                      _abi.SP_GEMM_SPLITK) else 15
        mu, sg = np.empty(n_in, np.float32), np.empty(n_in, np.float32)
        fs = feats.c_struct()
        self._check(lib.sp_fit_norm(self._h, C.byref(fs), idx.data_ptr(), int(idx.numel()), mu.ctypes.data,
                                    sg.ctypes.data, _stream_ptr(stream)))
        return mu, sg

    def load_model(self, model: dict, precision: str = "fp16") -> Model:
        """precision: "fp16" (tcgen05 tensor-core path) or "fp32" (CUDA cores); "bf16" is
        refused by the library (SP_E_UNSUPPORTED: it misses the 1e-2 latency bar)."""
        d = _abi.sp_mlp_desc()
        d.family = int(model["family"])
        d.n_in = int(model["n_in"])
        d.precision = _abi.PRECISIONS[precision]
        keep = []
        for k in _abi.MLP_ARRAYS:
            a = np.ascontiguousarray(model[k], dtype=np.float32)
            keep.append(a)
            setattr(d, k, a.ctypes.data)
        d.b4 = float(model["b4"])
        d.bn_eps = float(model.get("bn_eps", 1e-5))
        h = C.c_void_p()
        self._check(lib.sp_load_model(self._h, C.byref(d), C.byref(h)))
        del keep
        return Model(self, h.value, d.family, d.precision)

    # -- feature stage (a2..a9)
    def featurize(self, batch: DeviceBatch, specs: Specs, out: Features, pairs=None,
                  stream=None, scheduler: str = "rr", clamped: bool = False) -> Features:
        """sp_featurize (scheduler "rr"), sp_featurize_sched ("greedy", "minheap"), or
        sp_featurize_ex with SP_FEAT_CLAMPED (clamped edge tiles: GEMM, fused MoE, attention)."""
        if pairs is None:
            pairs = cross(0, len(specs))
        cb = batch.c_struct()
        fs = out.c_struct()
        if clamped:
            self._check(lib.sp_featurize_ex(self._h, C.byref(cb), specs.handle, C.byref(pairs),
                                            _abi.SCHEDULERS[scheduler], _abi.SP_FEAT_CLAMPED, C.byref(fs),
                                            _stream_ptr(stream)))
        elif scheduler == "rr":
            self._check(lib.sp_featurize(self._h, C.byref(cb), specs.handle, C.byref(pairs),
                                         C.byref(fs), _stream_ptr(stream)))
        else:
            self._check(lib.sp_featurize_sched(self._h, C.byref(cb), specs.handle, C.byref(pairs),
                                               _abi.SCHEDULERS[scheduler], C.byref(fs),
                                               _stream_ptr(stream)))
        return out

    # -- predictor stage (a10..a12)
    def predict(self, model: Model, feats: Features, latency: torch.Tensor,
                efficiency: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        assert latency.dtype == torch.float32 and latency.is_contiguous()
        assert latency.numel() >= feats.n_pairs
        fs = feats.c_struct()
        self._check(lib.sp_predict(self._h, model.handle, C.byref(fs), latency.data_ptr(),
                                   efficiency.data_ptr() if efficiency is not None else None,
                                   _stream_ptr(stream)))
        return latency

    def featurize_predict(self, batch: DeviceBatch, specs: Specs, model: Model, out: Features,
                          latency: torch.Tensor, efficiency: torch.Tensor | None = None, pairs=None,
                          stream=None) -> torch.Tensor:
        """sp_featurize_predict: the records of sp_featurize and the latencies of sp_predict in
        one fused pass (uniform families, CROSS, 16-bit model; otherwise the two calls)."""
        if pairs is None:
            pairs = cross(0, len(specs))
        assert latency.dtype == torch.float32 and latency.is_contiguous()
        cb = batch.c_struct()
        fs = out.c_struct()
        self._check(lib.sp_featurize_predict(self._h, C.byref(cb), specs.handle, C.byref(pairs), model.handle,
                                             C.byref(fs), latency.data_ptr(),
                                             efficiency.data_ptr() if efficiency is not None else None,
                                             _stream_ptr(stream)))
        return latency

    # -- performance-gap diagnosis (PAPER §VII-B)
    def perf_gap(self, feats: Features, eff_p80: torch.Tensor, measured_us: torch.Tensor, pairs=None,
                 n_configs: int = 0, n_specs: int = 0, n_bins: int = 100, gap_lo: float = -0.5,
                 gap_hi: float = 0.5, want_gap: bool = True, stream=None):
        """sp_perf_gap: returns (gap fp32 [n] or None, counts int64 [G, 2] = {valid,
        underperforming}, hist int64 [G, n_bins]) as device tensors."""
        if pairs is None:
            pairs = cross(0, n_specs)
        G = (pairs.spec_end - pairs.spec_begin) if pairs.kind == _abi.SP_PAIRS_CROSS else n_specs
        dev = self.torch_device
        n = feats.n_pairs
        gap = torch.empty(max(n, 1), dtype=torch.float32, device=dev) if want_gap else None
        counts = torch.empty((max(G, 1), 2), dtype=torch.int64, device=dev)
        hist = torch.empty((max(G, 1), n_bins), dtype=torch.int64, device=dev)
        fs = feats.c_struct()
        self._check(lib.sp_perf_gap(self._h, C.byref(fs), eff_p80.data_ptr(), measured_us.data_ptr(),
                                    C.byref(pairs), int(n_configs), int(n_specs), int(n_bins),
                                    float(gap_lo), float(gap_hi),
                                    gap.data_ptr() if gap is not None else None, counts.data_ptr(),
                                    hist.data_ptr(), _stream_ptr(stream)))
        return (gap[:n] if gap is not None else None), counts[:G], hist[:G]

    # -- end-to-end serving composition (PAPER §V-D; include/synperf.h sp_e2e_*)

    def load_comm_model(self, comm: dict) -> CommModel:
        """comm: {"bytes": [P], "allreduce_us": [G][P], "sendrecv_us": [G][P]} (fp64)."""
        b = np.ascontiguousarray(comm["bytes"], dtype=np.float64)
        ar = np.ascontiguousarray(comm["allreduce_us"], dtype=np.float64)
        sr = np.ascontiguousarray(comm["sendrecv_us"], dtype=np.float64)
        d = _abi.sp_comm_desc()
        d.n_specs, d.n_points = int(ar.shape[0]), int(b.shape[0])
        d.bytes, d.allreduce_us, d.sendrecv_us = b.ctypes.data, ar.ctypes.data, sr.ctypes.data
        h = C.c_void_p()
        self._check(lib.sp_load_comm_model(self._h, C.byref(d), C.byref(h)))
        return CommModel(self, h.value, d.n_specs)

    def e2e_plan(self, model: dict, traces, stream=None) -> E2EPlan:
        """model: n_layers, hidden, n_heads, n_kv_heads, head_dim, intermediate, vocab, tp, pp;
        traces: .req_off int64 [R+1], .input_len / .output_len int32 (host)."""
        m = _abi.sp_serving_model()
        for k in ("n_layers", "hidden", "n_heads", "n_kv_heads", "head_dim", "intermediate", "vocab"):
            setattr(m, k, int(model[k]))
        m.tp, m.pp, m.dtype = int(model.get("tp", 1)), int(model.get("pp", 1)), 0
        off, ins, outs = _trace_arrays(traces)
        h = C.c_void_p()
        self._check(lib.sp_e2e_plan_create(self._h, C.byref(m), len(off) - 1, off.ctypes.data,
                                           ins.ctypes.data, outs.ctypes.data, _stream_ptr(stream),
                                           C.byref(h)))
        return E2EPlan(self, h.value, model)

    def e2e_compose(self, plan: E2EPlan, spec_range, comm: CommModel | None, lat: dict,
                    step_us=None, trace_us=None, trace_cat=None, stream=None) -> None:
        """sp_e2e_compose: lat maps family -> fp32 device latencies (spec-major)."""
        L = _abi.sp_e2e_latencies()
        for f, name in ((_abi.SP_GEMM, "gemm"), (_abi.SP_ATTENTION, "attention"),
                        (_abi.SP_RMSNORM, "rmsnorm"), (_abi.SP_SILU_MUL, "silu_mul")):
            t = lat[f]
            assert t.dtype == torch.float32 and t.is_contiguous()
            setattr(L, name, t.data_ptr())

        def ptr(t, dt):
            if t is None:
                return None
            assert t.dtype == dt and t.is_contiguous()
            return t.data_ptr()

        g0, g1 = spec_range
        self._check(lib.sp_e2e_compose(self._h, plan.handle, int(g0), int(g1),
                                       comm.handle if comm is not None else None, C.byref(L),
                                       ptr(step_us, torch.float32), ptr(trace_us, torch.float64),
                                       ptr(trace_cat, torch.float64), _stream_ptr(stream)))

    def predict_e2e(self, plan: E2EPlan, specs: Specs, models: dict, comm: CommModel | None = None,
                    spec_range=None, step_latencies: bool = True, stream=None) -> E2EResult:
        """Featurise + predict every config batch of the plan on specs
        [g0, g1) (one sp_featurize + sp_predict per family) and compose the
        per-step and per-trace latencies (sp_e2e_compose).  Device in, device
        out; feature buffers are cached on the context."""
        g0, g1 = spec_range if spec_range is not None else (0, len(specs))
        G = g1 - g0
        inf = plan.info()
        dev = self.torch_device
        cache = self.__dict__.setdefault("_e2e_cache", {})
        lat = {}
        n_pairs = 0
        for f in E2EPlan.FAMILIES:
            b = plan.batch(f)
            n = G * b.n_configs
            n_pairs += n
            key = (f, max(n, 1))
            ent = cache.get(f)
            if ent is None or ent[0] < n:
                ent = (max(n, 1), Features.empty(f, max(n, 1), dev),
                       torch.empty(max(n, 1), dtype=torch.float32, device=dev))
                cache[f] = ent
            feats = ent[1]
            feats.n_pairs = n
            self.featurize_predict(b, specs, models[f], feats, ent[2], None, cross(g0, g1), stream)
            lat[f] = ent[2][:max(n, 1)]
        R, S = inf["n_traces"], inf["n_steps"]
        step = torch.empty((G, S), dtype=torch.float32, device=dev) if step_latencies else None
        tot = torch.empty((G, R), dtype=torch.float64, device=dev)
        cat = torch.empty((G, R, _abi.SP_E2E_NCAT), dtype=torch.float64, device=dev)
        self.e2e_compose(plan, (g0, g1), comm, lat, step, tot, cat, stream)
        return E2EResult(step, tot, cat, lat, n_pairs)

    def predict_e2e_host(self, model: dict, traces, specs: Specs, models: dict,
                         comm: CommModel | None = None, spec_range=None, stream=None):
        """The user-facing end-to-end call: host request traces in, host
        per-trace latencies out.  Uploads the requests (sp_e2e_plan_update on
        a cached plan), runs predict_e2e and copies back trace totals and the
        category breakdown: (trace_us [G, R], trace_cat [G, R, 5]) numpy fp64."""
        plans = self.__dict__.setdefault("_e2e_plans", {})
        key = tuple(sorted((k, int(v)) for k, v in model.items()))
        plan = plans.get(key)
        if plan is None:
            plan = plans[key] = self.e2e_plan(model, traces, stream)
        else:
            plan.update(traces, stream)
        r = self.predict_e2e(plan, specs, models, comm, spec_range, step_latencies=False, stream=stream)
        tot = torch.empty(r.trace_us.shape, dtype=torch.float64, pin_memory=True)
        cat = torch.empty(r.trace_cat.shape, dtype=torch.float64, pin_memory=True)
        tot.copy_(r.trace_us, non_blocking=True)
        cat.copy_(r.trace_cat, non_blocking=True)
        (stream or torch.cuda.current_stream(self.torch_device)).synchronize()
        return tot.numpy(), cat.numpy()

    def prepare(self, family: int, n_configs: int, specs: Specs, spec_range=None) -> None:
        """sp_prepare: build the attention plan of the spec range and grow the
        context scratch, so later calls at these sizes neither allocate nor
        synchronize (and can be captured in a CUDA graph)."""
        g0, g1 = spec_range if spec_range is not None else (0, len(specs))
        self._check(lib.sp_prepare(self._h, int(family), int(n_configs), specs.handle, g0, g1))

    # -- end-to-end: host configs in, host latencies out
    def predict_host(self, batch, specs: Specs, model: Model, spec_range=None,
                     out: np.ndarray | torch.Tensor | None = None, chunks=None,
                     stream=None) -> np.ndarray:
        """The user-facing call, sp_predict_host: host config arrays (numpy or
        torch; pinned memory gives asynchronous copies) -> pipelined H2D /
        featurize + predict / D2H inside the library -> fp32 latencies in
        spec-major order [spec][config] (a numpy view of `out`, pinned by
        default).  `chunks`: a slice count, or relative slice weights such as
        (1, 2, 3, 2); None = the library default."""
        g0, g1 = spec_range if spec_range is not None else (0, len(specs))
        fam = int(batch.family)

        def host_t(a, dt):
            if a is None:
                return None
            t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
            t = t if t.dtype == dt else t.to(dt)
            assert t.device.type == "cpu", "predict_host takes host arrays"
            return t.contiguous()

        fh = host_t(batch.fields, torch.int32)
        rh = host_t(batch.ragged, torch.int32)
        oh = host_t(batch.ragged_off, torch.int64)
        nf, C_ = int(fh.shape[0]), int(fh.shape[1])
        n = (g1 - g0) * C_
        if out is None:
            out_t = torch.empty(max(n, 1), dtype=torch.float32, pin_memory=True)
        else:
            out_t = out if isinstance(out, torch.Tensor) else torch.from_numpy(out)
        assert out_t.dtype == torch.float32 and out_t.is_contiguous() and out_t.numel() >= n
        if n == 0:
            return out_t[:0].numpy()
        cb = _abi.sp_config_batch(fam, nf, C_, C_, fh.data_ptr(),
                                  rh.data_ptr() if rh is not None and rh.numel() else None,
                                  oh.data_ptr() if oh is not None else None,
                                  rh.numel() if rh is not None else 0)
        w = None
        ns = 0
        if chunks is not None:
            if isinstance(chunks, int):
                ns = int(chunks)
            else:
                w = (C.c_float * len(chunks))(*[float(x) for x in chunks])
                ns = len(chunks)
        self._check(lib.sp_predict_host(self._h, C.byref(cb), specs.handle, g0, g1, model.handle,
                                        out_t.data_ptr(), w, ns, _stream_ptr(stream)))
        return out_t[:n].numpy()


def features_to_host(f: Features) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    n = f.n_pairs
    return (f.ints[:, :n].cpu().numpy(), f.flts[:, :n].cpu().numpy(), f.status[:n].cpu().numpy())
