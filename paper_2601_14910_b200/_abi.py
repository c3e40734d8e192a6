"""ctypes mirror of include/synperf.h (argument marshalling only).

Loads the in-tree libsynperf.so.  There is no fallback: if the library is
missing or cannot be loaded, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

# SYNPERF_LIB: an alternative in-tree build of the same library (kernel A/B experiments)
LIB_PATH = os.environ.get("SYNPERF_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsynperf.so")

# sp_status
SP_OK, SP_E_ARG, SP_E_DATA, SP_E_INTERNAL, SP_E_UNSUPPORTED = 0, 1, 2, 3, 4
STATUS_NAMES = {0: "SP_OK", 1: "SP_E_ARG", 2: "SP_E_DATA", 3: "SP_E_INTERNAL", 4: "SP_E_UNSUPPORTED"}
# sp_family
SP_GEMM, SP_ATTENTION, SP_FUSED_MOE, SP_RMSNORM, SP_SILU_MUL, SP_SCALED_MM, SP_GEMM_SPLITK = range(7)
NFIELDS = {SP_GEMM: 11, SP_ATTENTION: 12, SP_FUSED_MOE: 14, SP_RMSNORM: 6, SP_SILU_MUL: 6,
           SP_SCALED_MM: 11, SP_GEMM_SPLITK: 12}
# sp_pairing_kind
SP_PAIRS_CROSS, SP_PAIRS_LIST = 0, 1
# sp_precision
SP_MLP_FP32, SP_MLP_BF16, SP_MLP_FP16 = 0, 1, 2
PRECISIONS = {"fp32": SP_MLP_FP32, "bf16": SP_MLP_BF16, "fp16": SP_MLP_FP16}
SP_STRICT = 1
SP_FEAT_CLAMPED = 1
# sp_scheduler
SP_SCHED_RR, SP_SCHED_GREEDY, SP_SCHED_MINHEAP = 0, 1, 2
SCHEDULERS = {"rr": SP_SCHED_RR, "greedy": SP_SCHED_GREEDY, "minheap": SP_SCHED_MINHEAP}


class sp_gpu_spec(C.Structure):
    _fields_ = [
        ("name", C.c_char * 32),
        ("cc_major", C.c_int32), ("cc_minor", C.c_int32), ("num_sms", C.c_int32),
        ("th_tensor_bf16", C.c_int32), ("th_tensor_fp16", C.c_int32), ("th_tensor_fp8", C.c_int32),
        ("th_fma", C.c_int32), ("th_xu", C.c_int32), ("smem_bw_bytes_per_clk", C.c_int32),
        ("smem_per_sm_bytes", C.c_int32), ("regfile_per_sm_bytes", C.c_int32),
        ("max_warps_per_sm", C.c_int32), ("max_ctas_per_sm", C.c_int32), ("reserved_", C.c_int32),
        ("sm_clock_mhz", C.c_double), ("bw_global_gbps", C.c_double), ("bw_l2_gbps", C.c_double),
    ]


assert C.sizeof(sp_gpu_spec) == 112


class sp_config_batch(C.Structure):
    _fields_ = [
        ("family", C.c_int32), ("n_fields", C.c_int32), ("n_configs", C.c_int64),
        ("field_ld", C.c_int64), ("fields", C.c_void_p), ("ragged", C.c_void_p),
        ("ragged_off", C.c_void_p), ("n_ragged", C.c_int64),
    ]


class sp_pairing(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("spec_begin", C.c_int32), ("spec_end", C.c_int32),
        ("reserved_", C.c_int32), ("n_pairs", C.c_int64), ("cfg_idx", C.c_void_p),
        ("spec_idx", C.c_void_p),
    ]


class sp_features(C.Structure):
    _fields_ = [
        ("family", C.c_int32), ("reserved_", C.c_int32), ("n_pairs", C.c_int64), ("ld", C.c_int64),
        ("ints", C.c_void_p), ("flts", C.c_void_p), ("status", C.c_void_p),
    ]


class sp_serving_model(C.Structure):
    _fields_ = [(k, C.c_int32) for k in ("n_layers", "hidden", "n_heads", "n_kv_heads", "head_dim",
                                         "intermediate", "vocab", "tp", "pp", "dtype")]


class sp_e2e_info(C.Structure):
    _fields_ = [("n_traces", C.c_int32), ("max_batch", C.c_int32), ("n_requests", C.c_int64),
                ("n_steps", C.c_int64), ("n_ragged", C.c_int64), ("n_slots", C.c_int64),
                ("n_configs", C.c_int64 * 5)]


class sp_comm_desc(C.Structure):
    _fields_ = [("n_specs", C.c_int32), ("n_points", C.c_int32), ("bytes", C.c_void_p),
                ("allreduce_us", C.c_void_p), ("sendrecv_us", C.c_void_p)]


class sp_e2e_latencies(C.Structure):
    _fields_ = [("gemm", C.c_void_p), ("attention", C.c_void_p), ("rmsnorm", C.c_void_p),
                ("silu_mul", C.c_void_p)]


SP_E2E_NCAT = 5
E2E_CATEGORIES = ["gemm", "attention", "rmsnorm", "silu_mul", "comm"]


# sp_loss
SP_LOSS_MAPE, SP_LOSS_PINBALL = 0, 1
LOSSES = {"mape": SP_LOSS_MAPE, "pinball": SP_LOSS_PINBALL}


class sp_train_config(C.Structure):
    _fields_ = [("loss", C.c_int32), ("quantile", C.c_float), ("lr", C.c_float),
                ("weight_decay", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float),
                ("adam_eps", C.c_float), ("dropout", C.c_float), ("bn_momentum", C.c_float),
                ("max_batch", C.c_int32), ("seed", C.c_uint64)]


assert C.sizeof(sp_train_config) == 48


class sp_kernel_stat(C.Structure):
    _fields_ = [("kernel", C.c_char_p), ("launches", C.c_int64), ("total_ms", C.c_double)]


MLP_ARRAYS = ["mu", "sigma", "w1", "b1", "g1", "be1", "m1", "v1", "w2", "b2", "g2", "be2", "m2",
              "v2", "w3", "b3", "g3", "be3", "m3", "v3", "w4"]


class sp_mlp_desc(C.Structure):
    _fields_ = [("family", C.c_int32), ("n_in", C.c_int32), ("precision", C.c_int32),
                ("reserved_", C.c_int32)] + [(k, C.c_void_p) for k in MLP_ARRAYS] + [
        ("b4", C.c_float), ("bn_eps", C.c_float)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libsynperf.so not found at {LIB_PATH}; build it with "
            "`python paper_2601_14910_b200/build.py` or `python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, u32 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32
    sig = {
        "sp_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
        "sp_destroy": (None, [vp]),
        "sp_last_error": (C.c_char_p, [vp]),
        "sp_version": (C.c_char_p, []),
        "sp_device_sms": (i32, [vp]),
        "sp_load_gpu_specs": (C.c_int, [vp, vp, i32, u32, C.POINTER(vp)]),
        "sp_free_specs": (None, [vp]),
        "sp_specs_count": (i32, [vp]),
        "sp_load_model": (C.c_int, [vp, vp, C.POINTER(vp)]),
        "sp_free_model": (None, [vp]),
        "sp_featurize": (C.c_int, [vp, vp, vp, vp, vp, vp]),
        "sp_featurize_sched": (C.c_int, [vp, vp, vp, vp, i32, vp, vp]),
        "sp_featurize_ex": (C.c_int, [vp, vp, vp, vp, i32, u32, vp, vp]),
        "sp_predict": (C.c_int, [vp, vp, vp, vp, vp, vp]),
        "sp_featurize_predict": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        "sp_prepare": (C.c_int, [vp, i32, i64, vp, i32, i32]),
        "sp_predict_host": (C.c_int, [vp, C.POINTER(sp_config_batch), vp, i32, i32, vp, vp, vp, i32, vp]),
        "sp_perf_gap": (C.c_int, [vp, vp, vp, vp, vp, i64, i32, i32, C.c_float, C.c_float, vp, vp, vp, vp]),
        "sp_set_profiling": (C.c_int, [vp, i32]),
        "sp_profile_read": (i32, [vp, C.POINTER(sp_kernel_stat), i32, i32]),
        "sp_e2e_plan_create": (C.c_int, [vp, vp, i32, vp, vp, vp, vp, C.POINTER(vp)]),
        "sp_e2e_plan_update": (C.c_int, [vp, i32, vp, vp, vp, vp]),
        "sp_e2e_plan_expand": (C.c_int, [vp, vp]),
        "sp_free_e2e_plan": (None, [vp]),
        "sp_e2e_plan_info": (C.c_int, [vp, C.POINTER(sp_e2e_info)]),
        "sp_e2e_plan_batch": (C.c_int, [vp, i32, C.POINTER(sp_config_batch)]),
        "sp_load_comm_model": (C.c_int, [vp, C.POINTER(sp_comm_desc), C.POINTER(vp)]),
        "sp_free_comm_model": (None, [vp]),
        "sp_e2e_compose": (C.c_int, [vp, vp, i32, i32, vp, C.POINTER(sp_e2e_latencies), vp, vp, vp, vp]),
        "sp_train_create": (C.c_int, [vp, vp, C.POINTER(sp_train_config), C.POINTER(vp)]),
        "sp_train_destroy": (None, [vp]),
        "sp_train_step": (C.c_int, [vp, vp, vp, vp, i64, vp, vp]),
        "sp_train_eval": (C.c_int, [vp, vp, vp, vp, i64, vp, vp]),
        "sp_train_export_count": (i64, [vp]),
        "sp_train_export": (C.c_int, [vp, vp, vp]),
        "sp_train_export_grads": (C.c_int, [vp, vp, vp]),
        "sp_fit_norm": (C.c_int, [vp, vp, vp, i64, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


lib = _load()

EXPORTED = ["sp_create", "sp_destroy", "sp_last_error", "sp_version", "sp_device_sms",
            "sp_load_gpu_specs", "sp_free_specs", "sp_specs_count", "sp_load_model",
            "sp_free_model", "sp_featurize", "sp_featurize_sched", "sp_featurize_ex", "sp_predict", "sp_featurize_predict", "sp_predict_host", "sp_prepare", "sp_perf_gap", "sp_set_profiling", "sp_profile_read",
            "sp_e2e_plan_create", "sp_e2e_plan_update", "sp_e2e_plan_expand", "sp_free_e2e_plan", "sp_e2e_plan_info",
            "sp_e2e_plan_batch", "sp_load_comm_model", "sp_free_comm_model", "sp_e2e_compose",
            "sp_train_create", "sp_train_destroy", "sp_train_step", "sp_train_eval", "sp_train_export_count",
            "sp_train_export", "sp_train_export_grads", "sp_fit_norm"]
