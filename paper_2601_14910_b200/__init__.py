"""B200-native batched SynPerf predictor (arXiv 2601.14910).

Public API (thin binding over include/synperf.h / libsynperf.so):
    Context, Specs, Model, DeviceBatch, Features, cross, pair_list    (kernel-level prediction)
    E2EPlan, CommModel, E2EResult                                     (E2E serving composition, §V-D)
The feature stage, the MLP predictor, the workload expansion and the
composition run in hand-written sm_100a CUDA kernels; there is no CPU fallback.
"""
from ._abi import EXPORTED, LIB_PATH, lib  # noqa: F401  (raises if the library is missing)
from .api import (FLT_NAMES, INT_NAMES, CommModel, Context, DeviceBatch, E2EPlan,  # noqa: F401
                  E2EResult, Features, Model, Specs, SynPerfError, cross, features_to_host,
                  Trainer, pair_list)

__all__ = ["Context", "Specs", "Model", "DeviceBatch", "Features", "cross", "pair_list",
           "E2EPlan", "CommModel", "E2EResult", "Trainer", "SynPerfError", "features_to_host",
           "INT_NAMES", "FLT_NAMES"]
