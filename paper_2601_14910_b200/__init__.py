"""B200-native batched SynPerf predictor (arXiv 2601.14910).

Public API (thin binding over include/synperf.h / libsynperf.so):
    Context, Specs, Model, DeviceBatch, Features, cross, pair_list
The feature stage and the MLP predictor run in hand-written sm_100a CUDA
kernels; there is no CPU fallback.
"""
from ._abi import EXPORTED, LIB_PATH, lib  # noqa: F401  (raises if the library is missing)
from .api import (Context, DeviceBatch, Features, FLT_NAMES, INT_NAMES, Model, Specs,  # noqa: F401
                  SynPerfError, cross, features_to_host, pair_list)

__all__ = ["Context", "Specs", "Model", "DeviceBatch", "Features", "cross", "pair_list",
           "SynPerfError", "features_to_host", "INT_NAMES", "FLT_NAMES"]
