"""B200-native AutoFreeze freezing hot path (arXiv 2102.01386).

`FreezingModule` (af_layer_norms / af_update_and_decide) and `ActivationCache`
(af_cache_put / af_cache_get) bind the C ABI in include/af.h; the work runs in
the sm_100a kernels of libautofreeze.so.  Importing fails if the library has
not been built (no CPU fallback).
"""
from ._lib import (AF_ACC_DELTA, AF_ACC_STEP_SUMSQ, AF_DEC_DRY_RUN, AF_DEC_FIRST_INTERVAL, AF_DEC_NEAR_TIE,
                   AF_DEC_NONFINITE, AF_DEC_SKIPPED_FEW, AF_DT_BF16, AF_DT_F32, AF_SEG_HEAD, AF_SEG_POOL,
                   AF_SEG_PRE, AfError, LIB_PATH, lib)
from .api import (ActivationCache, FreezingModule, bootstrap_nccl_id, calibrate_forward_seconds,
                  calibrate_read_seconds, calibrate_should_cache, should_cache)

__all__ = ["FreezingModule", "ActivationCache", "should_cache", "bootstrap_nccl_id", "calibrate_read_seconds",
           "calibrate_forward_seconds", "calibrate_should_cache", "AfError", "LIB_PATH", "lib",
           "AF_SEG_PRE", "AF_SEG_POOL", "AF_SEG_HEAD", "AF_DT_F32", "AF_DT_BF16", "AF_ACC_DELTA",
           "AF_ACC_STEP_SUMSQ", "AF_DEC_FIRST_INTERVAL", "AF_DEC_SKIPPED_FEW", "AF_DEC_NEAR_TIE",
           "AF_DEC_NONFINITE", "AF_DEC_DRY_RUN"]
__version__ = "0.1.0"
