"""ctypes declarations of include/af.h (argument marshalling only).

Loads the in-tree libautofreeze.so built by `_build.py`.  There is no CPU or
PyTorch fallback: if the library is missing, importing the package fails.
"""
import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_size_t, c_uint32, c_void_p

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libautofreeze.so")

AF_MAX_SEGMENTS = 256
AF_MAX_WORLD = 64
AF_OK, AF_EINVAL, AF_ESTATE, AF_EWORKSPACE, AF_ECUDA, AF_ENCCL, AF_ENONFINITE, AF_EOWNER, AF_ERANGE = range(9)
AF_DT_F32, AF_DT_BF16 = 0, 1
AF_CACHE_OVERLAP_PREV = 0x1
AF_DEBUG_TAIL_DELAY_NS, AF_DEBUG_PEERS_ARRIVED, AF_DEBUG_UNSTAGED_TAIL, AF_DEBUG_FORCE_NCCL = 1, 2, 3, 4
AF_SEG_PRE, AF_SEG_POOL, AF_SEG_HEAD = 0, 1, 2
AF_ACC_DELTA, AF_ACC_STEP_SUMSQ = 0, 1
AF_PCT_LINEAR, AF_PCT_NEAREST_RANK = 0, 1
AF_INTERVAL_END, AF_DRY_RUN = 0x1, 0x2
AF_DEC_FIRST_INTERVAL, AF_DEC_SKIPPED_FEW, AF_DEC_NEAR_TIE, AF_DEC_NONFINITE, AF_DEC_DRY_RUN = 1, 2, 4, 8, 16
AF_DEC_EXCHANGE_TIMEOUT = 32
AF_IPC_HANDLE_BYTES = 128
AF_CACHE_IPC_HANDLE_BYTES = 256
AF_CACHE_ERR_RANGE, AF_CACHE_ERR_OWNER, AF_CACHE_ERR_IO = 1, 2, 4


class AfLayout(ctypes.Structure):
    _fields_ = [("n_segments", c_int32), ("seg_offsets", POINTER(c_int64)),
                ("seg_kinds", POINTER(c_int32)), ("grad_dtype", c_int)]


class AfConfig(ctypes.Structure):
    _fields_ = [("percentile", c_double), ("pct_method", c_int), ("acc_mode", c_int),
                ("tie_rel_eps", c_double), ("min_active", c_int32), ("rank", c_int32), ("world", c_int32),
                ("shard_active", c_int32)]


class AfDecision(ctypes.Structure):
    _fields_ = [("interval", c_int32), ("boundary_before", c_int32), ("boundary_after", c_int32),
                ("n_active", c_int32), ("threshold", c_double), ("flags", c_uint32),
                ("near_tie_seg", c_int32), ("sumsq", c_double * AF_MAX_SEGMENTS),
                ("norm", c_double * AF_MAX_SEGMENTS), ("eta", c_double * AF_MAX_SEGMENTS)]


class AfInfo(ctypes.Structure):
    _fields_ = [("n_segments", c_int32), ("n_pool", c_int32), ("rank", c_int32), ("world", c_int32),
                ("n_total", c_int64), ("shard_begin", c_int64), ("shard_end", c_int64),
                ("n_tiles", c_int32), ("tile_elems", c_int32),
                ("first_tile_of_pool", c_int32 * (AF_MAX_SEGMENTS + 1)),
                ("n_tiles_acc", c_int32), ("tile_elems_acc", c_int32),
                ("n_fin_ctas", c_int32), ("n_fin_chunks", c_int32)]


class AfAdamW(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_float), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float),
                ("eps", ctypes.c_float), ("weight_decay", ctypes.c_float), ("step", c_int32)]


class AfCacheInfo(ctypes.Structure):
    _fields_ = [("error_flags", c_uint32), ("pad", c_uint32), ("partition", c_int64), ("capacity", c_int64),
                ("n_valid", c_int64), ("n_hbm", c_int64), ("n_host", c_int64), ("n_dropped", c_int64),
                ("free_slots", c_int64), ("n_disk", c_int64)]


# name -> (restype, argtypes); every af_* symbol declared in include/af.h
SIGNATURES = {
    "af_ctx_create": (c_int, [POINTER(AfLayout), POINTER(AfConfig), POINTER(c_void_p)]),
    "af_ctx_workspace_bytes": (c_int, [c_void_p, POINTER(c_size_t), POINTER(c_size_t)]),
    "af_ctx_info": (c_int, [c_void_p, POINTER(AfInfo)]),
    "af_ctx_shard_of": (c_int, [c_void_p, c_int32, POINTER(c_int64), POINTER(c_int64)]),
    "af_ctx_bind": (c_int, [c_void_p, c_void_p, c_void_p]),
    "af_nccl_unique_id": (c_int, [c_void_p]),
    "af_ctx_set_comm": (c_int, [c_void_p, c_void_p]),
    "af_ctx_exchange_rows": (c_int, [c_void_p, POINTER(c_void_p)]),
    "af_ctx_exchange_ipc_handle": (c_int, [c_void_p, c_void_p]),
    "af_ctx_set_peers_ipc": (c_int, [c_void_p, c_void_p]),
    "af_ctx_set_peers_local": (c_int, [c_void_p, c_void_p]),
    "af_ctx_clear_peers": (c_int, [c_void_p]),
    "af_layer_norms": (c_int, [c_void_p, c_void_p, c_uint32, c_void_p]),
    "af_update_and_decide": (c_int, [c_void_p, c_uint32, c_void_p, c_void_p]),
    "af_interval_end": (c_int, [c_void_p, c_void_p, c_uint32, c_void_p, c_void_p]),
    "af_adamw_step": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, POINTER(AfAdamW), c_uint32,
                              c_void_p, c_void_p]),
    "af_ctx_set_max_ctas": (c_int, [c_void_p, c_int32]),
    "af_ctx_grad_ipc_handle": (c_int, [c_void_p, c_void_p, c_void_p]),
    "af_ctx_set_grad_peers_ipc": (c_int, [c_void_p, c_void_p]),
    "af_ctx_set_grad_peers_local": (c_int, [c_void_p, c_void_p]),
    "af_reduce_scatter_step": (c_int, [c_void_p, ctypes.c_float, c_void_p, c_uint32, c_void_p, c_void_p]),
    "af_reduce_scatter_adamw_step": (c_int, [c_void_p, ctypes.c_float, c_void_p, c_void_p, c_void_p, POINTER(AfAdamW),
                                             c_void_p, c_uint32, c_void_p, c_void_p]),
    "af_get_state": (c_int, [c_void_p, c_void_p, POINTER(c_size_t)]),
    "af_set_state": (c_int, [c_void_p, c_void_p, c_size_t]),
    "af_ctx_read_record": (c_int, [c_void_p, c_int32, POINTER(AfDecision)]),
    "af_ctx_set_debug": (c_int, [c_void_p, c_int32, c_int64]),
    "af_ctx_destroy": (c_int, [c_void_p]),
    "af_cache_create": (c_int, [c_int64, c_int64, c_int32, c_int32, POINTER(c_void_p)]),
    "af_cache_storage_bytes": (c_int, [c_void_p, POINTER(c_size_t), POINTER(c_size_t)]),
    "af_cache_bind": (c_int, [c_void_p, c_void_p, c_void_p]),
    "af_cache_put": (c_int, [c_void_p, c_void_p, c_int32, c_void_p, c_int32, c_void_p]),
    "af_cache_get": (c_int, [c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_void_p]),
    "af_cache_get_ex": (c_int, [c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_uint32, c_void_p]),
    "af_cache_status": (c_int, [c_void_p, POINTER(c_uint32), POINTER(c_int64)]),
    "af_cache_set_capacity": (c_int, [c_void_p, c_int64, c_int64]),
    "af_cache_host_bytes": (c_int, [c_void_p, POINTER(c_size_t)]),
    "af_cache_bind_host": (c_int, [c_void_p, c_void_p]),
    "af_cache_set_disk_tier": (c_int, [c_void_p, c_int64, c_int32, c_char_p]),
    "af_cache_disk_stage_bytes": (c_int, [c_void_p, POINTER(c_size_t)]),
    "af_cache_bind_disk_stage": (c_int, [c_void_p, c_void_p]),
    "af_cache_stats": (c_int, [c_void_p, POINTER(AfCacheInfo)]),
    "af_cache_exchange_ipc_handle": (c_int, [c_void_p, c_void_p]),
    "af_cache_set_peers_ipc": (c_int, [c_void_p, c_void_p]),
    "af_cache_set_peers_local": (c_int, [c_void_p, c_void_p]),
    "af_cache_put_global": (c_int, [c_void_p, c_void_p, c_int32, c_void_p, c_int32, c_void_p]),
    "af_cache_get_gemm": (c_int, [c_void_p, c_void_p, c_int32, c_int32, c_int32, c_int32, c_void_p, c_int32, c_void_p,
                                  c_void_p, c_void_p]),
    "af_cache_get_global": (c_int, [c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_void_p]),
    "af_cache_destroy": (c_int, [c_void_p]),
    "af_should_cache": (c_int, [c_int32, c_double, c_double]),
    "af_status_str": (c_char_p, [c_int]),
    "af_last_error": (c_char_p, []),
    "af_version": (c_char_p, []),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the sm_100a CUDA library first "
            "(python -m paper_2102_01386_b200._build or __graft_entry__.build()). "
            "There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class AfError(RuntimeError):
    def __init__(self, status, call):
        self.status = status
        msg = lib.af_status_str(status).decode()
        detail = (lib.af_last_error() or b"").decode()
        super().__init__(f"{call} -> {msg}: {detail}")


def check(status, call):
    if status != AF_OK:
        raise AfError(status, call)
    return status
