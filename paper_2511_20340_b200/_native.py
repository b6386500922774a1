"""ctypes declarations for libspecformer.so (include/specformer.h). Argument marshalling only.

The library is built in-tree by `paper_2511_20340_b200/build.py`; importing this module loads it
and fails loudly if it is missing -- there is no fallback implementation.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libspecformer.so")

SF_OK, SF_ERR_ARG, SF_ERR_SHAPE, SF_ERR_CAPACITY, SF_ERR_STATE, SF_ERR_CUDA, SF_ERR_NCCL, SF_ERR_NONFINITE, \
    SF_ERR_UNSUPPORTED = range(9)
STATUS_NAMES = ["SF_OK", "SF_ERR_ARG", "SF_ERR_SHAPE", "SF_ERR_CAPACITY", "SF_ERR_STATE", "SF_ERR_CUDA",
                "SF_ERR_NCCL", "SF_ERR_NONFINITE", "SF_ERR_UNSUPPORTED"]
SF_FP32, SF_BF16 = 0, 1
SF_FLAG_CUDA_GRAPH = 1 << 0
SF_FLAG_DRAFT_CAUSAL = 1 << 1
SF_FLAG_NO_LOGITS = 1 << 2
SF_FLAG_NO_POS_FFN = 1 << 3
SF_FLAG_DRAFT_PREFIX = 1 << 4
SF_FLAG_PAGE_POOL = 1 << 5
SF_FLAG_TP_F32_REDUCE = 1 << 6


class sf_config(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("d_ff", C.c_int32), ("vocab", C.c_int32),
                ("draft_len", C.c_int32), ("max_batch", C.c_int32), ("max_seq", C.c_int32),
                ("kv_block", C.c_int32), ("rope_theta", C.c_float), ("rms_eps", C.c_float),
                ("dtype", C.c_int32), ("tp_size", C.c_int32), ("tp_rank", C.c_int32), ("flags", C.c_uint64),
                ("draft_blocks", C.c_int32), ("pool_pages", C.c_int32)]


class sf_tensor_desc(C.Structure):
    _fields_ = [("name", C.c_char * 64), ("ndim", C.c_int32), ("shape", C.c_int64 * 4),
                ("offset_bytes", C.c_int64), ("dtype", C.c_int32), ("layout", C.c_int32)]


# every symbol include/specformer.h declares: (name, restype, argtypes)
_P = C.c_void_p
_I32P = C.POINTER(C.c_int32)
SIGNATURES = [
    ("sf_weight_table", C.c_int, [C.POINTER(sf_config), C.POINTER(sf_tensor_desc), C.c_int]),
    ("sf_weights_bytes", C.c_int64, [C.POINTER(sf_config)]),
    ("sf_workspace_bytes", C.c_int64, [C.POINTER(sf_config)]),
    ("specformer_init", C.c_int, [C.POINTER(sf_config), _P, _P, _P, C.POINTER(_P)]),
    ("specformer_prefill", C.c_int, [_P, _P, C.c_int32, C.c_int32, _P]),
    ("specformer_draft_step", C.c_int, [_P, _P, _P]),
    ("specformer_verify_step", C.c_int, [_P, _P, _P, _P]),
    ("specformer_accept_commit", C.c_int, [_P, _P, _P, _P]),
    ("specformer_release", C.c_int, [_P, C.c_int32]),
    ("specformer_prefill_slot", C.c_int, [_P, C.c_int32, _P, C.c_int32, _P]),
    ("specformer_decode_steps", C.c_int, [_P, C.c_int32, _P, _P]),
    ("specformer_sync", C.c_int, [_P]),
    ("specformer_last_error", C.c_char_p, [_P]),
    ("specformer_destroy", None, [_P]),
    ("specformer_kernel_launches", C.c_int64, [_P]),
    ("specformer_build_info", C.c_char_p, []),
    ("sf_debug_set_block_table", C.c_int, [_P, _P, C.c_int32, C.c_int32]),
    ("sf_debug_capture", C.c_int, [_P, C.c_int32, _P, C.POINTER(C.c_int64)]),
    ("sf_debug_force_drafts", C.c_int, [_P, _P, C.c_int32, _P]),
    ("sf_set_forced_drafts", C.c_int, [_P, _P, C.c_int32, _P, C.c_int32]),
    ("sf_profile", C.c_int, [_P, C.c_int32]),
    ("sf_profile_read", C.c_int, [_P, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                  C.POINTER(C.c_double)]),
    ("sf_pack_matrix", C.c_int, [C.c_int32, _P, _P, C.c_int64, C.c_int64, _P]),
    ("sf_test_gemm", C.c_int, [C.c_int32, _P, _P, _P, C.c_int32, C.c_int32, C.c_int32, _P]),
    ("sf_bench_gemm", C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P]),
    ("sf_debug_gemm_trace", C.c_int32, [_P, C.c_int32]),
    ("sf_debug_ktrace", C.c_int32, [_P, C.c_int32]),
    ("sf_debug_ktrace_enable", C.c_int32, [C.c_int32]),
    ("sf_nccl_unique_id", C.c_int32, [_P]),
    ("sf_nccl_attach", C.c_int, [_P, _P, C.c_int32, C.c_int32]),
    ("sf_local_group_create", _P, [C.c_int32]),
    ("sf_local_group_destroy", None, [_P]),
    ("sf_local_group_attach", C.c_int, [_P, _P, C.c_int32]),
    ("sf_tp_xch_handle", C.c_int, [_P, _P]),
    ("sf_tp_xch_attach", C.c_int, [_P, _P]),
    ("sf_local_group_xch_attach", C.c_int, [_P, _P]),
]


def load(path: str = LIB_PATH):
    if not os.path.exists(path):
        raise RuntimeError(f"libspecformer.so not built at {path}: run `python -m paper_2511_20340_b200.build` "
                           "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = load()
    return _lib


class SpecFormerError(RuntimeError):
    def __init__(self, status, msg=""):
        self.status = status
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")
