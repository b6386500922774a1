"""B200-native SpecFormer speculative-decoding hot path (arXiv 2511.20340).

Product path: libspecformer.so (hand-written sm_100a CUDA behind the C ABI in
include/specformer.h) + this thin ctypes binding. No CPU fallback: importing `Engine`
requires the built library and a CUDA device for any compute call.
"""
from .engine import Engine, EngineConfig, pack_weights, run_gemm, weight_table  # noqa: F401
from . import _native  # noqa: F401
