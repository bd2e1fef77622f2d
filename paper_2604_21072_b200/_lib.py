"""ctypes binding of the sm_100a codec library (include/bbcodec.h).

The CUDA library is the only compute path: if ``libbbcodec.so`` is missing or
no GPU is visible, every call raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbbcodec.so")

BB_OK, BB_ODD_LENGTH, BB_LANE_MISMATCH, BB_BACKEND_UNKNOWN = 0, 1, 2, 3
BB_CORRUPT_CONTAINER, BB_ERROR, BB_CUDA_ERROR, BB_INVALID_ARG = 4, 5, 6, 7
BB_CORRUPT_OFFSETS, BB_DIM_MISMATCH = 8, 9

EXPORTS = [
    "bb_last_error", "bb_version", "bb_ctx_create", "bb_ctx_destroy", "bb_split", "bb_merge",
    "bb_histogram256", "bb_compress_bound", "bb_compress", "bb_decompress", "bb_compress_batch",
    "bb_decompress_batch", "bb_backend_bound", "bb_backend_encode", "bb_backend_decode",
    "bb_compress_host", "bb_decompress_host", "bb_backend_encode_host", "bb_backend_decode_host",
    "bb_split_host", "bb_merge_host", "bb_histogram256_host", "bb_kernel_launches",
    "bb_stage_timing", "bb_stage_report", "bb_packed_bound", "bb_pack_sd", "bb_unpack_sd",
    "bb_gather_pages", "bb_enable_peer_access", "bb_ipc_export", "bb_ipc_import", "bb_ipc_close",
    "bb_copy_h2d", "bb_equal",
]

_u8p = C.c_void_p
_sz = C.c_size_t
_szp = C.POINTER(C.c_size_t)

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load the library (no CUDA work is done at load time)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: run __graft_entry__.build() "
                              "(the codec has no CPU fallback)")
        L = C.CDLL(path)
        L.bb_last_error.restype = C.c_char_p
        L.bb_version.restype = C.c_char_p
        L.bb_ctx_create.argtypes = [C.POINTER(C.c_void_p), C.c_int]
        L.bb_ctx_destroy.argtypes = [C.c_void_p]
        L.bb_split.argtypes = [_u8p, _sz, _u8p, _u8p, C.c_void_p]
        L.bb_merge.argtypes = [_u8p, _u8p, _sz, _u8p, C.c_void_p]
        L.bb_histogram256.argtypes = [_u8p, _sz, _u8p, C.c_void_p]
        L.bb_equal.argtypes = [C.c_void_p, _u8p, _u8p, _sz, C.POINTER(C.c_int), C.c_void_p]
        L.bb_compress_bound.restype = _sz
        L.bb_compress_bound.argtypes = [_sz, C.c_int, C.c_int]
        L.bb_backend_bound.restype = _sz
        L.bb_backend_bound.argtypes = [C.c_int, _sz]
        L.bb_compress.argtypes = [C.c_void_p, _u8p, _sz, C.c_int, C.c_int, _u8p, _sz, _szp, C.c_void_p]
        L.bb_decompress.argtypes = [C.c_void_p, _u8p, _sz, _u8p, _sz, _szp, C.c_void_p]
        L.bb_compress_batch.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_void_p), _szp, C.c_int,
                                        C.c_int, C.POINTER(C.c_void_p), _szp, _szp,
                                        C.POINTER(C.c_int), C.c_void_p]
        L.bb_decompress_batch.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_void_p), _szp,
                                          C.POINTER(C.c_void_p), _szp, _szp, C.POINTER(C.c_int),
                                          C.c_void_p]
        L.bb_backend_encode.argtypes = [C.c_void_p, C.c_int, _u8p, _sz, _u8p, _sz, _szp, C.c_void_p]
        L.bb_backend_decode.argtypes = [C.c_void_p, C.c_int, _u8p, _sz, _sz, _u8p, C.c_void_p]
        L.bb_compress_host.argtypes = [C.c_void_p, C.c_char_p, _sz, C.c_int, C.c_int, _u8p, _sz, _szp]
        L.bb_decompress_host.argtypes = [C.c_void_p, C.c_char_p, _sz, _u8p, _sz, _szp]
        L.bb_backend_encode_host.argtypes = [C.c_void_p, C.c_int, C.c_char_p, _sz, _u8p, _sz, _szp]
        L.bb_backend_decode_host.argtypes = [C.c_void_p, C.c_int, C.c_char_p, _sz, _sz, _u8p]
        L.bb_split_host.argtypes = [C.c_void_p, C.c_char_p, _sz, _u8p, _u8p]
        L.bb_merge_host.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, _sz, _u8p]
        L.bb_histogram256_host.argtypes = [C.c_void_p, C.c_char_p, _sz, _u8p]
        L.bb_packed_bound.restype = _sz
        L.bb_packed_bound.argtypes = [_sz, _sz, C.c_uint32]
        L.bb_pack_sd.argtypes = [_u8p, _sz, _sz, _u8p, C.POINTER(C.c_uint32), C.c_uint32, _u8p, _sz,
                                 _szp, C.c_void_p]
        L.bb_unpack_sd.argtypes = [_u8p, _sz, _sz, C.POINTER(C.c_uint32), _sz, C.POINTER(C.c_uint32),
                                   _szp, C.c_void_p]
        L.bb_gather_pages.argtypes = [_u8p, _sz, _sz, _u8p, C.c_uint32, _u8p, C.c_void_p]
        L.bb_enable_peer_access.argtypes = [C.c_int, C.c_int]
        L.bb_ipc_export.argtypes = [_u8p, C.c_void_p, _szp]
        L.bb_ipc_import.argtypes = [C.c_int, C.c_void_p, _sz, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]
        L.bb_ipc_close.argtypes = [C.c_void_p]
        L.bb_copy_h2d.argtypes = [C.c_void_p, C.c_void_p, _sz, C.c_void_p]
        L.bb_kernel_launches.restype = C.c_uint64
        L.bb_stage_timing.argtypes = [C.c_int]
        L.bb_stage_report.restype = C.c_char_p
        L.bb_stage_report.argtypes = [C.c_int]
        _lib = L
        return L


def last_error() -> str:
    return load().bb_last_error().decode(errors="replace")


_tls = threading.local()


def context(device: int = 0) -> C.c_void_p:
    """Per-thread, per-device bb_ctx (the C-ABI's contexts are not thread-safe)."""
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        L = load()
        h = C.c_void_p()
        rc = L.bb_ctx_create(C.byref(h), device)
        if rc:
            raise RuntimeError(f"bb_ctx_create failed ({rc}): {last_error()}")
        ctxs[device] = h
    return ctxs[device]


def kernel_launches() -> int:
    return int(load().bb_kernel_launches())


def k4_positions() -> tuple:
    """Cumulative lane positions profiled by K4's classic walk and by K4G (roofline coverage)."""
    out = (C.c_uint64 * 2)()
    load().bb_debug_k4_positions(out)
    return int(out[0]), int(out[1])


def stage_timing(enable: bool) -> None:
    load().bb_stage_timing(1 if enable else 0)


def stage_report(reset: bool = False) -> dict:
    import json
    return json.loads(load().bb_stage_report(1 if reset else 0).decode())
