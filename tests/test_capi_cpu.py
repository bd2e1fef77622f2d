"""CPU-side checks of the C-ABI library: it loads without a GPU and exports
every symbol include/bbcodec.h declares (no compute calls here)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "bbcodec.h")).read()
    return sorted(set(re.findall(r"BB_API\s+[\w\s\*]*?\b(bb_\w+)\s*\(", hdr)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("bb_compress", "bb_decompress", "bb_split", "bb_merge", "bb_histogram256",
              "bb_compress_batch", "bb_decompress_batch", "bb_backend_encode", "bb_backend_decode"):
        assert s in syms


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2604_21072_b200 import _lib
    L = _lib.load()
    for s in declared_symbols():
        assert hasattr(L, s), s
    assert L.bb_version().startswith(b"bbcodec-b200")
    # pure host helpers are callable without a GPU
    assert L.bb_compress_bound(1000, 0, 1) == 31 + 1000
    assert L.bb_compress_bound(1000, 1, 0) == 31 + 1000 + (1000 >> 12) + (1000 >> 14) + (1000 >> 25) + 13


def test_no_gpu_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        return
    from paper_2604_21072_b200 import _lib
    L = _lib.load()
    h = ctypes.c_void_p()
    assert L.bb_ctx_create(ctypes.byref(h), 0) != 0  # no silent CPU path
