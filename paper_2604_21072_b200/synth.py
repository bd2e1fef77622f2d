"""Synthetic activations for harnesses: the C++ drop-in generator
(paper_2604_21072_b200/cpp/synth.cpp = reference synth_gaussian_fp16 semantics,
plus the frozen bf16 variant).  Host-side input generation, not the hot path."""
from __future__ import annotations

import ctypes as C
import os

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libbeeplan_b200.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise ImportError(f"{_LIB} missing: run __graft_entry__.build()")
        _lib = C.CDLL(_LIB)
        _lib.beeplan_synth_gaussian.argtypes = [C.c_size_t, C.c_uint64, C.c_int, C.c_void_p]
    return _lib


def gaussian(elements: int, seed: int, bf16: bool = False) -> bytes:
    lib = _load()
    buf = bytearray(2 * elements)
    if elements:
        cbuf = (C.c_uint8 * len(buf)).from_buffer(buf)
        lib.beeplan_synth_gaussian(elements, seed, 1 if bf16 else 0, C.addressof(cbuf))
    return bytes(buf)
