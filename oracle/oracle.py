"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes loaders for
  * oracle/build/libbboracle.so  -- the CPU restatement (oracle/*.c), and
  * oracle/_ref/libbeeplan_ref.so -- the unmodified reference codec
    (reference proj/src/codec.cpp + synth.cpp, built by oracle/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this module -- never the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libbboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libbeeplan_ref.so")

_u8p = C.POINTER(C.c_uint8)


def build(quiet: bool = True) -> None:
    """Compile the oracle (and oracle/_ref where /root/reference exists)."""
    subprocess.run(["make", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _buf(b: bytes):
    return (C.c_uint8 * max(1, len(b))).from_buffer_copy(b if b else b"\0")


class OracleError(Exception):
    def __init__(self, status: int, msg: str = ""):
        super().__init__(f"status {status}: {msg}")
        self.status = status


class Oracle:
    """The CPU restatement (oracle/*.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.orc_compress_bound.restype = C.c_size_t
        L.orc_compress_bound.argtypes = [C.c_size_t]
        for name in ("orc_zlib_compress", "orc_zlib_compress_profiled", "orc_zlib_uncompress"):
            f = getattr(L, name)
            f.restype = C.c_int
            f.argtypes = [_u8p, C.c_size_t, _u8p, C.c_size_t, C.POINTER(C.c_size_t)]
        L.orc_match_profile.argtypes = [_u8p, C.c_size_t, C.POINTER(C.c_uint32)]
        L.orc_hash_prev.argtypes = [_u8p, C.c_size_t, C.POINTER(C.c_uint16)]
        L.orc_adler32.restype = C.c_uint32
        L.orc_adler32.argtypes = [C.c_uint32, _u8p, C.c_size_t]
        L.orc_container_bound.restype = C.c_size_t
        L.orc_container_bound.argtypes = [C.c_size_t, C.c_int, C.c_int]
        L.orc_compress.restype = C.c_int
        L.orc_compress.argtypes = [_u8p, C.c_size_t, C.c_int, C.c_int, _u8p, C.c_size_t,
                                   C.POINTER(C.c_size_t)]
        L.orc_decompress.restype = C.c_int
        L.orc_decompress.argtypes = [_u8p, C.c_size_t, _u8p, C.c_size_t, C.POINTER(C.c_size_t)]
        L.orc_entropy.restype = C.c_double
        L.orc_entropy.argtypes = [_u8p, C.c_size_t]
        L.orc_synth_fp16.argtypes = [C.c_size_t, C.c_uint64, _u8p]
        L.orc_synth_bf16.argtypes = [C.c_size_t, C.c_uint64, _u8p]
        self.lib = L

    # zlib level-6 stream of one lane
    def zlib_compress(self, data: bytes, profiled: bool = False) -> bytes:
        cap = self.lib.orc_compress_bound(len(data))
        out = (C.c_uint8 * cap)()
        n = C.c_size_t()
        f = self.lib.orc_zlib_compress_profiled if profiled else self.lib.orc_zlib_compress
        rc = f(_buf(data), len(data), out, cap, C.byref(n))
        if rc:
            raise OracleError(rc, "compress")
        return bytes(out[: n.value])

    def zlib_uncompress(self, blob: bytes, expected: int) -> bytes:
        out = (C.c_uint8 * max(1, expected))()
        n = C.c_size_t()
        rc = self.lib.orc_zlib_uncompress(_buf(blob), len(blob), out, expected, C.byref(n))
        if rc:
            raise OracleError(4, f"zlib rc {rc}")
        return bytes(out[: n.value])

    def match_profile(self, data: bytes):
        import numpy as np
        prof = np.zeros(2 * max(1, len(data)), dtype=np.uint32)
        self.lib.orc_match_profile(_buf(data), len(data),
                                   prof.ctypes.data_as(C.POINTER(C.c_uint32)))
        return prof[: 2 * len(data)].reshape(-1, 2)

    def hash_prev(self, data: bytes):
        import numpy as np
        pd = np.zeros(max(1, len(data)), dtype=np.uint16)
        self.lib.orc_hash_prev(_buf(data), len(data), pd.ctypes.data_as(C.POINTER(C.c_uint16)))
        return pd[: len(data)]

    def adler32(self, data: bytes, start: int = 1) -> int:
        return self.lib.orc_adler32(start, _buf(data), len(data))

    def compress(self, stream: bytes, backend: int = 1, split: bool = True) -> bytes:
        cap = self.lib.orc_container_bound(len(stream), backend, int(split))
        out = (C.c_uint8 * max(cap, 64))()
        n = C.c_size_t()
        rc = self.lib.orc_compress(_buf(stream), len(stream), backend, int(split), out,
                                   max(cap, 64), C.byref(n))
        if rc:
            raise OracleError(rc, "compress")
        return bytes(out[: n.value])

    def decompress(self, container: bytes) -> bytes:
        n = C.c_size_t()
        src = _buf(container)
        rc = self.lib.orc_decompress(src, len(container), None, 0, C.byref(n))
        if rc:
            raise OracleError(rc, "decompress")
        out = (C.c_uint8 * max(1, n.value))()
        rc = self.lib.orc_decompress(src, len(container), out, n.value, C.byref(n))
        if rc:
            raise OracleError(rc, "decompress")
        return bytes(out[: n.value])

    def entropy(self, data: bytes) -> float:
        return self.lib.orc_entropy(_buf(data), len(data))

    def synth_fp16(self, elements: int, seed: int) -> bytes:
        out = (C.c_uint8 * max(1, 2 * elements))()
        self.lib.orc_synth_fp16(elements, seed, out)
        return bytes(out[: 2 * elements])

    def synth_bf16(self, elements: int, seed: int) -> bytes:
        out = (C.c_uint8 * max(1, 2 * elements))()
        self.lib.orc_synth_bf16(elements, seed, out)
        return bytes(out[: 2 * elements])


class Reference:
    """The unmodified reference codec (oracle/_ref/libbeeplan_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        pp = C.POINTER(_u8p)
        L.bbref_compress.restype = C.c_int
        L.bbref_compress.argtypes = [_u8p, C.c_size_t, C.c_int, C.c_int, pp, C.POINTER(C.c_size_t)]
        L.bbref_decompress.restype = C.c_int
        L.bbref_decompress.argtypes = [_u8p, C.c_size_t, pp, C.POINTER(C.c_size_t)]
        L.bbref_backend_encode.restype = C.c_int
        L.bbref_backend_encode.argtypes = [C.c_int, _u8p, C.c_size_t, pp, C.POINTER(C.c_size_t)]
        L.bbref_backend_decode.restype = C.c_int
        L.bbref_backend_decode.argtypes = [C.c_int, _u8p, C.c_size_t, C.c_size_t, pp,
                                           C.POINTER(C.c_size_t)]
        L.bbref_synth_fp16.restype = C.c_int
        L.bbref_synth_fp16.argtypes = [C.c_size_t, C.c_ulonglong, _u8p]
        L.bbref_entropy.restype = C.c_double
        L.bbref_entropy.argtypes = [_u8p, C.c_size_t]
        L.bbref_last_error.restype = C.c_char_p
        L.bbref_free.argtypes = [C.c_void_p]
        L.bbref_pack_encode.restype = C.c_int
        L.bbref_pack_encode.argtypes = [C.c_void_p, C.POINTER(C.c_size_t), C.POINTER(C.c_uint),
                                        C.c_uint, pp, C.POINTER(C.c_size_t)]
        L.bbref_decode_packed.restype = C.c_int
        L.bbref_decode_packed.argtypes = [_u8p, C.c_size_t, C.c_size_t, pp, C.POINTER(C.c_size_t)]
        L.bbref_unpack_check.restype = C.c_int
        L.bbref_unpack_check.argtypes = [C.POINTER(C.c_uint), C.c_size_t, C.c_size_t, C.c_size_t]
        self.lib = L

    def _take(self, rc, p, n):
        if rc:
            raise OracleError(rc, self.lib.bbref_last_error().decode())
        b = C.string_at(p, n.value) if n.value else b""
        self.lib.bbref_free(p)
        return b

    def compress(self, stream: bytes, backend: int = 1, split: bool = True) -> bytes:
        p, n = _u8p(), C.c_size_t()
        rc = self.lib.bbref_compress(_buf(stream), len(stream), backend, int(split), C.byref(p),
                                     C.byref(n))
        return self._take(rc, p, n)

    def decompress(self, container: bytes) -> bytes:
        p, n = _u8p(), C.c_size_t()
        rc = self.lib.bbref_decompress(_buf(container), len(container), C.byref(p), C.byref(n))
        return self._take(rc, p, n)

    def encode(self, backend: int, lane: bytes) -> bytes:
        p, n = _u8p(), C.c_size_t()
        rc = self.lib.bbref_backend_encode(backend, _buf(lane), len(lane), C.byref(p), C.byref(n))
        return self._take(rc, p, n)

    def decode(self, backend: int, blob: bytes, expected: int) -> bytes:
        p, n = _u8p(), C.c_size_t()
        rc = self.lib.bbref_backend_decode(backend, _buf(blob), len(blob), expected, C.byref(p),
                                           C.byref(n))
        return self._take(rc, p, n)

    def synth_fp16(self, elements: int, seed: int) -> bytes:
        out = (C.c_uint8 * max(1, 2 * elements))()
        rc = self.lib.bbref_synth_fp16(elements, seed, out)
        if rc:
            raise OracleError(rc)
        return bytes(out[: 2 * elements])

    def entropy(self, data: bytes) -> float:
        return self.lib.bbref_entropy(_buf(data), len(data))

    def pack_encode(self, per_request) -> bytes:
        """encode_packed(pack(per_request)); per_request = list of lists of float sequences."""
        import numpy as np
        vecs = [np.asarray(v, dtype=np.float32).reshape(-1) for st in per_request for v in st]
        flat = np.concatenate(vecs) if vecs else np.zeros(1, np.float32)
        dims = (C.c_size_t * max(1, len(vecs)))(*[v.size for v in vecs])
        counts = (C.c_uint * max(1, len(per_request)))(*[len(st) for st in per_request])
        p, n = _u8p(), C.c_size_t()
        rc = self.lib.bbref_pack_encode(flat.ctypes.data, dims, counts, len(per_request), C.byref(p),
                                        C.byref(n))
        return self._take(rc, p, n)

    def decode_packed(self, data: bytes, hidden_dim: int) -> bytes:
        """encode_packed(decode_packed(data, hidden_dim)) (raises OracleError 8 = CorruptOffsets)."""
        p, n = _u8p(), C.c_size_t()
        rc = self.lib.bbref_decode_packed(_buf(data), len(data), hidden_dim, C.byref(p), C.byref(n))
        return self._take(rc, p, n)

    def unpack_check(self, offsets, hidden_dim: int, payload_floats: int) -> int:
        arr = (C.c_uint * max(1, len(offsets)))(*offsets)
        return self.lib.bbref_unpack_check(arr, len(offsets), hidden_dim, payload_floats)
