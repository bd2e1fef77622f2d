"""Python mirror of the reference codec API (reference proj/include/beeplan/codec.hpp).

Same names, argument meaning and error behaviour as the reference's C++ API,
executed on the B200 through the C-ABI (include/bbcodec.h):

  byte_split / byte_merge          codec.hpp:21-22   -> bb_split_host / bb_merge_host
  entropy_bits_per_byte            codec.hpp:26      -> bb_histogram256_host (+ host log2 sum)
  CodecBackend, backend_by_id/name codec.hpp:29-41   (ids 0 identity, 1 deflate)
  CodecContainer, serialize/parse  codec.hpp:43-60   (31-byte BBC1 header)
  compress / decompress            codec.hpp:62-65   -> bb_compress_host / bb_decompress_host
  EntropyReport, analyze           codec.hpp:67-79

Exceptions mirror include/beeplan/errors.hpp:40-56.  For HBM-resident tensors
use :class:`DeviceCodec` (stream-ordered, no host round trip).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import struct
import sys
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

from . import _lib

kBackendIdentity = 0
kBackendDeflate = 1
kContainerHeaderSize = 31
kContainerVersion = 1


class Error(RuntimeError):
    """beeplan::Error"""


class OddLength(Error):
    pass


class LaneLengthMismatch(Error):
    pass


class BackendUnknown(Error):
    pass


class CorruptContainer(Error):
    pass


class CudaError(Error):
    pass


class CorruptOffsets(Error):
    """beeplan::CorruptOffsets (errors.hpp:71)"""


class DimMismatch(Error):
    """beeplan::DimMismatch (errors.hpp:67)"""


_STATUS = {1: OddLength, 2: LaneLengthMismatch, 3: BackendUnknown, 4: CorruptContainer, 5: Error,
           6: CudaError, 7: ValueError, 8: CorruptOffsets, 9: DimMismatch}


def _check(rc: int) -> None:
    if rc:
        raise _STATUS.get(rc, Error)(_lib.last_error())


def _device() -> int:
    """The device of the module-level (host-buffer) calls: BEEPLAN_CUDA_DEVICE, else the caller's
    current torch device when torch has initialised CUDA (a torchrun worker bound to GPU k stays on
    GPU k), else 0 -- the C++ drop-in's rule (cpp/codec.cpp)."""
    env = os.environ.get("BEEPLAN_CUDA_DEVICE")
    if env:
        return int(env)
    torch = sys.modules.get("torch")
    if torch is not None and torch.cuda.is_initialized():
        return torch.cuda.current_device()
    return 0


def _ctx():
    return _lib.context(_device())


def _out(n: int):
    return (C.c_uint8 * max(1, n))()


@dataclass
class LanePair:
    high: bytes
    low: bytes


def byte_split(stream: bytes) -> LanePair:
    """high[k] = stream[2k+1], low[k] = stream[2k] (reference codec.cpp:86-99)."""
    stream = bytes(stream)
    if len(stream) % 2:
        raise OddLength(f"byte_split: stream length must be even, got {len(stream)}")
    L = _lib.load()
    n = len(stream) // 2
    hi, lo = _out(n), _out(n)
    _check(L.bb_split_host(_ctx(), stream, len(stream), hi, lo))
    return LanePair(bytes(hi)[:n], bytes(lo)[:n])


def byte_merge(high: bytes, low: bytes) -> bytes:
    high, low = bytes(high), bytes(low)
    if len(high) != len(low):
        raise LaneLengthMismatch(
            f"byte_merge: lane lengths differ ({len(high)} vs {len(low)})")
    L = _lib.load()
    out = _out(2 * len(high))
    _check(L.bb_merge_host(_ctx(), high, low, len(high), out))
    return bytes(out)[: 2 * len(high)]


def histogram256(data: bytes) -> List[int]:
    L = _lib.load()
    counts = (C.c_uint64 * 256)()
    _check(L.bb_histogram256_host(_ctx(), bytes(data), len(data), counts))
    return list(counts)


def entropy_from_counts(counts: Sequence[int], total: int) -> float:
    """Same double-precision summation order as codec.cpp:113-125."""
    if total == 0:
        return 0.0
    e = 0.0
    t = float(total)
    for c in counts:
        if c == 0:
            continue
        p = float(c) / t
        e -= p * math.log2(p)
    return e


def entropy_bits_per_byte(data: bytes) -> float:
    if len(data) == 0:
        return 0.0
    return entropy_from_counts(histogram256(data), len(data))


def _backend_encode(backend: int) -> Callable[[bytes], bytes]:
    def encode(lane: bytes) -> bytes:
        lane = bytes(lane)
        L = _lib.load()
        cap = L.bb_backend_bound(backend, len(lane))
        out = _out(cap)
        n = C.c_size_t()
        _check(L.bb_backend_encode_host(_ctx(), backend, lane, len(lane), out, cap, C.byref(n)))
        return bytes(out)[: n.value]
    return encode


def _backend_decode(backend: int) -> Callable[[bytes, int], bytes]:
    def decode(blob: bytes, expected_size: int) -> bytes:
        blob = bytes(blob)
        L = _lib.load()
        out = _out(expected_size)
        _check(L.bb_backend_decode_host(_ctx(), backend, blob, len(blob), expected_size, out))
        return bytes(out)[:expected_size]
    return decode


@dataclass(frozen=True)
class CodecBackend:
    id: int
    name: str
    encode: Callable[[bytes], bytes]
    decode: Callable[[bytes, int], bytes]


_BACKENDS = (
    CodecBackend(kBackendIdentity, "identity", _backend_encode(0), _backend_decode(0)),
    CodecBackend(kBackendDeflate, "deflate", _backend_encode(1), _backend_decode(1)),
)


def backends():
    return _BACKENDS


def backend_by_id(id: int) -> CodecBackend:
    for b in _BACKENDS:
        if b.id == id:
            return b
    raise BackendUnknown(f"codec backend id {id} is not registered")


def backend_by_name(name: str) -> CodecBackend:
    for b in _BACKENDS:
        if b.name == name:
            return b
    raise BackendUnknown(f"codec backend '{name}' is not registered")


@dataclass
class CodecContainer:
    backend_id: int = 0
    flags: int = 0
    element_count: int = 0
    high_blob: bytes = b""
    low_blob: bytes = b""

    def split(self) -> bool:
        return (self.flags & 0x01) != 0


def serialize_container(c: CodecContainer) -> bytes:
    return (b"BBC1" + bytes([kContainerVersion, c.backend_id & 0xFF, c.flags & 0xFF])
            + struct.pack("<QQQ", c.element_count, len(c.high_blob), len(c.low_blob))
            + bytes(c.high_blob) + bytes(c.low_blob))


def parse_container(data: bytes) -> CodecContainer:
    data = bytes(data)
    if len(data) < kContainerHeaderSize:
        raise CorruptContainer("container: truncated header")
    if data[:4] != b"BBC1":
        raise CorruptContainer("container: bad magic")
    if data[4] != kContainerVersion:
        raise CorruptContainer(f"container: unsupported version {data[4]}")
    count, hl, ll = struct.unpack_from("<QQQ", data, 7)
    avail = len(data) - kContainerHeaderSize
    if hl > avail or ll > avail - hl or hl + ll != avail:
        raise CorruptContainer("container: blob lengths do not match the payload")
    return CodecContainer(data[5], data[6], count, data[31:31 + hl], data[31 + hl:31 + hl + ll])


def compress_serialized(stream: bytes, backend_id: int, split: bool) -> bytes:
    """serialize_container(compress(...)) in one C-ABI call."""
    stream = bytes(stream)
    L = _lib.load()
    cap = L.bb_compress_bound(len(stream), backend_id, int(split))
    out = _out(cap)
    n = C.c_size_t()
    _check(L.bb_compress_host(_ctx(), stream, len(stream), backend_id, int(split), out, cap,
                              C.byref(n)))
    return bytes(out)[: n.value]


def compress(stream: bytes, backend_id: int, split: bool) -> CodecContainer:
    return parse_container(compress_serialized(stream, backend_id, split))


def decompress_serialized(data: bytes) -> bytes:
    data = bytes(data)
    L = _lib.load()
    need = C.c_size_t()
    _check(L.bb_decompress_host(_ctx(), data, len(data), None, 0, C.byref(need)))
    out = _out(need.value)
    n = C.c_size_t()
    _check(L.bb_decompress_host(_ctx(), data, len(data), out, need.value, C.byref(n)))
    return bytes(out)[: n.value]


def decompress(container: CodecContainer) -> bytes:
    return decompress_serialized(serialize_container(container))


@dataclass
class EntropyReport:
    raw_entropy: float = 0.0
    high_entropy: float = 0.0
    low_entropy: float = 0.0
    raw_size: int = 0
    lane_size: int = 0
    raw_mode_compressed: int = 0
    high_lane_compressed: int = 0
    low_lane_compressed: int = 0
    split_mode_compressed: int = 0
    ratio: float = 0.0


def analyze(stream: bytes, backend_id: int) -> EntropyReport:
    """reference codec.cpp:194-213"""
    stream = bytes(stream)
    r = EntropyReport()
    r.raw_size = len(stream)
    r.raw_entropy = entropy_bits_per_byte(stream)
    lanes = byte_split(stream)
    r.lane_size = len(lanes.high)
    r.high_entropy = entropy_bits_per_byte(lanes.high)
    r.low_entropy = entropy_bits_per_byte(lanes.low)
    raw_mode = compress(stream, backend_id, False)
    split_mode = compress(stream, backend_id, True)
    r.raw_mode_compressed = len(raw_mode.high_blob)
    r.high_lane_compressed = len(split_mode.high_blob)
    r.low_lane_compressed = len(split_mode.low_blob)
    r.split_mode_compressed = r.high_lane_compressed + r.low_lane_compressed
    r.ratio = 0.0 if not stream else r.split_mode_compressed / r.raw_size
    return r


# ---------------------------------------------------------------------------
# HBM-resident path


class DeviceCodec:
    """Stream-ordered codec over CUDA tensors (uint8, contiguous, on ``device``)."""

    def __init__(self, device: int = 0):
        import torch
        self.torch = torch
        self.device = device
        self.L = _lib.load()
        _lib.context(device)

    @property
    def ctx(self):
        """The calling thread's C-ABI context (contexts are per host thread), so one
        DeviceCodec can be driven from several threads, each on its own stream."""
        return _lib.context(self.device)

    def _stream(self, stream=None) -> int:
        s = stream if stream is not None else self.torch.cuda.current_stream(self.device)
        return s.cuda_stream

    def compress_bound(self, n: int, backend: int = kBackendDeflate, split: bool = True) -> int:
        return int(self.L.bb_compress_bound(n, backend, int(split)))

    def compress_into(self, x, out, backend: int = kBackendDeflate, split: bool = True,
                      stream=None) -> int:
        n = C.c_size_t()
        _check(self.L.bb_compress(self.ctx, x.data_ptr(), x.numel(), backend, int(split),
                                  out.data_ptr(), out.numel(), C.byref(n), self._stream(stream)))
        return n.value

    def compress(self, x, backend: int = kBackendDeflate, split: bool = True, stream=None):
        out = self.torch.empty(self.compress_bound(x.numel(), backend, split),
                               dtype=self.torch.uint8, device=x.device)
        n = self.compress_into(x, out, backend, split, stream)
        return out[:n]

    def compress_batch(self, xs, outs, backend: int = kBackendDeflate, split: bool = True,
                       stream=None) -> List[int]:
        k = len(xs)
        ins = (C.c_void_p * k)(*[x.data_ptr() for x in xs])
        ns = (C.c_size_t * k)(*[x.numel() for x in xs])
        os_ = (C.c_void_p * k)(*[o.data_ptr() for o in outs])
        caps = (C.c_size_t * k)(*[o.numel() for o in outs])
        lens = (C.c_size_t * k)()
        st = (C.c_int * k)()
        _check(self.L.bb_compress_batch(self.ctx, k, ins, ns, backend, int(split), os_, caps, lens,
                                        st, self._stream(stream)))
        return list(lens)

    def compress_batch_ptr(self, xs, out_ptrs, out_caps, backend: int = kBackendDeflate, split: bool = True,
                           stream=None) -> List[int]:
        """compress_batch into raw device addresses (e.g. the next stage's inbox mapped by CUDA IPC)."""
        k = len(xs)
        ins = (C.c_void_p * k)(*[x.data_ptr() for x in xs])
        ns = (C.c_size_t * k)(*[x.numel() for x in xs])
        os_ = (C.c_void_p * k)(*[int(p) for p in out_ptrs])
        caps = (C.c_size_t * k)(*[int(c) for c in out_caps])
        lens = (C.c_size_t * k)()
        st = (C.c_int * k)()
        _check(self.L.bb_compress_batch(self.ctx, k, ins, ns, backend, int(split), os_, caps, lens,
                                        st, self._stream(stream)))
        return list(lens)

    def decoded_size(self, c, stream=None) -> int:
        n = C.c_size_t()
        _check(self.L.bb_decompress(self.ctx, c.data_ptr(), c.numel(), None, 0, C.byref(n),
                                    self._stream(stream)))
        return n.value

    def decompress_into(self, c, out, stream=None) -> int:
        n = C.c_size_t()
        _check(self.L.bb_decompress(self.ctx, c.data_ptr(), c.numel(), out.data_ptr(), out.numel(),
                                    C.byref(n), self._stream(stream)))
        return n.value

    def decompress(self, c, stream=None):
        out = self.torch.empty(max(1, self.decoded_size(c, stream)), dtype=self.torch.uint8,
                               device=c.device)
        n = self.decompress_into(c, out, stream)
        return out[:n]

    def decompress_batch(self, cs, outs, stream=None) -> List[int]:
        k = len(cs)
        ins = (C.c_void_p * k)(*[c.data_ptr() for c in cs])
        ns = (C.c_size_t * k)(*[c.numel() for c in cs])
        os_ = (C.c_void_p * k)(*[o.data_ptr() for o in outs])
        caps = (C.c_size_t * k)(*[o.numel() for o in outs])
        lens = (C.c_size_t * k)()
        st = (C.c_int * k)()
        _check(self.L.bb_decompress_batch(self.ctx, k, ins, ns, os_, caps, lens, st,
                                          self._stream(stream)))
        return list(lens)

    def split(self, x, high, low, stream=None) -> None:
        _check(self.L.bb_split(x.data_ptr(), x.numel(), high.data_ptr(), low.data_ptr(),
                               self._stream(stream)))

    def merge(self, high, low, out, stream=None) -> None:
        _check(self.L.bb_merge(high.data_ptr(), low.data_ptr(), high.numel(), out.data_ptr(),
                               self._stream(stream)))

    def histogram256(self, x, counts, stream=None) -> None:
        _check(self.L.bb_histogram256(x.data_ptr(), x.numel(), counts.data_ptr(),
                                      self._stream(stream)))
