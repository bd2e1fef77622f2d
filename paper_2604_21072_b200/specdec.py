"""Speculative-decoding token-tree payloads.

Mirror of the reference's packed layout (proj/include/beeplan/specdec.hpp:57-76,
proj/src/specdec.cpp:153-220) plus the device path that produces it from HBM:

  PackedBatch                    specdec.hpp:59-66   hidden_dim, f32 payload [sum N', D], u32 offsets
  pack(per_request)              specdec.cpp:153-165 raises DimMismatch
  unpack(batch)                  specdec.cpp:167-189 raises CorruptOffsets
  encode_packed(batch)           specdec.cpp:192-198 u32 count | u32 offsets[] | f32 payload (LE)
  decode_packed(data, dim)       specdec.cpp:200-220 raises CorruptOffsets
  DevicePacker.pack_encode       bb_pack_sd: keep-mask scan + warp-per-row gather on the B200,
                                 output == encode_packed(pack(kept rows per request)) byte for byte
  DevicePacker.open              bb_unpack_sd: decode_packed's checks on an HBM image, f32 view

The host functions operate on host Python data exactly as the reference's do;
the token trees of a serving stage live in HBM and go through DevicePacker,
then through the BBC1 codec into ``PackedSd`` BBF1 frames (wire.hpp:18).
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from . import _lib
from .codec import CorruptOffsets, DimMismatch, _check

__all__ = ["PackedBatch", "pack", "unpack", "encode_packed", "decode_packed", "DevicePacker",
           "CorruptOffsets", "DimMismatch"]


@dataclass
class PackedBatch:
    hidden_dim: int = 0
    payload: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))
    offsets: List[int] = field(default_factory=list)

    def request_count(self) -> int:
        return len(self.offsets) - 1 if self.offsets else 0

    def total_states(self) -> int:
        return self.offsets[-1] if self.offsets else 0


def pack(per_request: Sequence[Sequence[Sequence[float]]]) -> PackedBatch:
    """Concatenate each request's retained vectors; offsets are prefix sums of the counts.
    The first vector fixes hidden_dim (specdec.cpp:158-160)."""
    dim, rows, offsets = 0, [], [0]
    for states in per_request:
        for vec in states:
            v = np.asarray(vec, dtype=np.float32).reshape(-1)
            if dim == 0:
                dim = v.size
            if v.size != dim:
                raise DimMismatch("pack: hidden vectors must share one dimension")
            rows.append(v)
        offsets.append(offsets[-1] + len(states))
    payload = np.concatenate(rows) if rows else np.zeros(0, np.float32)
    return PackedBatch(dim, payload.astype(np.float32, copy=False), offsets)


def _check_offsets(batch: PackedBatch) -> None:
    off = batch.offsets
    if not off or off[0] != 0:
        raise CorruptOffsets("unpack: offsets must start at 0")
    for i in range(1, len(off)):
        if off[i] < off[i - 1]:
            raise CorruptOffsets("unpack: offsets must be non-decreasing")
    n = len(batch.payload)
    if (n != 0) if batch.hidden_dim == 0 else (n != off[-1] * batch.hidden_dim):
        raise CorruptOffsets("unpack: payload length does not match offsets")


def unpack(batch: PackedBatch) -> List[List[np.ndarray]]:
    _check_offsets(batch)
    d = batch.hidden_dim
    return [[batch.payload[s * d:(s + 1) * d] for s in range(batch.offsets[r], batch.offsets[r + 1])]
            for r in range(len(batch.offsets) - 1)]


def encode_packed(batch: PackedBatch) -> bytes:
    head = struct.pack(f"<I{len(batch.offsets)}I", len(batch.offsets), *batch.offsets)
    return head + np.asarray(batch.payload, dtype="<f4").tobytes()


def decode_packed(data: bytes, hidden_dim: int) -> PackedBatch:
    if len(data) < 4:
        raise CorruptOffsets("packed batch: truncated offset count")
    (count,) = struct.unpack_from("<I", data, 0)
    if count < 1 or len(data) < 4 + 4 * count:
        raise CorruptOffsets("packed batch: truncated offsets")
    offsets = list(struct.unpack_from(f"<{count}I", data, 4))
    off = 4 + 4 * count
    nbytes = len(data) - off
    if nbytes % 4 != 0 or nbytes // 4 != offsets[-1] * hidden_dim:
        raise CorruptOffsets("packed batch: payload length does not match offsets")
    batch = PackedBatch(hidden_dim, np.frombuffer(data, dtype="<f4", offset=off).astype(np.float32),
                        offsets)
    _check_offsets(batch)
    return batch


class DevicePacker:
    """Packs HBM-resident token-tree states into the PackedBatch wire image on the GPU."""

    def __init__(self, device: int = 0):
        import torch
        self.torch = torch
        self.device = device
        self.L = _lib.load()

    def _stream(self, stream=None) -> int:
        s = stream if stream is not None else self.torch.cuda.current_stream(self.device)
        return s.cuda_stream

    def bound(self, n_rows: int, hidden_dim: int, n_requests: int) -> int:
        return int(self.L.bb_packed_bound(n_rows, hidden_dim, n_requests))

    def pack_encode(self, rows, keep, request_rows: Sequence[int], out=None, stream=None):
        """rows: [R, D] float32 CUDA tensor; keep: [R] bool/uint8 (pruning result);
        request_rows: R-boundaries of the requests (len n_requests + 1, starts at 0).
        Returns a uint8 CUDA view holding encode_packed(pack(...))."""
        t = self.torch
        if rows.dtype != t.float32 or rows.dim() != 2 or not rows.is_contiguous():
            raise ValueError("pack_encode: rows must be a contiguous [R, D] float32 tensor")
        keep = keep.to(t.uint8).contiguous()
        n_rows, dim = rows.shape
        n_req = len(request_rows) - 1
        if n_req < 0:
            raise ValueError("pack_encode: request_rows needs at least one entry")
        if out is None:
            out = t.empty(self.bound(n_rows, dim, n_req), dtype=t.uint8, device=rows.device)
        req = (C.c_uint32 * (n_req + 1))(*request_rows)
        n = C.c_size_t()
        _check(self.L.bb_pack_sd(rows.data_ptr(), n_rows, dim, keep.data_ptr(), req, n_req,
                                 out.data_ptr(), out.numel(), C.byref(n), self._stream(stream)))
        return out[:n.value]

    def open(self, packed, hidden_dim: int, stream=None):
        """decode_packed's checks on an HBM image; returns (offsets, payload [total, D] f32 view)."""
        cnt = C.c_uint32()
        _check(self.L.bb_unpack_sd(packed.data_ptr(), packed.numel(), hidden_dim, None, 0,
                                   C.byref(cnt), None, self._stream(stream)))
        offs = (C.c_uint32 * cnt.value)()
        poff = C.c_size_t()
        _check(self.L.bb_unpack_sd(packed.data_ptr(), packed.numel(), hidden_dim, offs, cnt.value,
                                   C.byref(cnt), C.byref(poff), self._stream(stream)))
        offsets = list(offs)
        payload = packed[poff.value:]
        total = offsets[-1]
        if hidden_dim == 0 or total == 0:
            return offsets, self.torch.empty((total, hidden_dim), dtype=self.torch.float32,
                                             device=packed.device)
        return offsets, payload.view(self.torch.float32).view(total, hidden_dim)
