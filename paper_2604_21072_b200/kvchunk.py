"""KV-cache offload chunks (BASELINE configs[3]).

BloomBee offloads KV caches to host / peer memory; the reference repository only
models the cost (proj/src/cost_model.cpp:30-47: KV bytes = 2 * layers * ctx * d * 2 B,
offload fraction alpha).  The chunk unit here is SURVEY §8 config 4's: one
(layer, K|V, sequence) slab [ctx, d] of fp16 = 40 MiB for LLaMA-2-13B at 4K context.

  chunk_id(layer, kind, seq, batch)     (2 * layer + kind) * batch + seq
  KvChunker.chunks(k, v, layer)         contiguous [B, T, D] caches: zero-copy views
  KvChunker.gather(pool, page_ids, ...) paged caches: bb_gather_pages on the B200
  KvChunker.compress(chunks)            BBC1 containers through one bb_compress_batch
  KvChunker.frames(...)                 BBF1 frames (batch_id = chunk id) for the hand-off
"""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence, Tuple

from . import _lib
from .codec import DeviceCodec, _check

K_CACHE, V_CACHE = 0, 1


def chunk_id(layer: int, kind: int, seq: int, batch: int) -> int:
    return (2 * layer + kind) * batch + seq


class KvChunker:
    def __init__(self, device: int = 0, codec: DeviceCodec | None = None):
        import torch
        self.torch = torch
        self.device = device
        self.L = _lib.load()
        self.codec = codec or DeviceCodec(device)

    def chunks(self, k, v, layer: int) -> List[Tuple[int, object]]:
        """(chunk id, uint8 view) per (K|V, sequence) of one layer's [B, T, D] caches."""
        out = []
        for kind, t in ((K_CACHE, k), (V_CACHE, v)):
            if not t.is_contiguous():
                raise ValueError("KvChunker.chunks: caches must be contiguous [B, T, D]")
            b = t.shape[0]
            flat = t.view(b, -1).view(self.torch.uint8)
            for s in range(b):
                out.append((chunk_id(layer, kind, s, b), flat[s]))
        return out

    def gather(self, pool, page_ids, out=None, stream=None):
        """Contiguous chunk from a paged cache: pool [n_pool, page elems...] (any dtype),
        page_ids [n] int32/uint32 on the device (a sequence's page table)."""
        t = self.torch
        pool_u8 = pool.contiguous().view(t.uint8).view(pool.shape[0], -1)
        ids = page_ids.to(t.int32).contiguous()
        page_bytes = pool_u8.shape[1]
        if out is None:
            out = t.empty(ids.numel() * page_bytes, dtype=t.uint8, device=pool.device)
        s = stream if stream is not None else t.cuda.current_stream(self.device)
        _check(self.L.bb_gather_pages(pool_u8.data_ptr(), pool_u8.shape[0], page_bytes, ids.data_ptr(),
                                      ids.numel(), out.data_ptr(), s.cuda_stream))
        return out

    def compress(self, chunks: Sequence, outs=None, backend: int = 1, split: bool = True):
        """BBC1 containers of many chunks through one batched codec pipeline."""
        t = self.torch
        views = [c[1] if isinstance(c, tuple) else c for c in chunks]
        if outs is None:
            outs = [t.empty(self.codec.compress_bound(x.numel(), backend, split), dtype=t.uint8,
                            device=x.device) for x in views]
        lens = self.codec.compress_batch(views, outs, backend, split)
        return [o[:n] for o, n in zip(outs, lens)]

    def frames(self, chunks: Sequence[Tuple[int, object]], containers: Sequence):
        """BBF1 frames (compressed + byte split) with batch_id = chunk id."""
        import torch
        from .pipeline import FLAG_BYTE_SPLIT, FLAG_COMPRESSED, FRAME_HEADER, frame_header
        hdrs = b"".join(frame_header(0, cid, 0, FLAG_COMPRESSED | FLAG_BYTE_SPLIT, int(c.numel()))
                        for (cid, _), c in zip(chunks, containers))
        if not containers:
            return []
        h = torch.frombuffer(bytearray(hdrs), dtype=torch.uint8).to(containers[0].device)
        return [torch.cat([h[FRAME_HEADER * i:FRAME_HEADER * (i + 1)], c]) for i, c in enumerate(containers)]
