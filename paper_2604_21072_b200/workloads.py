"""Synthetic inputs of the BASELINE.json configs (shapes, seeds, recipes).

One definition shared by bench.py, the GPU parity tests and the full-size golden
generator (tests/golden/make_fullsize_golden.py), so the bytes the benchmark times are
the bytes whose reference containers are pinned.  Every generator takes a ``synth``
callable ``synth(elements, seed, bf16) -> bytes``: the product harnesses pass the C++
drop-in generator (paper_2604_21072_b200/synth.py), the golden generator passes the
oracle's; both are pinned to the reference's synth_gaussian_fp16 (proj/src/synth.cpp:66-94).

  config1  [1,128,4096] fp16 hidden state, seed 1                       (configs[0])
  config2  8 micro-batches of [16,512,4096] bf16 per stage boundary;
           stage ``rank`` micro-batch i uses seed 1000*(rank+1)+i         (configs[1])
  config3  32 token trees per pass (width 64 x depth 8 = 512 states, d=4096) as f32
           (exact upcast of synth fp16, seed 7+r) with a 60 % keep mask (PCG64 7000+r),
           packed into encode_packed's layout                            (configs[2])
  config4  LLaMA-2-13B KV chunks [4096, 5120] fp16, seed = chunk id        (configs[3])
  config5  d=8192 fp16 rows, 1 MiB .. 4 GiB; 1 MiB block b of size index si uses
           seed 50000 + 4096*si + b + 1000000*rank; cut into 512 MiB frames (configs[4])
"""
from __future__ import annotations

from typing import Callable, List, Tuple

MiB = 1 << 20

C1_ELEMS = 128 * 4096
C2_MICRO, C2_ELEMS = 8, 16 * 512 * 4096
SD_REQUESTS, SD_NODES, SD_DIM, SD_KEEP_PCT = 32, 64 * 8, 4096, 60
KV_BATCH, KV_CTX, KV_DIM = 32, 4096, 5120
SWEEP_DIM = 8192
SWEEP_PIECE = 512 * MiB  # frames carry <= 1 GiB (wire.cpp:31): larger tensors are cut

Synth = Callable[[int, int, bool], bytes]


def config2_seed(rank: int, i: int) -> int:
    return 1000 * (rank + 1) + i


def config2_micro(synth: Synth, rank: int, i: int) -> bytes:
    return synth(C2_ELEMS, config2_seed(rank, i), True)


def kv_chunk_id(layer: int, kind: int, seq: int, batch: int = KV_BATCH) -> int:
    return (2 * layer + kind) * batch + seq


def kv_layer_ids(layer: int) -> List[int]:
    """Chunk ids of one layer in offload order: K of every sequence, then V."""
    return [kv_chunk_id(layer, kind, s) for kind in (0, 1) for s in range(KV_BATCH)]


def kv_chunk(synth: Synth, cid: int) -> bytes:
    return synth(KV_CTX * KV_DIM, cid, False)


def sd_request(synth: Synth, r: int):
    """Request r's token tree: [512, 4096] f32 states + uint8 keep mask."""
    import numpy as np
    states = np.frombuffer(synth(SD_NODES * SD_DIM, 7 + r, False), dtype="<f2").astype(np.float32)
    keep = (np.random.default_rng(7000 + r).integers(0, 100, SD_NODES) < SD_KEEP_PCT).astype(np.uint8)
    return states.reshape(SD_NODES, SD_DIM), keep


def sd_packed_image(synth: Synth, first: int = 0, n: int = SD_REQUESTS) -> Tuple[bytes, list]:
    """Host encode_packed(pack(kept rows per request)) of requests first..first+n-1
    (specdec.cpp:153-198 layout: u32 count | u32 offsets[count] | f32 rows)."""
    import struct

    import numpy as np
    rows, offsets = [], [0]
    for r in range(first, first + n):
        st, kp = sd_request(synth, r)
        kept = st[kp.astype(bool)]
        rows.append(kept)
        offsets.append(offsets[-1] + kept.shape[0])
    head = struct.pack(f"<I{len(offsets)}I", len(offsets), *offsets)
    return head + np.concatenate(rows).astype("<f4").tobytes(), offsets


def sweep_sizes(max_mib: int = 1024) -> List[int]:
    sizes = [MiB << (2 * k) for k in range(6)]  # 1, 4, 16, 64, 256, 1024 MiB
    if max_mib >= 4096:
        sizes.append(4096 * MiB)
    return sizes


def sweep_block_seed(si: int, b: int, rank: int = 0) -> int:
    return 50000 + 4096 * si + b + 1000000 * rank


def sweep_tensor(synth: Synth, si: int, size: int, rank: int = 0) -> bytes:
    """Size index si of the sweep: size // 1 MiB blocks of 64 rows x d=8192 fp16."""
    return b"".join(synth(MiB // 2, sweep_block_seed(si, b, rank), False) for b in range(size // MiB))
