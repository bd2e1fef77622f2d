"""Single-process view of the fused NVLink hand-off (for ncu's nvltx / nvlrx counters, which
cannot be collected on a multi-rank torchrun command): GPU 0 compresses config2's 8 micro-batches
with its containers' destinations in GPU 1's HBM (peer access, as PeerInbox's IPC-imported slots),
so the codec's emit / header kernels write the frames over NVLink; GPU 1 then decodes them and the
round trip is checked.

    python tools/fused_peer.py
    ncu --metrics nvltx__bytes.sum,nvlrx__bytes.sum,gpu__time_duration.sum \
        -k regex:"k_emit|k_zero|k_container_header|k_adler_final" python tools/fused_peer.py
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    import torch

    from paper_2604_21072_b200 import _lib, codec
    from paper_2604_21072_b200 import synth as S
    from paper_2604_21072_b200 import workloads as W
    assert torch.cuda.device_count() >= 2, "needs two GPUs"
    L = _lib.load()
    assert L.bb_enable_peer_access(0, 1) == 0, _lib.last_error()
    syn = lambda n, s, bf16: S.gaussian(n, s, bf16)  # noqa: E731
    hs = [W.config2_micro(syn, 0, i) for i in range(W.C2_MICRO)]
    torch.cuda.set_device(0)
    dc0 = codec.DeviceCodec(0)
    xs = [torch.frombuffer(bytearray(h), dtype=torch.uint8).to("cuda:0") for h in hs]
    caps = [dc0.compress_bound(x.numel()) for x in xs]
    inbox = [torch.empty(c, dtype=torch.uint8, device="cuda:1") for c in caps]  # GPU 1's HBM
    for _ in range(2):
        lens = dc0.compress_batch_ptr(xs, [b.data_ptr() for b in inbox], caps)
    torch.cuda.synchronize(0)
    total = sum(lens)
    torch.cuda.set_device(1)
    dc1 = codec.DeviceCodec(1)
    decs = [torch.empty(x.numel(), dtype=torch.uint8, device="cuda:1") for x in xs]
    dc1.decompress_batch([b[:n] for b, n in zip(inbox, lens)], decs)
    torch.cuda.synchronize(1)
    ok = all(torch.equal(d.cpu(), x.cpu()) for d, x in zip(decs, xs))
    print(f"containers {total} B written into GPU 1 by GPU 0's codec kernels (x2 calls); lossless={ok}")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
