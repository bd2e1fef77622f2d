"""Sequential-inflate probe: device time of one container decode per payload size, with the
parallel decoder bypassed (BB_INFLATE_SEQ=1) or at the default routing.

    python tools/seq_probe.py            # default routing
    BB_INFLATE_SEQ=1 python tools/seq_probe.py
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    import torch

    from paper_2604_21072_b200 import codec
    from paper_2604_21072_b200 import synth as S
    dc = codec.DeviceCodec(0)
    for n in (4096, 16384, 104100, 416400):
        h = S.gaussian(n // 2, 77, False)
        x = torch.frombuffer(bytearray(h), dtype=torch.uint8).cuda()
        c = dc.compress(x)
        out = torch.empty(n, dtype=torch.uint8, device="cuda")
        for _ in range(2):
            dc.decompress_batch([c], [out])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            dc.decompress_batch([c], [out])
        e1.record()
        torch.cuda.synchronize()
        ok = torch.equal(out, x)
        print(f"{n:8d} B payload -> {c.numel():8d} B container: decode {e0.elapsed_time(e1) / 5:.3f} ms, lossless={ok}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
