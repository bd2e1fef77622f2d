"""Debug helper: decompress config2-like micro-batches and report parallel / fallback counts."""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2604_21072_b200 import _lib, codec, synth  # noqa: E402

L = _lib.load()
L.bb_debug_inflate_counts.argtypes = [C.c_void_p]


def counts():
    out = (C.c_uint64 * 3)()
    L.bb_debug_inflate_counts(out)
    return list(out)


dc = codec.DeviceCodec(0)
for seed in (1000, 1001):
    raw = synth.gaussian(16 * 512 * 4096, seed, True)
    x = torch.frombuffer(bytearray(raw), dtype=torch.uint8).cuda()
    c = dc.compress(x)
    b = counts()
    t = time.time()
    y = dc.decompress(c)
    torch.cuda.synchronize()
    a = counts()
    print(seed, "ok" if torch.equal(x, y) else "MISMATCH", "par_ok/fallback/seq delta", [a[i] - b[i] for i in range(3)],
          f"{time.time() - t:.3f}s", flush=True)
