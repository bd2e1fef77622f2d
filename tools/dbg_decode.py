import sys, zlib, random, time
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2604_21072_b200 import codec
dec = codec.backend_by_id(1).decode
rng = random.Random(21)
cases = [("rand200k", rng.randbytes(200000)), ("ab200k", bytes(rng.choice(b"ab") for _ in range(200000))),
         ("sk64", np.random.default_rng(3).integers(0, 64, 200000, dtype=np.uint8).tobytes())]
for name, data in cases:
    for level in (6, 1, 9, 0):
        blob = zlib.compress(data, level)
        t = time.time()
        out = dec(blob, len(data))
        print(name, level, len(blob), out == data, "%.3f s" % (time.time() - t), flush=True)
import ctypes as C
from paper_2604_21072_b200 import _lib
L = _lib.load()
wd = (C.c_ulonglong * 8)()
L.bb_debug_inflate_watchdog(wd)
print("watchdog", list(wd))
