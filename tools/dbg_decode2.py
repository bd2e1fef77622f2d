import sys, zlib, time
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2604_21072_b200 import codec
dec = codec.backend_by_id(1).decode
data = np.random.default_rng(3).integers(0, 64, 200000, dtype=np.uint8).tobytes()
blob = zlib.compress(data, 6)
print("blob", len(blob), flush=True)
t = time.time()
out = dec(blob, len(data))
print("ok", out == data, time.time() - t, flush=True)
