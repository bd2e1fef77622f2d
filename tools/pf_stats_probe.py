import ctypes as C, sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2604_21072_b200 import _lib, codec, synth as S, workloads as W
L = _lib.load()
L.bb_debug_pf_stats.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
dc = codec.DeviceCodec(0)
syn = lambda n, s, b: S.gaussian(n, s, b)
for name, hs in [("config2", [W.config2_micro(syn, 0, i) for i in range(2)]), ("config4", [W.kv_chunk(syn, i) for i in range(2)])]:
    xs = [torch.frombuffer(bytearray(h), dtype=torch.uint8).cuda() for h in hs]
    outs = [torch.empty(dc.compress_bound(x.numel()), dtype=torch.uint8, device="cuda") for x in xs]
    st = (C.c_ulonglong * 4)()
    L.bb_debug_pf_stats(st, 1)
    dc.compress_batch(xs, outs)
    torch.cuda.synchronize()
    L.bb_debug_pf_stats(st, 0)
    fl, rec, it, bt = list(st)
    print(name, "batches", bt, "flushes", fl, "recorded", rec, "warp iterations", it, "iter*32/recorded", round(it * 32 / max(1, rec), 2), "recorded per flush", round(rec / max(1, fl), 1))
