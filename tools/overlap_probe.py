"""Encode / decode overlap probe on one GPU (config2 step: 8 x 64 MiB bf16 micro-batches).

seq:    compress_batch(all 8) then decompress_batch(all 8) on one thread / stream (bench.py's step)
pipeK:  the 8 micro-batches in K groups; an encode thread compresses group g while a decode thread
        (own codec context and stream) decompresses group g-1 -- the schedule of a stage GPU that
        decodes its inbound micro-batches while it encodes its outbound ones.

    python tools/overlap_probe.py [--steps 5]
"""
from __future__ import annotations

import argparse
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    import torch

    from paper_2604_21072_b200 import codec
    from paper_2604_21072_b200 import synth as S
    from paper_2604_21072_b200 import workloads as W
    syn = lambda n, s, bf16: S.gaussian(n, s, bf16)  # noqa: E731
    hs = [W.config2_micro(syn, 0, i) for i in range(W.C2_MICRO)]
    dc = codec.DeviceCodec(0)
    xs = [torch.frombuffer(bytearray(h), dtype=torch.uint8).cuda() for h in hs]
    outs = [torch.empty(dc.compress_bound(x.numel()), dtype=torch.uint8, device="cuda") for x in xs]
    decs = [torch.empty_like(x) for x in xs]
    se, sd = torch.cuda.Stream(), torch.cuda.Stream()
    raw = sum(x.numel() for x in xs)

    def seq():
        with torch.cuda.stream(se):
            lens = dc.compress_batch(xs, outs, stream=se)
            dc.decompress_batch([o[:n] for o, n in zip(outs, lens)], decs, stream=se)

    def pipe(k):
        groups = [list(range(g * len(xs) // k, (g + 1) * len(xs) // k)) for g in range(k)]
        ready = [threading.Event() for _ in groups]
        lens = [0] * len(xs)
        err = []

        def enc():
            try:
                for g, idx in enumerate(groups):
                    got = dc.compress_batch([xs[i] for i in idx], [outs[i] for i in idx], stream=se)
                    for i, n in zip(idx, got):
                        lens[i] = n
                    ready[g].set()
            except Exception as e:  # noqa: BLE001
                err.append(e)
                for r in ready:
                    r.set()

        def dec():
            try:
                for g, idx in enumerate(groups):
                    ready[g].wait()
                    if err:
                        return
                    dc.decompress_batch([outs[i][:lens[i]] for i in idx], [decs[i] for i in idx], stream=sd)
            except Exception as e:  # noqa: BLE001
                err.append(e)

        te, td = threading.Thread(target=enc), threading.Thread(target=dec)
        te.start(), td.start()
        te.join(), td.join()
        if err:
            raise err[0]

    for name, fn in [("seq", seq), ("pipe2", lambda: pipe(2)), ("pipe4", lambda: pipe(4)),
                     ("pipe8", lambda: pipe(8)), ("seq", seq)]:
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            fn()
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3 / args.steps
        ok = all(torch.equal(d, x) for d, x in zip(decs, xs))
        for d in decs:
            d.zero_()
        print(f"{name:6s} {ms:8.2f} ms/step  {2 * raw / ms / 1e6:6.2f} GB/s (enc+dec bytes)  lossless={ok}", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
