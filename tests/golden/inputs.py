"""Deterministic input recipes for the golden vectors (test infrastructure).

Every golden entry names its input by a spec string so the fixture stays small
(SHA-256 + sizes, not blobs) and the same bytes can be rebuilt on the GPU box,
where /root/reference does not exist:

  fp16:<elements>:<seed>     reference synth_gaussian_fp16 (proj/src/synth.cpp:66-94)
  bf16:<elements>:<seed>     the frozen bf16 variant (same Box-Muller stream, bf16 RNE)
  rand:<bytes>:<seed>        numpy PCG64 random bytes
  const:<bytes>:<value>      one repeated byte
  skew:<bytes>:<seed>:<k>    uniform over a k-letter alphabet
  period:<bytes>:<seed>:<p>  a random p-byte pattern repeated
  runs:<bytes>:<seed>        runs of 1..600 of four byte values
"""
from __future__ import annotations

import numpy as np


def make_input(spec: str, oracle=None) -> bytes:
    kind, *a = spec.split(":")
    if kind in ("fp16", "bf16"):
        if oracle is None:
            from oracle.oracle import Oracle
            oracle = Oracle()
        n, seed = int(a[0]), int(a[1])
        return oracle.synth_fp16(n, seed) if kind == "fp16" else oracle.synth_bf16(n, seed)
    n = int(a[0])
    if kind == "rand":
        return np.random.default_rng(int(a[1])).bytes(n)
    if kind == "const":
        return bytes([int(a[1])]) * n
    if kind == "skew":
        rng = np.random.default_rng(int(a[1]))
        return rng.integers(0, int(a[2]), n, dtype=np.uint8).tobytes()
    if kind == "period":
        rng = np.random.default_rng(int(a[1]))
        pat = rng.bytes(int(a[2]))
        return (pat * (n // len(pat) + 1))[:n]
    if kind == "runs":
        rng = np.random.default_rng(int(a[1]))
        out = bytearray()
        while len(out) < n:
            out += bytes([int(rng.integers(0, 4))]) * int(rng.integers(1, 601))
        return bytes(out[:n])
    raise ValueError(spec)
