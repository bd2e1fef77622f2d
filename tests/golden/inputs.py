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


def sd_tree(spec: str):
    """Speculative-decoding token-tree batch (config 3 shape family), numpy only.

    spec = sdtree:<requests>:<nodes>:<dim>:<seed>:<keep_percent>:<kind>
      nodes per request is ragged: nodes - U[0, nodes/4] (some requests may be empty when
      nodes is small); kind "f32" = N(0,1) floats, "bf16up" = bf16-representable values
      (low 16 bits zero, as a bf16 model's states upcast), "special" = f32 with NaN/Inf/-0
      payloads.
    Returns (rows float32 [R, dim], keep uint8 [R], request_rows list[int], per_request lists).
    """
    _, nreq, nodes, dim, seed, keep_pct, kind = spec.split(":")
    nreq, nodes, dim, seed, keep_pct = int(nreq), int(nodes), int(dim), int(seed), int(keep_pct)
    rng = np.random.default_rng(seed)
    counts = [max(0, nodes - int(rng.integers(0, nodes // 4 + 1))) for _ in range(nreq)]
    total = sum(counts)
    rows = rng.standard_normal((total, dim), dtype=np.float32)
    if kind == "bf16up":
        rows = (rows.view(np.uint32) & np.uint32(0xFFFF0000)).view(np.float32)
    elif kind == "special":
        bits = rows.view(np.uint32).copy()
        sel = rng.integers(0, 64, bits.shape)
        bits[sel == 0] = 0x7FC00001  # quiet NaN with payload
        bits[sel == 1] = 0x7F800000  # +inf
        bits[sel == 2] = 0x80000000  # -0
        bits[sel == 3] = 0x00000001  # denormal
        rows = bits.view(np.float32)
    keep = (rng.integers(0, 100, total) < keep_pct).astype(np.uint8)
    request_rows = [0]
    for c in counts:
        request_rows.append(request_rows[-1] + c)
    per_request = []
    for r in range(nreq):
        lo, hi = request_rows[r], request_rows[r + 1]
        per_request.append([rows[i] for i in range(lo, hi) if keep[i]])
    return rows, keep, request_rows, per_request
