"""Pins the CPU oracle (oracle/*.c) before anything is checked against it.

1. against the committed golden vectors generated from the reference itself
   (tests/golden/make_golden.py -> reference codec.cpp + zlib 1.3);
2. against the live reference (oracle/_ref) where it was built;
3. differentially against Python's zlib (the same system libz 1.3) on a corpus
   aimed at zlib's window / block / lazy-match corner cases.
"""
import hashlib
import random
import zlib

import numpy as np
import pytest
from inputs import make_input


def test_zlib_is_the_pinned_version():
    assert zlib.ZLIB_RUNTIME_VERSION == "1.3"


def test_backend_kats(oracle, golden):
    kat = golden["kat"]
    assert oracle.zlib_compress(b"").hex() == kat["deflate_empty"]
    assert oracle.zlib_compress(b"hello world").hex() == kat["deflate_hello_world"]
    assert oracle.zlib_compress(b"\x12").hex() == kat["deflate_0x12"]
    assert oracle.zlib_compress(b"\x34").hex() == kat["deflate_0x34"]
    assert kat["deflate_empty"] == "789c030000000001"


def test_synth_pinned_to_reference_generator(oracle, golden):
    kat = golden["kat"]
    assert hashlib.sha256(oracle.synth_fp16(524288, 1)).hexdigest() == kat["synth_fp16_524288_1_sha256"]
    assert (hashlib.sha256(oracle.synth_fp16(1000000, 424242)).hexdigest()
            == kat["synth_fp16_1000000_424242_sha256"])


def test_identity_golden_container(oracle):
    # reference tests/test_codec.cpp:76-97
    c = oracle.compress(bytes([0x34, 0x12, 0x78, 0x56]), backend=0, split=True)
    expected = (b"BBC1\x01\x00\x01" + (2).to_bytes(8, "little") * 3 + bytes([0x12, 0x56, 0x34, 0x78]))
    assert c == expected and len(c) == 35
    assert oracle.decompress(c) == bytes([0x34, 0x12, 0x78, 0x56])


def test_oracle_matches_every_golden_container(oracle, golden):
    cache = {}
    for e in golden["entries"]:
        data = cache.get(e["spec"])
        if data is None:
            data = make_input(e["spec"], oracle)
            data = data[: len(data) // 2 * 2]
            cache[e["spec"]] = data
        c = oracle.compress(data, e["backend"], e["split"])
        assert len(c) == e["len"], e
        assert hashlib.sha256(c).hexdigest() == e["sha256"], e
        if "hex" in e:
            assert c.hex() == e["hex"]
        assert oracle.decompress(c) == data


def test_config1_sizes(oracle):
    # high 375,194 B, low 524,454 B, container 899,679 B
    c = oracle.compress(oracle.synth_fp16(524288, 1), 1, True)
    assert len(c) == 899679
    assert int.from_bytes(c[15:23], "little") == 375194
    assert int.from_bytes(c[23:31], "little") == 524454


def test_oracle_vs_live_reference(oracle, reference):
    rng = random.Random(3)
    for trial in range(60):
        n = 2 * rng.randrange(0, 3000)
        data = rng.randbytes(n) if trial % 2 else bytes(rng.choice(b"\x00\x3c\xbc") for _ in range(n))
        for backend in (0, 1):
            for split in (False, True):
                assert oracle.compress(data, backend, split) == reference.compress(data, backend, split)
    s = reference.synth_fp16(4096, 9)
    assert oracle.synth_fp16(4096, 9) == s
    assert oracle.entropy(s) == reference.entropy(s)


def _corpus(seed, count):
    rng = random.Random(seed)
    for i in range(count):
        kind = i % 6
        n = rng.choice([rng.randint(0, 3000), rng.randint(60000, 70000), rng.randint(90000, 140000)])
        if kind == 0:
            yield rng.randbytes(n)
        elif kind == 1:
            yield bytes(rng.choice(b"ab") for _ in range(n))
        elif kind == 2:
            per = rng.randint(1, 300)
            pat = rng.randbytes(per)
            yield (pat * (n // per + 1))[:n]
        elif kind == 3:
            out = bytearray()
            while len(out) < n:
                out += bytes([rng.randrange(4)]) * rng.randint(1, 600)
            yield bytes(out[:n])
        elif kind == 4:
            yield np.random.default_rng(i).integers(0, 64, n, dtype=np.uint8).tobytes()
        else:
            out = bytearray(rng.randbytes(n))
            for _ in range(n // 500):
                d = rng.choice([32506, 32507, 32505, 4096, 4097, 32768, rng.randint(1, 40000)])
                L = rng.randint(3, 300)
                p = rng.randint(0, max(0, n - L - 1))
                if p - d >= 0:
                    out[p:p + L] = out[p - d:p - d + L]
            yield bytes(out)


@pytest.mark.parametrize("profiled", [False, True])
def test_oracle_differential_vs_libz(oracle, profiled):
    for data in _corpus(11, 48):
        assert oracle.zlib_compress(data, profiled=profiled) == zlib.compress(data, 6)


def test_nil_head_after_late_slide(oracle):
    """A chain head exactly MAX_DIST back reads as NIL right after a slide at
    strstart == wsize + MAX_DIST (possible only in the last 262 bytes)."""
    rng = np.random.default_rng(5)
    hits = 0
    for extra in range(10, 262, 4):
        n = 65274 + extra + 1
        d = bytearray(rng.integers(0, 64, n, dtype=np.uint8).tobytes())
        d[32768:32778] = b"XYZABCDEFG"
        d[65274:65284] = b"XYZABCDEFG"
        d = bytes(d)
        hits += int(oracle.match_profile(d)[65274][0]) >> 31
        z = zlib.compress(d, 6)
        assert oracle.zlib_compress(d, profiled=True) == z
        assert oracle.zlib_compress(d) == z
    assert hits > 10


def test_uncompress_error_parity(oracle):
    data = random.Random(1).randbytes(5000)
    z = zlib.compress(data, 6)
    assert oracle.zlib_uncompress(z, len(data)) == data
    assert oracle.zlib_uncompress(z + b"trailing", len(data)) == data  # trailing bytes ignored
    from oracle.oracle import OracleError
    for bad in (z[:-1], z[:10], b"\x78\x9d" + z[2:], bytes([z[0] ^ 1]) + z[1:]):
        with pytest.raises(OracleError):
            oracle.zlib_uncompress(bad, len(data))
    with pytest.raises(OracleError):
        oracle.zlib_uncompress(z, len(data) - 1)
    # uncompress2 with destLen 0 uses a 1-byte scratch buffer
    assert oracle.zlib_uncompress(zlib.compress(b"x"), 0) == b""
    with pytest.raises(OracleError):
        oracle.zlib_uncompress(zlib.compress(b"xy"), 0)


def test_uncompress_fuzz_matches_libz(oracle):
    rng = random.Random(12)
    base = zlib.compress(rng.randbytes(700) + bytes(300), 6)
    for trial in range(1500):
        blob = bytearray(base)
        for _ in range(1 + rng.randrange(6)):
            blob[rng.randrange(len(blob))] ^= 1 << rng.randrange(8)
        blob = bytes(blob)
        try:
            want = zlib.decompress(blob)
            ok = True
        except zlib.error:
            ok = False
        try:
            got = oracle.zlib_uncompress(blob, 1000)
            gok = True
        except Exception:
            gok = False
        if ok and len(want) == 1000:
            assert gok and got == want
        elif not ok:
            assert not gok


def test_oracle_restatement_at_full_config2_size(oracle):
    """The C restatement (oracle/zlib6.c) reproduces the reference's container of a whole config2
    micro-batch (64 MiB bf16, seed 1000): the full-size golden is pinned by two implementations."""
    import hashlib
    import json
    import os

    from paper_2604_21072_b200 import workloads as W
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fullsize_golden.json")))
    (e,) = [g for g in gold["entries"] if g["config"] == "config2" and g["index"] == 0]
    syn = lambda n, s, bf16: oracle.synth_bf16(n, s) if bf16 else oracle.synth_fp16(n, s)  # noqa: E731
    data = W.config2_micro(syn, 0, 0)
    assert hashlib.sha256(data).hexdigest() == e["raw_sha256"]
    c = oracle.compress(data, 1, True)
    assert len(c) == e["len"] == 47056924
    assert hashlib.sha256(c).hexdigest() == e["sha256"]


def test_zlib_hash_keeps_all_of_a_trigram_but_z():
    """K4G's k_gram4 compares chain candidates by z = the top three bits of bytes 0-2 (+ byte 3)
    instead of the bytes themselves.  That is exact because zlib's 15-bit hash
    ((b0 << 10) ^ (b1 << 5) ^ b2) & 0x7fff, with z, determines the 3-gram: every entry of a
    position's chain has its hash, so on a chain "same 3-gram" is "same z"."""
    import numpy as np
    b = np.arange(1 << 24, dtype=np.uint32)
    b0, b1, b2 = b & 0xff, (b >> 8) & 0xff, b >> 16
    h = ((b0 << 10) ^ (b1 << 5) ^ b2) & 0x7fff
    z = (b0 >> 5) | ((b1 >> 5) << 3) | ((b2 >> 5) << 6)
    key = (h << 9) | z  # injective on all 2^24 trigrams iff (hash, z) determines the trigram
    assert np.unique(key).size == 1 << 24
