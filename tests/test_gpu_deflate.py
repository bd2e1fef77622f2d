"""GPU parity for the zlib-exact deflate backend (K3-K7) through the C ABI.

Bit-exact: every compressed byte must equal the reference codec's output
(golden SHA-256 from the reference itself) and zlib 1.3 level 6 (Python's zlib
is the same system libz).  K3/K4 intermediates are checked against the oracle's
decomposition (oracle/zlib6.c) so a mismatch is localised to one kernel.
"""
import ctypes as C
import hashlib
import random
import zlib

import numpy as np
import pytest
from inputs import make_input

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def codec():
    import torch
    assert torch.cuda.is_available()
    from paper_2604_21072_b200 import codec as c
    return c


def _corpus():
    rng = random.Random(21)
    yield b""
    yield b"\x00"
    yield b"ab"
    yield b"hello world"
    yield bytes(300)
    yield b"\x42" * 65536
    for n in (258, 259, 262, 1000, 4096, 16383, 32506, 32768, 65273, 65274, 65275, 65536, 70000,
              131072, 200000):
        yield rng.randbytes(n)
        yield bytes(rng.choice(b"ab") for _ in range(n))
        yield np.random.default_rng(n).integers(0, 64, n, dtype=np.uint8).tobytes()
    for per in (1, 2, 3, 7, 258, 300):
        pat = rng.randbytes(per)
        yield (pat * (150000 // per + 1))[:150000]
    # hash heads exactly MAX_DIST (32506) back: zlib compares the head before its
    # limit test, so these matches must be found (one head per K4 segment phase)
    # (background from a 4-symbol alphabet, chunk from bytes 128-255: the chunk's
    # 3-grams have no other occurrence, so the head is exactly the first copy)
    for at in (100, 16000, 40000):
        buf = bytearray(rng.choice(b"\x00\x01\x02\x03") for _ in range(at + 32506 + 5000))
        buf[at:at + 24] = bytes(rng.randrange(128, 256) for _ in range(24))
        buf[at + 32506:at + 32506 + 24] = buf[at:at + 24]
        yield bytes(buf)


@pytest.mark.parametrize("walk", ["k4g", "classic"])
def test_hash_prev_and_profiles_match_oracle(codec, oracle, walk, monkeypatch):
    """K3 links and K4 profiles (both walks: K4G's 4-gram subsequence, K4's full chain walk)
    against the oracle's decomposition."""
    import torch
    if walk == "classic":
        monkeypatch.setenv("BB_K4_CLASSIC", "1")
    else:
        monkeypatch.delenv("BB_K4_CLASSIC", raising=False)
    from paper_2604_21072_b200 import _lib
    L = _lib.load()
    fn = L.bb_debug_hash_prev_profile
    fn.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p]
    rng = np.random.default_rng(11)
    inputs = [oracle.synth_fp16(100000, 1)[1::2], oracle.synth_bf16(120000, 2)[1::2],
              oracle.synth_bf16(300000, 5)[1::2], oracle.synth_fp16(200000, 4)[0::2],
              random.Random(1).randbytes(70000), b"\x07" * 40000, b"ab" * 30000 + b"c" * 5,
              np.random.default_rng(3).integers(0, 4, 90000, dtype=np.uint8).tobytes(),
              rng.integers(0, 2, 70000, dtype=np.uint8).tobytes(),
              bytes(rng.integers(0, 3, 50, dtype=np.uint8)) * 2000,  # periodic: long matches
              bytes(range(256)) * 300, b"xyz", b"ab"]
    for data in inputs:
        x = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
        pd = torch.zeros(len(data), dtype=torch.int16, device="cuda")
        prof = torch.zeros(2 * len(data), dtype=torch.int32, device="cuda")
        rc = fn(x.data_ptr(), len(data), pd.data_ptr(), prof.data_ptr(),
                torch.cuda.current_stream().cuda_stream)
        assert rc == 0, _lib.last_error()
        want_pd = oracle.hash_prev(data)
        got_pd = pd.cpu().numpy().view(np.uint16)
        bad = np.nonzero(got_pd != want_pd)[0]
        assert bad.size == 0, f"pd mismatch at {bad[:5]}: {got_pd[bad[:5]]} vs {want_pd[bad[:5]]}"
        want = oracle.match_profile(data)
        got = prof.cpu().numpy().view(np.uint32).reshape(-1, 2)
        bad = np.nonzero((got != want).any(axis=1))[0]
        assert bad.size == 0, f"profile mismatch at {bad[:5]}: {got[bad[:5]]} vs {want[bad[:5]]}"


def test_sorted_chain_profiles_match_oracle(codec, oracle):
    """K3S + K4S (bucket-sorted chains, the default encoder path) give the oracle's profiles
    bit for bit: chain budgets 32 / 128, distance rules, nice_match, first maximum, long matches."""
    import torch
    from paper_2604_21072_b200 import _lib
    L = _lib.load()
    fn = L.bb_debug_profile_sorted
    fn.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]
    rng = np.random.default_rng(11)
    inputs = [oracle.synth_fp16(100000, 1)[1::2], oracle.synth_bf16(120000, 2)[1::2],
              oracle.synth_bf16(300000, 5)[1::2], oracle.synth_fp16(200000, 4)[0::2],
              random.Random(1).randbytes(70000), b"\x07" * 40000, b"ab" * 30000 + b"c" * 5,
              rng.integers(0, 4, 90000, dtype=np.uint8).tobytes(),
              rng.integers(0, 2, 70000, dtype=np.uint8).tobytes(),
              bytes(rng.integers(0, 3, 50, dtype=np.uint8)) * 2000,  # periodic: long matches
              b"xyz", b"ab", b"", bytes(range(256)) * 300]
    for data in inputs:
        if not data:
            continue
        x = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
        prof = torch.zeros(2 * len(data), dtype=torch.int32, device="cuda")
        rc = fn(x.data_ptr(), len(data), prof.data_ptr(), torch.cuda.current_stream().cuda_stream)
        assert rc == 0, _lib.last_error()
        want = oracle.match_profile(data)
        got = prof.cpu().numpy().view(np.uint32).reshape(-1, 2)
        bad = np.nonzero((got != want).any(axis=1))[0]
        assert bad.size == 0, f"{len(data)} B: profile mismatch at {bad[:5]}: {got[bad[:5]]} vs {want[bad[:5]]}"


def test_lane_encode_matches_zlib(codec):
    enc = codec.backend_by_id(codec.kBackendDeflate).encode
    for data in _corpus():
        got = enc(data)
        want = zlib.compress(data, 6)
        assert got == want, (len(data), len(got), len(want))


def test_deflate_containers_match_golden(codec, golden, oracle):
    cache = {}
    for e in golden["entries"]:
        if e["backend"] != 1:
            continue
        data = cache.setdefault(e["spec"], make_input(e["spec"], oracle))
        data = data[: len(data) // 2 * 2]
        c = codec.compress_serialized(data, 1, e["split"])
        assert len(c) == e["len"], (e["spec"], e["split"], len(c), e["len"])
        assert hashlib.sha256(c).hexdigest() == e["sha256"], e


def test_config1_kat(codec, oracle):
    stream = oracle.synth_fp16(524288, 1)
    c = codec.compress(stream, codec.kBackendDeflate, True)
    assert len(c.high_blob) == 375194 and len(c.low_blob) == 524454
    assert len(codec.serialize_container(c)) == 899679


def test_batch_compress_matches_single(codec, oracle):
    import torch
    dev = codec.DeviceCodec(0)
    streams = [oracle.synth_fp16(n, s) for n, s in ((1, 1), (5000, 2), (70001, 3), (0, 4), (131072, 5))]
    streams += [oracle.synth_bf16(90000, 6)]
    xs = [torch.frombuffer(bytearray(s + b"\0"), dtype=torch.uint8)[: len(s)].cuda() for s in streams]
    outs = [torch.zeros(dev.compress_bound(len(s)), dtype=torch.uint8, device="cuda") for s in streams]
    lens = dev.compress_batch(xs, outs)
    for s, o, n in zip(streams, outs, lens):
        assert o[:n].cpu().numpy().tobytes() == oracle.compress(s, 1, True)


def test_lane_decode_roundtrip_and_foreign_streams(codec):
    dec = codec.backend_by_id(codec.kBackendDeflate).decode
    for data in _corpus():
        for level in (6, 1, 9, 0):
            blob = zlib.compress(data, level)
            assert dec(blob, len(data)) == data
        assert dec(zlib.compress(data, 6) + b"trailing", len(data)) == data


def test_decode_error_parity_with_oracle(codec, oracle):
    from oracle.oracle import OracleError
    dec = codec.backend_by_id(codec.kBackendDeflate).decode
    rng = random.Random(12)
    base = zlib.compress(rng.randbytes(700) + bytes(300), 6)
    for trial in range(400):
        blob = bytearray(base)
        for _ in range(1 + rng.randrange(6)):
            blob[rng.randrange(len(blob))] ^= 1 << rng.randrange(8)
        if trial % 7 == 0:
            blob = blob[: rng.randrange(len(blob) + 1)]
        blob = bytes(blob)
        expected = 1000 if trial % 5 else rng.choice([0, 1, 999, 1001])
        try:
            want = oracle.zlib_uncompress(blob, expected)
            want_ok = len(want) == expected
        except OracleError:
            want_ok = False
        try:
            got = dec(blob, expected)
            got_ok = True
        except codec.CorruptContainer:
            got_ok = False
        assert got_ok == want_ok, (trial, expected)
        if got_ok:
            assert got == want


def test_container_roundtrip_golden_inputs(codec, golden, oracle):
    cache = {}
    for e in golden["entries"]:
        if e["backend"] != 1 or e["len"] > 3_000_000:
            continue
        data = cache.setdefault(e["spec"], make_input(e["spec"], oracle))
        data = data[: len(data) // 2 * 2]
        c = oracle.compress(data, 1, e["split"])
        assert codec.decompress_serialized(c) == data


def _inflate_counts():
    from paper_2604_21072_b200 import _lib
    L = _lib.load()
    out = (C.c_uint64 * 3)()
    L.bb_debug_inflate_counts(out)
    return list(out)


def test_parallel_inflate_large_streams(codec, oracle):
    """Streams >= 64 KiB take the parallel decoder; it must validate them itself
    (no silent fallback) and reproduce the input exactly."""
    dec = codec.backend_by_id(codec.kBackendDeflate).decode
    cases = [oracle.synth_fp16(600000, 1)[1::2], oracle.synth_fp16(600000, 1)[0::2],
             oracle.synth_bf16(700000, 2)[1::2], oracle.synth_bf16(300000, 3),
             np.random.default_rng(4).integers(0, 64, 500000, dtype=np.uint8).tobytes(),
             random.Random(5).randbytes(300000), b"\x42" * 400000,
             make_input("runs:400000:6"), make_input("period:300000:7:300")]
    for data in cases:
        for level in (6, 1, 9):
            blob = zlib.compress(data, level)
            if len(blob) < (1 << 16):
                continue
            before = _inflate_counts()
            assert dec(blob, len(data)) == data
            after = _inflate_counts()
            assert after[0] == before[0] + 1, (len(data), level, before, after)


def test_parallel_inflate_rejects_corruption(codec, oracle):
    from oracle.oracle import OracleError
    dec = codec.backend_by_id(codec.kBackendDeflate).decode
    data = oracle.synth_bf16(200000, 8)
    base = zlib.compress(data, 6)
    rng = random.Random(9)
    for trial in range(40):
        blob = bytearray(base)
        for _ in range(1 + rng.randrange(4)):
            blob[rng.randrange(len(blob))] ^= 1 << rng.randrange(8)
        blob = bytes(blob)
        try:
            want_ok = len(oracle.zlib_uncompress(blob, len(data))) == len(data)
        except OracleError:
            want_ok = False
        try:
            got = dec(blob, len(data))
            assert got == data or want_ok
            got_ok = True
        except codec.CorruptContainer:
            got_ok = False
        assert got_ok == want_ok


def _structured(rng, n):
    """Random mixture of the structures the level-6 rules branch on: small and large
    alphabets, runs, copies at distances around MAX_DIST (32506) and WSIZE, copies
    longer than MAX_MATCH (258) and nice_length (128), near-matches that differ in one
    byte (first-maximum ties), and text from this repo's own sources."""
    import glob
    import os
    text = b"".join(open(f, "rb").read() for f in sorted(glob.glob(
        os.path.join(os.path.dirname(__file__), "*.py"))))
    out = bytearray()
    while len(out) < n:
        kind = rng.randrange(7)
        m = rng.randrange(1, 3000)
        if kind == 0:
            out += rng.randbytes(m)
        elif kind == 1:
            k = rng.choice((2, 3, 4, 16))
            out += bytes(rng.randrange(k) for _ in range(m))
        elif kind == 2:
            out += bytes([rng.randrange(256)]) * m
        elif kind in (3, 4) and out:
            d = rng.choice((1, 2, 3, 257, 258, 259, 4096, 32505, 32506, 32507, 32768,
                            rng.randrange(1, 40000)))
            d = min(d, len(out))
            ln = rng.choice((3, 4, 127, 128, 129, 258, 259, 600, m))
            src = len(out) - d
            for i in range(ln):
                out.append(out[src + i])
            if kind == 4 and ln > 4:
                out[-rng.randrange(1, ln)] ^= 1 << rng.randrange(8)
        else:
            s = rng.randrange(max(1, len(text) - m))
            out += text[s:s + m]
    return bytes(out[:n])


def test_lane_encode_structured_fuzz(codec):
    enc = codec.backend_by_id(codec.kBackendDeflate).encode
    dec = codec.backend_by_id(codec.kBackendDeflate).decode
    rng = random.Random(2604)
    for trial in range(40):
        n = rng.choice((rng.randrange(1, 5000), rng.randrange(5000, 80000), rng.randrange(80000, 400000)))
        data = _structured(rng, n)
        got = enc(data)
        want = zlib.compress(data, 6)
        assert got == want, (trial, n, len(got), len(want))
        assert dec(got, n) == data, (trial, n)


def test_parallel_inflate_long_copy_chains(codec):
    """Copy chains that run back across hundreds of 32 KiB resolution windows (periods of
    7 B to 30 KB repeated for MiBs, with sparse literals) take the pointer-doubling rounds
    before the chase; the output must still be exact, and corruption still caught."""
    dec = codec.backend_by_id(codec.kBackendDeflate).decode
    rng = random.Random(77)
    for period, n, lit in ((4096, 4 << 20, 8), (30000, 6 << 20, 8), (7, 4 << 20, 6)):
        buf = bytearray((rng.randbytes(period) * (n // period + 1))[:n])
        for _ in range(n >> lit):  # sparse literals break some chains part-way
            buf[rng.randrange(n)] = rng.randrange(256)
        data = bytes(buf)
        blob = zlib.compress(data, 6)
        assert len(blob) >= 1 << 16  # the parallel decoder's range
        before = _inflate_counts()
        assert dec(blob, n) == data, (period, n)
        assert _inflate_counts()[0] == before[0] + 1
        bad = bytearray(blob)
        bad[len(bad) // 2] ^= 0x10
        with pytest.raises(codec.CorruptContainer):
            dec(bytes(bad), n)


def test_parallel_inflate_checks_the_zlib_header(codec, oracle):
    """lanes of >= 64 KiB take the parallel inflate, which starts decoding at bit 16; a bad
    CMF / FLG (FCHECK, CM != 8, CINFO > 7, FDICT set with a valid FCHECK) must still be rejected, as
    zlib's uncompress does (inflate.c HEAD state; reference codec.cpp:27-38)."""
    from oracle.oracle import OracleError
    dec = codec.backend_by_id(codec.kBackendDeflate).decode
    data = oracle.synth_bf16(300000, 12)
    base = bytearray(zlib.compress(data, 6))
    assert len(base) >= 1 << 16 and bytes(base[:2]) == b"\x78\x9c"

    def fcheck(cmf, flg_hi):  # FLG with FCHECK making (CMF * 256 + FLG) % 31 == 0
        flg = flg_hi & 0xe0
        return flg | (31 - ((cmf << 8) | flg) % 31) % 31

    cases = {
        "fcheck": (0x78, 0x9d),
        "cm": (0x77, fcheck(0x77, 0x80)),
        "cinfo": (0x88, fcheck(0x88, 0x80)),
        "fdict": (0x78, fcheck(0x78, 0xa0)),
    }
    for name, (cmf, flg) in cases.items():
        blob = bytes([cmf, flg]) + bytes(base[2:])
        with pytest.raises(OracleError):
            oracle.zlib_uncompress(blob, len(data))
        with pytest.raises(zlib.error):  # the pinned system zlib agrees
            zlib.decompress(blob)
        with pytest.raises(codec.CorruptContainer):
            dec(blob, len(data))
    assert dec(bytes(base), len(data)) == data


def test_sequential_inflate_on_large_streams(codec, oracle, monkeypatch):
    """The exact sequential decoder (the fallback that defines uncompress() status) on streams
    the parallel path would normally take: CTA-copied stored blocks longer than the 32 KiB window,
    matches reaching exactly 32768 back through the shared-memory window, mixed block types,
    and corruption status parity with the oracle."""
    from oracle.oracle import OracleError
    dec = codec.backend_by_id(codec.kBackendDeflate).decode
    monkeypatch.setenv("BB_INFLATE_SEQ", "1")
    rng = random.Random(31)
    far = bytearray(rng.choice(b"\x00\x01\x02\x03") for _ in range(32768 + 40000))
    far[1000:1030] = bytes(rng.randrange(128, 256) for _ in range(30))
    far[1000 + 32768:1030 + 32768] = far[1000:1030]  # a match exactly 32768 back
    cases = [random.Random(5).randbytes(300000), oracle.synth_bf16(200000, 3),
             oracle.synth_fp16(150000, 2)[1::2], b"\x42" * 200000, bytes(far),
             random.Random(6).randbytes(70000) + b"\x07" * 70000 + random.Random(7).randbytes(70000)]
    before = _inflate_counts()
    for data in cases:
        for level in (0, 1, 6, 9):
            blob = zlib.compress(data, level)
            assert dec(blob, len(data)) == data, (len(data), level)
            assert dec(blob + b"tail", len(data)) == data
    after = _inflate_counts()
    assert after[0] == before[0], "BB_INFLATE_SEQ must keep every stream on the sequential decoder"
    # status parity on corrupted large streams (stored and compressed blocks)
    for trial in range(24):
        data = cases[trial % 3]
        blob = bytearray(zlib.compress(data, (0, 6)[trial % 2]))
        for _ in range(1 + rng.randrange(4)):
            blob[rng.randrange(len(blob))] ^= 1 << rng.randrange(8)
        if trial % 5 == 0:
            blob = blob[: rng.randrange(len(blob) + 1)]
        blob = bytes(blob)
        expected = len(data) if trial % 6 else rng.choice([0, len(data) - 1, len(data) + 1])
        try:
            want = oracle.zlib_uncompress(blob, expected)
            want_ok = len(want) == expected
        except OracleError:
            want_ok = False
        try:
            got = dec(blob, expected)
            got_ok = True
        except codec.CorruptContainer:
            got_ok = False
        assert got_ok == want_ok, (trial, expected)
        if got_ok:
            assert got == want


@pytest.mark.parametrize("walk", ["BB_K4G", "BB_K4_CLASSIC"])
def test_forced_k4_walk_matches_zlib(codec, walk, monkeypatch):
    """Either K4 walk forced for every lane (the default picks one per lane from sampled chain
    statistics) gives zlib's bytes, on lanes large enough for the selection to matter."""
    monkeypatch.setenv(walk, "1")
    enc = codec.backend_by_id(codec.kBackendDeflate).encode
    from paper_2604_21072_b200 import synth as S
    cases = [S.gaussian(1 << 20, 3, True)[1::2], S.gaussian(1 << 20, 4, False)[1::2],
             S.gaussian(600000, 5, True), np.random.default_rng(6).integers(0, 3, 1 << 20, dtype=np.uint8).tobytes()]
    for data in cases:
        assert enc(data) == zlib.compress(data, 6), (walk, len(data))
