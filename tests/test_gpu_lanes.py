"""GPU parity for K1/K2 (split, merge, identity container, histogram) through the C ABI."""
import hashlib
import random

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


def test_split_kat(codec):
    lanes = codec.byte_split(bytes([0x34, 0x12, 0x78, 0x56]))
    assert lanes.high == bytes([0x12, 0x56]) and lanes.low == bytes([0x34, 0x78])
    assert codec.byte_merge(lanes.high, lanes.low) == bytes([0x34, 0x12, 0x78, 0x56])
    with pytest.raises(codec.OddLength):
        codec.byte_split(b"\x01")
    with pytest.raises(codec.LaneLengthMismatch):
        codec.byte_merge(b"\x01", b"")


def test_split_merge_ragged_sizes(codec, oracle):
    rng = random.Random(5)
    for n in list(range(0, 70, 2)) + [2 * rng.randrange(1, 40000) for _ in range(20)]:
        s = rng.randbytes(n)
        lanes = codec.byte_split(s)
        assert lanes.high == s[1::2] and lanes.low == s[0::2]
        assert codec.byte_merge(lanes.high, lanes.low) == s


def test_identity_containers_match_golden(codec, golden, oracle):
    cache = {}
    for e in golden["entries"]:
        if e["backend"] != 0:
            continue
        data = cache.setdefault(e["spec"], make_input(e["spec"], oracle))
        data = data[: len(data) // 2 * 2]
        c = codec.compress_serialized(data, 0, e["split"])
        assert len(c) == e["len"] and hashlib.sha256(c).hexdigest() == e["sha256"], e
        assert codec.decompress_serialized(c) == data


def test_identity_golden_bytes(codec):
    c = codec.compress_serialized(bytes([0x34, 0x12, 0x78, 0x56]), 0, True)
    assert c.hex() == "4242433101000102000000000000000200000000000000020000000000000012563478"


def test_histogram_and_entropy(codec, oracle):
    rng = np.random.default_rng(3)
    for n in (0, 1, 15, 16, 17, 1000, 1 << 20, (1 << 20) + 7):
        d = rng.integers(0, 23, n, dtype=np.uint8).tobytes()
        assert codec.histogram256(d) == np.bincount(np.frombuffer(d, np.uint8), minlength=256).tolist()
        assert codec.entropy_bits_per_byte(d) == oracle.entropy(d)


def test_device_identity_unaligned(codec, oracle):
    import torch
    dev = codec.DeviceCodec(0)
    data = oracle.synth_fp16(100003, 4)
    for off in (0, 1, 2, 3, 7, 13):
        base = torch.frombuffer(bytearray(bytes(off) + data + b"\0" * 64), dtype=torch.uint8).cuda()
        x = base[off: off + len(data)]
        for split in (True, False):
            c = dev.compress(x, backend=0, split=split)
            assert c.cpu().numpy().tobytes() == oracle.compress(data, 0, split)
            out = torch.zeros(len(data) + 32, dtype=torch.uint8, device="cuda")
            n = dev.decompress_into(c, out[off:])
            assert n == len(data) and out[off:off + n].cpu().numpy().tobytes() == data


def test_large_identity_roundtrip(codec, oracle):
    import torch
    dev = codec.DeviceCodec(0)
    x = torch.randint(0, 256, (64 << 20,), dtype=torch.uint8, device="cuda")
    c = dev.compress(x, backend=0, split=True)
    assert torch.equal(c[31:31 + (32 << 20)], x[1::2])
    assert torch.equal(dev.decompress(c), x)
