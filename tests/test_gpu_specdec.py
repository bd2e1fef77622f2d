"""GPU parity for the packed speculative-decoding payload path.

The device packer (bb_pack_sd: keep-mask scan + warp-per-row gather) must write
exactly the reference's encode_packed(pack(kept rows per request)) bytes
(specdec.cpp:153-165,192-198; golden SHA-256 from the reference), and the GPU
codec must turn them into the reference's BBC1 container.  bb_unpack_sd must
reproduce decode_packed's CorruptOffsets decisions (specdec.cpp:200-220).
"""
import hashlib
import json
import os

import numpy as np
import pytest

from inputs import sd_tree

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "specdec_golden.json")))


@pytest.fixture(scope="module")
def dev():
    import torch
    assert torch.cuda.is_available()
    from paper_2604_21072_b200 import codec, specdec
    return torch, specdec.DevicePacker(0), codec.DeviceCodec(0)


def _upload(torch, spec):
    rows, keep, request_rows, per = sd_tree(spec)
    dim = int(spec.split(":")[3])
    r = torch.from_numpy(rows.reshape(-1, dim).copy()).cuda()
    k = torch.from_numpy(keep.copy()).cuda()
    return r, k, request_rows, per, dim


@pytest.mark.parametrize("entry", GOLD["entries"], ids=lambda e: e["spec"])
def test_device_pack_and_compress_match_reference(dev, entry):
    torch, packer, codec = dev
    r, k, request_rows, _, dim = _upload(torch, entry["spec"])
    packed = packer.pack_encode(r, k, request_rows)
    b = packed.cpu().numpy().tobytes()
    assert len(b) == entry["packed_len"]
    assert hashlib.sha256(b).hexdigest() == entry["packed_sha256"]
    c = codec.compress(packed).cpu().numpy().tobytes()
    assert len(c) == entry["container_len"]
    assert hashlib.sha256(c).hexdigest() == entry["container_sha256"]
    # round trip on the device: decompress -> open -> rows equal the kept rows, bit for bit
    back = codec.decompress(codec.compress(packed))
    offsets, payload = packer.open(back, dim)
    assert offsets == [int(x) for x in np.cumsum([0] + [int(k[request_rows[i]:request_rows[i + 1]].sum())
                                                        for i in range(len(request_rows) - 1)])]
    want = r[k.bool()]
    assert torch.equal(payload.view(torch.int32), want.view(torch.int32))


@pytest.mark.parametrize("case", GOLD["decode_cases"], ids=lambda c: c["name"])
def test_device_open_matches_decode_packed(dev, case):
    torch, packer, _ = dev
    from paper_2604_21072_b200.codec import CorruptOffsets
    data = bytes.fromhex(case["hex"])
    t = torch.tensor(list(data) or [0], dtype=torch.uint8, device="cuda")[:len(data)]
    if case["status"]:
        with pytest.raises(CorruptOffsets) as e:
            packer.open(t, case["hidden_dim"])
        assert str(e.value) == case["message"]
    else:
        offsets, payload = packer.open(t, case["hidden_dim"])
        assert offsets == list(np.frombuffer(data, "<u4", count=len(offsets), offset=4))
        assert payload.numel() == offsets[-1] * case["hidden_dim"]


def test_edge_batches(dev):
    torch, packer, _ = dev
    from paper_2604_21072_b200 import specdec as sd
    # no requests; requests with no rows; nothing kept; hidden_dim 0
    z = torch.zeros((0, 4), dtype=torch.float32, device="cuda")
    zk = torch.zeros(0, dtype=torch.uint8, device="cuda")
    assert packer.pack_encode(z, zk, [0]).cpu().numpy().tobytes() == sd.encode_packed(sd.pack([]))
    assert packer.pack_encode(z, zk, [0, 0, 0]).cpu().numpy().tobytes() == sd.encode_packed(sd.pack([[], []]))
    r = torch.randn(10, 3, device="cuda")
    none = torch.zeros(10, dtype=torch.uint8, device="cuda")
    assert packer.pack_encode(r, none, [0, 4, 10]).cpu().numpy().tobytes() == \
        sd.encode_packed(sd.PackedBatch(3, np.zeros(0, np.float32), [0, 0, 0]))
    e = torch.zeros((5, 0), dtype=torch.float32, device="cuda")
    ones = torch.ones(5, dtype=torch.uint8, device="cuda")
    got = packer.pack_encode(e, ones, [0, 2, 5]).cpu().numpy().tobytes()
    assert got == sd.encode_packed(sd.PackedBatch(0, np.zeros(0, np.float32), [0, 2, 5]))
    with pytest.raises(ValueError):  # request ranges out of order
        packer.pack_encode(r, ones[:1].expand(10).contiguous(), [0, 6, 4])


def test_packed_sd_frames_roundtrip(dev):
    torch, packer, codec = dev
    from paper_2604_21072_b200 import pipeline as pl
    r, k, request_rows, _, dim = _upload(torch, "sdtree:4:64:512:31:55:bf16up")
    packed = packer.pack_encode(r, k, request_rows)
    frames = pl.build_frames([codec.compress(packed)], batch_id=3, flags=3, device=r.device,
                             msg_type=pl.T_PACKED_SD)
    meta, payloads = pl.open_frames(frames)
    assert meta == [(pl.T_PACKED_SD, 3, 0, 3)]
    offsets, payload = packer.open(codec.decompress(payloads[0]), dim)
    assert torch.equal(payload.view(torch.int32), r[k.bool()].view(torch.int32))
