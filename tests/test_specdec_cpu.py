"""Packed speculative-decoding payloads: host mirror vs the reference (CPU only).

Golden data: tests/golden/specdec_golden.json, generated from the unmodified reference
specdec.cpp (tests/golden/make_specdec_golden.py).  Cases follow the reference's
tests/test_specdec.cpp pack/unpack/encode_packed/decode_packed list.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from inputs import sd_tree
from paper_2604_21072_b200 import specdec as sd
from paper_2604_21072_b200.codec import CorruptOffsets, DimMismatch

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "specdec_golden.json")))


def test_pack_offsets_prefix_sums():
    b = sd.pack([[[1.0, 2.0]] * 3, [[3.0, 4.0]], [[5.0, 6.0]] * 2])
    assert b.offsets == [0, 3, 4, 6] and b.hidden_dim == 2 and b.total_states() == 6
    assert b.request_count() == 3
    assert sd.encode_packed(b).hex() == GOLD["pack_offsets_0346"]


def test_pack_ragged_dims_raise_dim_mismatch():
    with pytest.raises(DimMismatch) as e:
        sd.pack([[[1.0, 2.0]], [[1.0, 2.0, 3.0]]])
    assert GOLD["pack_ragged_status"] == 9 and str(e.value) == GOLD["pack_ragged_message"]


@pytest.mark.parametrize("case", GOLD["unpack_checks"], ids=lambda c: str(c["offsets"]))
def test_unpack_checks_match_reference(case):
    b = sd.PackedBatch(case["hidden_dim"], np.zeros(case["payload"], np.float32), list(case["offsets"]))
    if case["status"]:
        with pytest.raises(CorruptOffsets):
            sd.unpack(b)
    else:
        sd.unpack(b)


@pytest.mark.parametrize("case", GOLD["decode_cases"], ids=lambda c: c["name"])
def test_decode_packed_matches_reference(case):
    data = bytes.fromhex(case["hex"])
    if case["status"]:
        with pytest.raises(CorruptOffsets) as e:
            sd.decode_packed(data, case["hidden_dim"])
        assert str(e.value) == case["message"]
    else:
        assert sd.encode_packed(sd.decode_packed(data, case["hidden_dim"])) == data


@pytest.mark.parametrize("entry", [e for e in GOLD["entries"] if e["packed_len"] < 200000],
                         ids=lambda e: e["spec"])
def test_host_pack_matches_reference_bytes(entry):
    _, _, _, per_request = sd_tree(entry["spec"])
    packed = sd.encode_packed(sd.pack(per_request))
    assert len(packed) == entry["packed_len"]
    assert hashlib.sha256(packed).hexdigest() == entry["packed_sha256"]
    dim = int(entry["spec"].split(":")[3])
    b = sd.decode_packed(packed, dim)
    again = sd.unpack(b)
    assert [len(r) for r in again] == [len(r) for r in per_request]
    for got, want in zip(again, per_request):
        for g, w in zip(got, want):
            assert g.tobytes() == w.tobytes()  # bit-exact incl. NaN payloads / -0


def test_random_ragged_identity():
    rng = np.random.default_rng(11)
    per = [[rng.standard_normal(5).astype(np.float32) for _ in range(int(rng.integers(0, 6)))]
           for _ in range(20)]
    b = sd.pack(per)
    out = sd.unpack(sd.decode_packed(sd.encode_packed(b), 5))
    assert all(np.array_equal(x, y) for r1, r2 in zip(per, out) for x, y in zip(r1, r2))


def test_live_reference_pack(reference):
    for spec in ("sdtree:3:4:3:2:70:f32", "sdtree:4:9:5:8:100:special", "sdtree:6:5:2:21:40:f32"):
        _, _, _, per = sd_tree(spec)
        assert sd.encode_packed(sd.pack(per)) == reference.pack_encode(per)
