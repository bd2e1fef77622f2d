"""Byte parity at the FULL BASELINE.json config sizes (GPU).

Every container the bench's workloads produce is compared, by SHA-256, with the reference's
container on the same input (tests/golden/fullsize_golden.json, generated here by
tests/golden/make_fullsize_golden.py from oracle/_ref = the unmodified
/root/reference/proj/src/codec.cpp:163-179 + zlib 1.3 compress2 level 6, codec.cpp:17-25).
The inputs are rebuilt on the GPU box from the recipes in paper_2604_21072_b200/workloads.py
(their SHA-256s are pinned too), and every container is decoded back on the device.
"""
from __future__ import annotations

import hashlib
import json
import os
from concurrent.futures import ThreadPoolExecutor

import pytest

from paper_2604_21072_b200 import workloads as W

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "fullsize_golden.json")))["entries"]

pytestmark = pytest.mark.gpu


def _synth(n, seed, bf16):
    from paper_2604_21072_b200 import synth
    return synth.gaussian(n, seed, bf16)


def _pool(fn, items):
    with ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 1)) as ex:
        return list(ex.map(fn, items))


def _sha(t) -> str:
    return hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()


def _entries(config):
    return [e for e in GOLD if e["config"] == config]


def _roundtrip(dev, host_inputs, entries, group=8):
    """compress_batch on the device in groups; compare every container and decode it back."""
    import torch
    assert len(host_inputs) == len(entries)
    bad = []
    for g in range(0, len(host_inputs), group):
        hs, es = host_inputs[g:g + group], entries[g:g + group]
        for h, e in zip(hs, es):
            assert len(h) == e["raw_len"] and hashlib.sha256(h).hexdigest() == e["raw_sha256"], e["name"]
        xs = [torch.frombuffer(bytearray(h), dtype=torch.uint8).cuda() for h in hs]
        outs = [torch.empty(dev.compress_bound(x.numel()), dtype=torch.uint8, device="cuda") for x in xs]
        lens = dev.compress_batch(xs, outs)
        cs = [o[:n] for o, n in zip(outs, lens)]
        for c, e in zip(cs, es):
            if c.numel() != e["len"] or _sha(c) != e["sha256"]:
                bad.append((e["name"], int(c.numel()), e["len"]))
        decs = [torch.empty_like(x) for x in xs]
        dev.decompress_batch(cs, decs)
        torch.cuda.synchronize()
        for d, x, e in zip(decs, xs, es):
            assert torch.equal(d, x), f"round trip {e['name']}"
        del xs, outs, cs, decs
        torch.cuda.empty_cache()
    assert not bad, bad


@pytest.fixture(scope="module")
def dev():
    from paper_2604_21072_b200 import codec
    return codec.DeviceCodec(0)


def test_config1_container_matches_reference(dev):
    es = _entries("config1")
    _roundtrip(dev, [_synth(W.C1_ELEMS, 1, False)], es)


def test_config2_all_micro_batches_match_reference(dev):
    """The bench's timed step at N=1: 8 x 64 MiB bf16 micro-batches (seeds 1000..1007)."""
    es = _entries("config2")
    assert len(es) == W.C2_MICRO
    hs = _pool(lambda e: W.config2_micro(_synth, e["rank"], e["index"]), es)
    _roundtrip(dev, hs, es, group=8)


def test_config4_kv_layer_matches_reference(dev):
    """All 64 KV chunks (40 MiB each, 2.5 GiB) of the bench's layer 0."""
    es = _entries("config4")
    assert [e["chunk_id"] for e in es] == W.kv_layer_ids(0)
    for g in range(0, len(es), 16):
        part = es[g:g + 16]
        hs = _pool(lambda e: W.kv_chunk(_synth, e["chunk_id"]), part)
        _roundtrip(dev, hs, part, group=16)


def test_config3_packed_step_matches_reference(dev):
    """32 token trees packed ON THE DEVICE into encode_packed's layout, then compressed: the image and
    the container both equal the reference's (specdec.cpp:153-198 + codec.cpp:163-179)."""
    import numpy as np
    import torch

    from paper_2604_21072_b200 import specdec
    (e,) = _entries("config3")
    reqs = _pool(lambda r: W.sd_request(_synth, r), range(e["first_request"], e["first_request"] + e["requests"]))
    rows = torch.from_numpy(np.concatenate([s for s, _ in reqs])).cuda()
    keep = torch.from_numpy(np.concatenate([k for _, k in reqs])).cuda()
    req_rows = [i * W.SD_NODES for i in range(e["requests"] + 1)]
    img = specdec.DevicePacker(0).pack_encode(rows, keep, req_rows)
    assert img.numel() == e["raw_len"] and _sha(img) == e["raw_sha256"]
    c = dev.compress(img)
    assert c.numel() == e["len"] and _sha(c) == e["sha256"]
    back = dev.decompress(c)
    torch.cuda.synchronize()
    assert torch.equal(back, img)


@pytest.mark.parametrize("size_mib", [1, 4, 16, 64, 256, 1024])
def test_config5_sweep_matches_reference(dev, size_mib):
    """d=8192 fp16 sweep tensors; the 1 GiB tensor travels as two 512 MiB frames (wire.cpp:31)."""
    es = [e for e in _entries("config5") if e["tensor_bytes"] == size_mib * W.MiB]
    si = es[0]["size_index"]
    blocks = _pool(lambda b: _synth(W.MiB // 2, W.sweep_block_seed(si, b), False), range(size_mib))
    data = b"".join(blocks)
    del blocks
    pieces = [data[e["offset"]:e["offset"] + e["piece_bytes"]] for e in es]
    del data
    _roundtrip(dev, pieces, es, group=2)
