"""GPU checks for the KV-cache offload chunk producer.

Chunks of a contiguous [B, T, D] cache are zero-copy views; paged caches are
gathered by bb_gather_pages.  Every chunk's container must equal the reference
codec's container of the same bytes (bit-exact) and round-trip losslessly.
"""
import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kv():
    import torch
    assert torch.cuda.is_available()
    from paper_2604_21072_b200.kvchunk import KvChunker
    return torch, KvChunker(0)


def test_chunk_ids_and_views(kv):
    torch, ch = kv
    from paper_2604_21072_b200.kvchunk import chunk_id
    k = torch.randn(3, 16, 8, device="cuda").half()
    v = torch.randn(3, 16, 8, device="cuda").half()
    chunks = ch.chunks(k, v, layer=5)
    assert [c for c, _ in chunks] == [chunk_id(5, kind, s, 3) for kind in (0, 1) for s in range(3)]
    assert chunks[0][0] == 30 and chunks[-1][0] == 35
    assert torch.equal(chunks[4][1], v[1].reshape(-1).view(torch.uint8))
    assert chunks[4][1].data_ptr() == v[1].data_ptr()  # zero-copy


def test_paged_gather_matches_indexing(kv):
    torch, ch = kv
    pool = torch.randint(0, 255, (97, 16, 40), dtype=torch.uint8, device="cuda")  # 640 B pages
    ids = torch.tensor([5, 0, 96, 5, 33, 7], dtype=torch.int32, device="cuda")
    got = ch.gather(pool, ids)
    assert torch.equal(got, pool[ids.long()].reshape(-1))
    odd = torch.randint(0, 255, (9, 13), dtype=torch.uint8, device="cuda")  # unaligned 13-B pages
    assert torch.equal(ch.gather(odd, torch.tensor([8, 1], device="cuda")), odd[[8, 1]].reshape(-1))
    with pytest.raises(ValueError):
        ch.gather(pool, torch.tensor([97], dtype=torch.int32, device="cuda"))


def test_chunk_containers_match_reference(kv, reference):
    torch, ch = kv
    from paper_2604_21072_b200 import synth
    # two layers' worth of small chunks from the reference generator (fp16 Gaussian, seed = chunk id)
    B, T, D = 2, 64, 320
    k = torch.empty(B, T, D, dtype=torch.float16, device="cuda")
    v = torch.empty_like(k)
    chunks = ch.chunks(k, v, layer=3)
    for cid, view in chunks:
        view.copy_(torch.frombuffer(bytearray(synth.gaussian(T * D, cid)), dtype=torch.uint8))
    cs = ch.compress(chunks)
    for (cid, view), c in zip(chunks, cs):
        want = reference.compress(view.cpu().numpy().tobytes(), 1, True)
        assert hashlib.sha256(c.cpu().numpy().tobytes()).hexdigest() == hashlib.sha256(want).hexdigest()
    frames = ch.frames(chunks, cs)
    from paper_2604_21072_b200 import pipeline as pl
    meta, payloads = pl.open_frames(frames)
    assert [m[1] for m in meta] == [cid for cid, _ in chunks]
    outs = [torch.empty(view.numel(), dtype=torch.uint8, device="cuda") for _, view in chunks]
    ch.codec.decompress_batch(payloads, outs)
    assert all(torch.equal(o, view) for o, (_, view) in zip(outs, chunks))


def test_paged_chunk_roundtrip(kv):
    torch, ch = kv
    # vLLM-style paged layer: pool [n_blocks, block_size=16, heads*dh] fp16, one block table per sequence
    rng = np.random.default_rng(3)
    pool = torch.from_numpy(rng.standard_normal((64, 16, 512)).astype(np.float16)).cuda()
    table = torch.tensor(rng.permutation(64)[:20], dtype=torch.int32, device="cuda")
    chunk = ch.gather(pool, table)
    c = ch.compress([chunk])[0]
    back = ch.codec.decompress(c)
    assert torch.equal(back, pool[table.long()].reshape(-1).view(torch.uint8))
