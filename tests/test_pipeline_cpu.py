"""Host-side logic of the stage hand-off (no GPU): BBF1 frames (reference
tests/test_wire.cpp cases), ShapedWriter pacing math, micro-batch spans, and the
ring exchange protocol over gloo with world_size 2."""
import os
import random

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_21072_b200.pipeline import (FRAME_HEADER, FrameCorrupt, ShapedLink, StageRing,
                                            ValidationError, WireFrame, decode_frame, encode_frame,
                                            step_spans)


def test_frame_golden_bytes():
    # reference test_wire.cpp:19-46
    f = WireFrame(1, 0x0102030405060708, 0xBEEF, 0x03, bytes([0xAA, 0xBB]))
    wire = encode_frame(f)
    assert wire == (b"BBF1\x01" + bytes([8, 7, 6, 5, 4, 3, 2, 1]) + bytes([0xEF, 0xBE, 0x03, 2, 0, 0, 0])
                    + bytes([0xAA, 0xBB]))
    assert len(wire) == FRAME_HEADER + 2
    assert decode_frame(wire) == f


def test_frame_corruption_and_fuzz():
    wire = encode_frame(WireFrame(payload=bytes([1, 2, 3])))
    for bad in (b"X" + wire[1:], wire[:4] + b"\x09" + wire[5:], wire[:-1]):
        with pytest.raises(FrameCorrupt):
            decode_frame(bad)
    rng = random.Random(21)
    valid = encode_frame(WireFrame(batch_id=5, payload=rng.randbytes(64)))
    for trial in range(2000):
        fz = bytearray(valid)
        for _ in range(1 + rng.randrange(6)):
            fz[rng.randrange(len(fz))] ^= 1 << rng.randrange(8)
        if trial % 4 == 0:
            fz = fz[: rng.randrange(len(fz) + 1)]
        try:
            d = decode_frame(bytes(fz))
            assert len(d.payload) + FRAME_HEADER == len(fz)
        except FrameCorrupt:
            pass
    for t in range(4):
        assert decode_frame(encode_frame(WireFrame(msg_type=t, batch_id=7))).msg_type == t


def test_step_spans():
    assert step_spans(16, 3) == [(0, 6), (6, 6), (12, 4)]
    assert sum(b for _, b in step_spans(1 << 20, 8)) == 1 << 20
    with pytest.raises(ValidationError):
        step_spans(7, 2)


class FakeClock:
    def __init__(self):
        self.t = 0.0

    def __call__(self):
        return self.t

    def sleep(self, d):
        self.t += max(0.0, d)


def test_shaped_link_token_bucket():
    # reference acceptance #9: 416,400 B at 20 Mbps ~ 166.56 ms
    c = FakeClock()
    link = ShapedLink(20e6, 0.0, clock=c, sleep=c.sleep)
    link.pace(416400)
    assert abs(c.t - 0.16656) < 1e-9
    # reference test_wire.cpp:154-168: 1 MB at 8 Mbps ~ 1 s
    c2 = FakeClock()
    l2 = ShapedLink(8e6, 0.0, clock=c2, sleep=c2.sleep)
    l2.pace(1_000_000)
    assert abs(c2.t - 1.0) < 1e-6
    # as in wire.cpp:224-238, a chunk admitted after sleeping through the latency
    # restarts the wire clock, so rate + latency pace every 64 KiB chunk
    c4 = FakeClock()
    l4 = ShapedLink(8e6, 50.0, clock=c4, sleep=c4.sleep)
    l4.pace(2 * 65536)
    assert abs(c4.t - 2 * (65536 / 1e6 + 0.05)) < 1e-9
    c3 = FakeClock()
    l3 = ShapedLink(0.0, 50.0, clock=c3, sleep=c3.sleep)
    l3.pace(123)
    assert abs(c3.t - 0.05) < 1e-9


def _ring_worker(rank, world, port, ring, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r = StageRing(ring=ring)
    frames = [torch.frombuffer(bytearray(encode_frame(WireFrame(batch_id=rank, micro_index=m,
                                                                  payload=bytes([rank] * (m + 1))))),
                               dtype=torch.uint8) for m in range(3)]
    got = r.exchange(frames if r.has_next() else [], 3 if r.has_prev() else 0)
    dec = [decode_frame(g.numpy().tobytes()) for g in got]
    q.put((rank, [(d.batch_id, d.micro_index, d.payload) for d in dec]))
    dist.destroy_process_group()


@pytest.mark.parametrize("ring", [True, False])
def test_stage_ring_gloo(ring):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + random.randrange(1000)
    ps = [ctx.Process(target=_ring_worker, args=(r, 2, port, ring, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(60)
    # rank 1 always receives rank 0's frames; rank 0 receives rank 1's only in ring mode
    assert res[1] == [(0, m, bytes([0] * (m + 1))) for m in range(3)]
    assert res[0] == ([(1, m, bytes([1] * (m + 1))) for m in range(3)] if ring else [])


def test_read_frame_rejects_payloads_over_one_gib():
    """wire.cpp:260: read_frame refuses a declared payload_len > 1 GiB before reading it."""
    from paper_2604_21072_b200.pipeline import FrameCorrupt, MAX_PAYLOAD, frame_header, read_frame_header
    ok = frame_header(0, 1, 0, 3, MAX_PAYLOAD)
    assert read_frame_header(ok)[4] == MAX_PAYLOAD
    with pytest.raises(FrameCorrupt, match="implausible payload length"):
        read_frame_header(frame_header(0, 1, 0, 3, MAX_PAYLOAD + 1))
