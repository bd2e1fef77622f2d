"""Multi-GPU stage hand-off: one pipeline stage per GPU, compressed BBF1 frames
passed stage to stage over NVLink (NCCL point-to-point), optional WAN shaping.

Reference (proj/src/wire.cpp, proj/include/beeplan/wire.hpp):
  BBF1 frames            encode_frame / decode_frame      wire.cpp:342-370, wire.hpp:14-29
  link shaping           ShapedWriter token bucket         wire.cpp:201-248
  micro-batch slicing    make_step_slices                  wire.cpp:315-336
  roles                  run_wire_source / stage / sink    wire.cpp:388-602
  harness + metrics      run_wire_local, join_hop_metrics  wire.cpp:372-386,604-684

B200 design: the reference relays frames over loopback TCP between threads; here
every stage is one process bound to one GPU (torch.distributed, NCCL), frames
live in HBM, the codec runs on the GPU that owns the stage, and the hop is an
NCCL send/recv (NVLink P2P through NVSwitch).  The ShapedWriter pacing math is
kept verbatim on the sending host thread so shaped runs are comparable with the
reference's 20-500 Mbps experiments.

    torchrun --nproc-per-node N -m paper_2604_21072_b200.pipeline --payload 67108864 \
        --micro-batches 8 --steps 4 [--rate-mbps 100 --latency-ms 5] [--no-compress]
"""
from __future__ import annotations

import argparse
import json
import os
import struct
import sys
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from .codec import Error


class FrameCorrupt(Error):
    """beeplan::FrameCorrupt"""


class ValidationError(Error):
    """beeplan::ValidationError"""


FRAME_MAGIC = b"BBF1"
FRAME_HEADER = 20
MAX_PAYLOAD = 1 << 30  # wire.cpp:31
CHUNK_BYTES = 64 * 1024  # wire.cpp:30

T_ACTIVATIONS, T_PACKED_SD, T_ACK, T_SHUTDOWN = 0, 1, 2, 3
FLAG_COMPRESSED, FLAG_BYTE_SPLIT = 0x01, 0x02


@dataclass
class WireFrame:
    msg_type: int = T_ACTIVATIONS
    batch_id: int = 0
    micro_index: int = 0
    flags: int = 0
    payload: bytes = b""


def frame_header(msg_type: int, batch_id: int, micro_index: int, flags: int, payload_len: int) -> bytes:
    """"BBF1" | u8 type | u64 batch_id | u16 micro | u8 flags | u32 len (LE, 20 bytes)."""
    return FRAME_MAGIC + struct.pack("<BQHBI", msg_type, batch_id, micro_index, flags, payload_len)


def encode_frame(f: WireFrame) -> bytes:
    return frame_header(f.msg_type, f.batch_id, f.micro_index, f.flags, len(f.payload)) + bytes(f.payload)


def parse_frame_header(h: bytes):
    """Header validation of decode_frame / read_frame (wire.cpp:250-267,356-370)."""
    if len(h) < FRAME_HEADER:
        raise FrameCorrupt("frame: truncated header")
    if h[:4] != FRAME_MAGIC:
        raise FrameCorrupt("frame: bad magic")
    msg_type, batch_id, micro, flags, plen = struct.unpack_from("<BQHBI", h, 4)
    if msg_type > 3:
        raise FrameCorrupt(f"frame: unknown msg_type {msg_type}")
    return msg_type, batch_id, micro, flags, plen


def read_frame_header(h: bytes):
    """read_frame's header rules (wire.cpp:250-267): decode_frame's checks plus the 1 GiB cap on
    the declared payload length, checked before any payload byte is received."""
    msg_type, batch_id, micro, flags, plen = parse_frame_header(h)
    if plen > MAX_PAYLOAD:
        raise FrameCorrupt("frame: implausible payload length")
    return msg_type, batch_id, micro, flags, plen


def decode_frame(data: bytes) -> WireFrame:
    data = bytes(data)
    msg_type, batch_id, micro, flags, plen = parse_frame_header(data)
    if len(data) != FRAME_HEADER + plen:
        raise FrameCorrupt("frame: payload length does not match the header")
    return WireFrame(msg_type, batch_id, micro, flags, data[FRAME_HEADER:])


def step_spans(payload_bytes: int, micro_batches: int):
    """make_step_slices' spans (wire.cpp:321-336): elements split into M spans,
    the first `rem` spans one element longer.  Returns (offset, bytes) pairs."""
    if payload_bytes % 2:
        raise ValidationError("payload_bytes: must be even (FP16)")
    elements = payload_bytes // 2
    base, rem = divmod(elements, micro_batches)
    spans, off = [], 0
    for k in range(micro_batches):
        e = base + (1 if k < rem else 0)
        spans.append((off * 2, e * 2))
        off += e
    return spans


class ShapedLink:
    """ShapedWriter pacing (wire.cpp:207-242): a virtual wire clock advanced by
    chunk/rate per 64 KiB chunk; every chunk waits until wire_free + latency."""

    def __init__(self, rate_bps: float = 0.0, latency_ms: float = 0.0, clock=time.monotonic,
                 sleep=time.sleep):
        self.rate_bps, self.latency_ms = rate_bps, latency_ms
        self.clock, self.sleep = clock, sleep
        self.wire_free = 0.0

    def pace(self, nbytes: int) -> float:
        """Blocks as the reference sender would for a frame of nbytes; returns
        the offer time (s)."""
        t_offer = self.clock()
        if self.rate_bps <= 0:
            if self.latency_ms > 0:
                self.sleep(max(0.0, t_offer + self.latency_ms / 1e3 - self.clock()))
            return t_offer
        rate = self.rate_bps / 8.0
        off = 0
        while off < nbytes:
            chunk = min(CHUNK_BYTES, nbytes - off)
            now = self.clock()
            if self.wire_free < now:
                self.wire_free = now
            self.wire_free += chunk / rate
            target = self.wire_free + self.latency_ms / 1e3
            d = target - self.clock()
            if d > 0:
                self.sleep(d)
            off += chunk
        return t_offer


class StageRing:
    """Point-to-point hand-off between neighbouring stages (rank r -> r+1).

    exchange() sends this stage's frames to the next stage and receives the
    previous stage's frames: first the u64 lengths, then one concatenated byte
    buffer, both as paired isend/irecv (NCCL P2P over NVLink on GPUs, gloo on
    CPU).  ring=True closes the ring (last -> first) so every stage does the
    same work (weak scaling)."""

    def __init__(self, ring: bool = True, device=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.ring = ring
        self.device = device if device is not None else torch.device("cpu")
        self.next = (self.rank + 1) % self.world
        self.prev = (self.rank - 1) % self.world

    def has_next(self) -> bool:
        return self.ring or self.rank < self.world - 1

    def has_prev(self) -> bool:
        return self.ring or self.rank > 0

    def exchange(self, frames: Sequence, count_in: int):
        torch, dist = self.torch, self.dist
        ops = []
        lens_out = None
        if self.has_next():
            lens_out = torch.tensor([int(f.numel()) for f in frames], dtype=torch.int64, device=self.device)
            ops.append(dist.P2POp(dist.isend, lens_out, self.next))
        lens_in = None
        if self.has_prev():
            lens_in = torch.empty(count_in, dtype=torch.int64, device=self.device)
            ops.append(dist.P2POp(dist.irecv, lens_in, self.prev))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        ops = []
        if self.has_next():
            buf_out = torch.cat(list(frames)) if len(frames) > 1 else frames[0]
            ops.append(dist.P2POp(dist.isend, buf_out, self.next))
        out = []
        if self.has_prev():
            sizes = [int(x) for x in lens_in.tolist()]
            buf_in = torch.empty(sum(sizes), dtype=torch.uint8, device=self.device)
            ops.append(dist.P2POp(dist.irecv, buf_in, self.prev))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        if self.has_prev():
            off = 0
            for s in sizes:
                out.append(buf_in[off:off + s])
                off += s
        return out


class PeerInbox:
    """Direct stage-to-stage hand-off over NVLink.

    Each stage allocates `slots` inbox buffers in its own HBM; the previous stage
    imports them into its device context (CUDA IPC, include/bbcodec.h
    bb_ipc_export / bb_ipc_import), so the codec's final kernels (bit emission,
    container header) write the compressed frames straight into the receiving
    GPU's memory over NVLink -- the transfer is fused into the compress pipeline
    instead of a separate NCCL copy.  Only the frame lengths go through NCCL P2P:
    a small "doorbell" that also orders buffer reuse (slot k % slots is rewritten
    only after the receiver has posted the doorbell of the step after k, i.e.
    finished decoding k).  Frame m of a step sits at a fixed offset: 20-byte BBF1
    header, then the container.

    Back-pressure: the doorbell alone only orders a stage after its *previous* stage,
    and NCCL's small sends complete before the matching receive is posted, so in a ring
    of three or more GPUs a stage could run ahead of its next stage and rewrite a slot
    still being decoded.  After decoding step k a stage therefore acks k to its previous
    stage (release()); a stage waits for its next stage's ack of step k - slots before the
    codec writes that slot again (out_ptrs())."""

    def __init__(self, caps, device, slots: int = 2):
        import ctypes as C

        import torch
        import torch.distributed as dist

        from . import _lib
        from .codec import _check
        self.C, self.torch, self.dist, self._check = C, torch, dist, _check
        self.L = _lib.load()
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.next, self.prev = (self.rank + 1) % self.world, (self.rank - 1) % self.world
        self.device = device
        self.offsets, off = [], 0
        for c in caps:
            self.offsets.append(off)
            off = (off + FRAME_HEADER + int(c) + 255) & ~255
        self.slot_bytes = off
        self.slots = slots
        self.caps = [int(c) for c in caps]
        self.inbox = [torch.empty(self.slot_bytes, dtype=torch.uint8, device=device) for _ in range(slots)]
        exported = []
        for b in self.inbox:
            h = (C.c_uint8 * 64)()
            o = C.c_size_t()
            _check(self.L.bb_ipc_export(b.data_ptr(), h, C.byref(o)))
            exported.append((bytes(h), o.value))
        gathered = [None] * self.world
        dist.all_gather_object(gathered, exported)
        self.out_base, self.out_ptr = [], []
        for hb, o in gathered[self.next]:
            p, base = C.c_void_p(), C.c_void_p()
            hbuf = (C.c_uint8 * 64).from_buffer_copy(hb)
            _check(self.L.bb_ipc_import(device.index, hbuf, o, C.byref(p), C.byref(base)))
            self.out_ptr.append(p.value)
            self.out_base.append(base.value)
        torch.cuda.set_device(device)
        self.acks = {}  # step -> (works, tensors) of the ack exchange issued after decoding step

    def out_ptrs(self, slot: int):
        """Container destinations inside the next stage's inbox (after each frame header).
        Blocks (stream-ordered) until the next stage acked the previous use of the slot."""
        pending = self.acks.pop(slot - self.slots, None)
        if pending is not None:
            for w in pending[0]:
                w.wait()
        base = self.out_ptr[slot % self.slots]
        return [base + o + FRAME_HEADER for o in self.offsets], self.caps

    def post(self, slot: int, lens, batch_id: int, flags: int, msg_type: int = T_ACTIVATIONS):
        """Write the frame headers next to the containers already in the peer's inbox and
        exchange lengths with both neighbours; returns the previous stage's frames (views
        of this stage's inbox)."""
        C, torch, dist = self.C, self.torch, self.dist
        stream = torch.cuda.current_stream(self.device)
        base = self.out_ptr[slot % self.slots]
        hdrs = [frame_header(msg_type, batch_id, m, flags, int(n)) for m, n in enumerate(lens)]
        for o, h in zip(self.offsets, hdrs):
            self._check(self.L.bb_copy_h2d(base + o, h, FRAME_HEADER, stream.cuda_stream))
        stream.synchronize()  # containers + headers are in the peer's HBM
        out = torch.tensor([int(n) for n in lens], dtype=torch.int64, device=self.device)
        got = torch.empty(len(lens), dtype=torch.int64, device=self.device)
        for r in dist.batch_isend_irecv([dist.P2POp(dist.isend, out, self.next),
                                         dist.P2POp(dist.irecv, got, self.prev)]):
            r.wait()
        ib = self.inbox[slot % self.slots]
        return [ib[o:o + FRAME_HEADER + int(n)] for o, n in zip(self.offsets, got.tolist())]

    def release(self, slot: int):
        """This stage finished decoding `slot`'s frames (stream-ordered): ack it to the
        previous stage and receive the next stage's ack of the same step (one symmetric
        NCCL group, so the ring cannot deadlock)."""
        dist, torch = self.dist, self.torch
        ack = torch.full((1,), slot, dtype=torch.int64, device=self.device)
        got = torch.empty(1, dtype=torch.int64, device=self.device)
        works = dist.batch_isend_irecv([dist.P2POp(dist.isend, ack, self.prev),
                                        dist.P2POp(dist.irecv, got, self.next)])
        self.acks[slot] = (works, (ack, got))

    def drain(self):
        for works, _ in self.acks.values():
            for w in works:
                w.wait()
        self.acks.clear()

    def close(self):
        self.drain()
        for b in self.out_base:
            self.L.bb_ipc_close(b)
        self.out_base, self.out_ptr = [], []


def build_frames(containers, batch_id: int, flags: int, device, msg_type: int = T_ACTIVATIONS):
    """BBF1 frames on the device: host-built 20-byte headers + container bytes
    (msg_type T_PACKED_SD for speculative-decoding token-tree payloads)."""
    import torch
    hdrs = b"".join(frame_header(msg_type, batch_id, m, flags, int(c.numel()))
                    for m, c in enumerate(containers))
    h = torch.frombuffer(bytearray(hdrs), dtype=torch.uint8).to(device, non_blocking=True)
    return [torch.cat([h[FRAME_HEADER * m:FRAME_HEADER * (m + 1)], c]) for m, c in enumerate(containers)]


def open_frames(frames):
    """Validates received headers (one device->host gather) and returns payload views."""
    import torch
    if not frames:
        return [], []
    heads = torch.cat([f[:FRAME_HEADER] for f in frames]).cpu().numpy().tobytes()
    meta, payloads = [], []
    for m, f in enumerate(frames):
        t, b, mi, fl, plen = read_frame_header(heads[FRAME_HEADER * m:FRAME_HEADER * (m + 1)])
        if f.numel() != FRAME_HEADER + plen:
            raise FrameCorrupt("frame: payload length does not match the header")
        meta.append((t, b, mi, fl))
        payloads.append(f[FRAME_HEADER:])
    return meta, payloads


# ---------------------------------------------------------------------------
# bench-wire analogue: source (rank 0) -> stages -> sink (last rank)

def run_pipeline(args) -> dict:
    import torch
    import torch.distributed as dist

    from . import codec, synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import datetime  # a failed stage must not block its neighbours forever (NCCL watchdog)
        dist.init_process_group("nccl", device_id=dev,
                                timeout=datetime.timedelta(seconds=int(os.environ.get("BB_NCCL_TIMEOUT_S", "600"))))
    rank = dist.get_rank() if world > 1 else 0
    dc = codec.DeviceCodec(local)
    spans = step_spans(args.payload, args.micro_batches)
    link = ShapedLink(args.rate_mbps * 1e6, args.latency_ms)
    ring = StageRing(ring=False, device=dev) if world > 1 else None
    flags = (FLAG_COMPRESSED | FLAG_BYTE_SPLIT) if args.compress else 0
    ok = True
    codec_ms = 0.0
    sent_bytes = 0
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for step in range(args.steps):
        # source: regenerate the step's stream (make_step_slices), slice, compress
        if rank == 0:
            stream = synth.gaussian(args.payload // 2, args.seed + step, False)
            xs = [torch.frombuffer(bytearray(stream[o:o + b]), dtype=torch.uint8).to(dev)
                  for o, b in spans]
        else:
            xs = None
        if rank > 0:
            frames = ring.exchange([], len(spans))
            meta, payloads = open_frames(frames)
            tc = time.perf_counter()
            if args.compress:
                outs = [torch.empty(b, dtype=torch.uint8, device=dev) for _, b in spans]
                dc.decompress_batch(payloads, outs)
                xs = outs
            else:
                xs = list(payloads)
            codec_ms += 1e3 * (time.perf_counter() - tc)
        if args.compute_ms > 0:
            time.sleep(args.compute_ms / 1e3)
        last = world == 1 or rank == world - 1
        if not last:
            tc = time.perf_counter()
            if args.compress:
                bufs = [torch.empty(dc.compress_bound(x.numel()), dtype=torch.uint8, device=dev) for x in xs]
                lens = dc.compress_batch(xs, bufs)
                cs = [b[:n] for b, n in zip(bufs, lens)]
            else:
                cs = xs
            codec_ms += 1e3 * (time.perf_counter() - tc)
            frames = build_frames(cs, step, flags, dev)
            for f in frames:
                link.pace(int(f.numel()))  # ShapedWriter pacing per frame
                sent_bytes += int(f.numel())
            ring.exchange(frames, 0)
        else:
            # sink: bit-exact reassembly against the regenerated stream
            want = synth.gaussian(args.payload // 2, args.seed + step, False)
            if world == 1 and args.compress:
                bufs = [torch.empty(dc.compress_bound(x.numel()), dtype=torch.uint8, device=dev) for x in xs]
                lens = dc.compress_batch(xs, bufs)
                outs = [torch.empty(x.numel(), dtype=torch.uint8, device=dev) for x in xs]
                dc.decompress_batch([b[:n] for b, n in zip(bufs, lens)], outs)
                xs = outs
            got = torch.cat(xs).cpu().numpy().tobytes()
            ok = ok and got == want
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2e = time.perf_counter() - t0
    res = {"rank": rank, "world": world, "steps": args.steps, "micro_batches": args.micro_batches,
           "payload_bytes": args.payload, "compress": args.compress, "e2e_ms": 1e3 * e2e,
           "throughput_tokens_per_s": args.steps / e2e,  # wire.cpp:678-679 definition
           "rows_per_s": args.steps * args.payload / 2 / args.hidden / e2e,
           "codec_ms_total": codec_ms, "sent_bytes": sent_bytes, "payload_ok": ok,
           "shape": {"rate_mbps": args.rate_mbps, "latency_ms": args.latency_ms}}
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, res)
        dist.destroy_process_group()
        res = {"stages": gathered, "e2e_ms": max(g["e2e_ms"] for g in gathered),
               "payload_ok": gathered[-1]["payload_ok"]}
        res["throughput_tokens_per_s"] = args.steps / (res["e2e_ms"] / 1e3)
    return res


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="BBF1 stage hand-off over NVLink (bench-wire analogue)")
    ap.add_argument("--payload", type=int, default=4 * 128 * 4096 * 2)
    ap.add_argument("--micro-batches", type=int, default=4)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--compute-ms", type=float, default=0.0)
    ap.add_argument("--rate-mbps", type=float, default=0.0)
    ap.add_argument("--latency-ms", type=float, default=0.0)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--no-compress", dest="compress", action="store_false")
    args = ap.parse_args(argv)
    res = run_pipeline(args)
    if int(os.environ.get("RANK", "0")) == 0:
        print(json.dumps(res))
    return 0 if res.get("payload_ok", True) else 1


if __name__ == "__main__":
    sys.exit(main())
