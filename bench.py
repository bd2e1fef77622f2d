#!/usr/bin/env python
"""bench.py -- BBC1 activation codec (BloomBee hot path) on B200.

Metric (BASELINE.json): codec GB/s (enc+dec, bit-exact) vs HBM roofline;
pipelined tokens/s at 1/2/4/8.

Default workload = BASELINE configs[1] (LLaMA-2-7B, 8 pipeline stages, 8
micro-batches of [16, 512, 4096] bf16 activations): a step = one stage boundary,
the 8 micro-batch tensors (64 MiB each, 512 MiB per step) compressed into BBC1
containers (byte split + zlib-1.3-level-6-exact deflate, bit-identical to the
reference) and decompressed back, on the GPU.  value = raw bytes / step time.

Other BASELINE configs (parity-test cases; measured with --workload):
  config1  [1,128,4096] fp16 hidden state (the reference's CPU case)
  config3  speculative-decoding token trees: 32 requests x (64 wide x 8 deep = 512
           states) x d=4096, pruned (keep mask) and packed on the device into the
           reference's encode_packed f32 layout, then compressed (PackedSd frames)
  config4  LLaMA-2-13B KV-cache offload: one layer = 64 chunks of [4096, 5120] fp16
  config5  d=8192 fp16 tensor sweep 1 MiB .. 1 GiB (--sweep-max-mib 4096 adds 4 GiB,
           chunked at 512 MiB per frame), with the 100 Mbps ShapedWriter link time

  python bench.py [--gpus N --steps K --warmup W] [--workload config2|config1|config3|config4|config5]
  python bench.py --impl reference ...   # the reference C++ codec on the host cores

N > 1 (torchrun, one process per GPU): every rank is one pipeline stage; each
step its compressed BBF1 frames go to the next stage over NVLink (NCCL P2P
ring) and the previous stage's frames are decompressed (weak scaling).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SD_REQUESTS, SD_NODES, SD_DIM, SD_KEEP_PCT = 32, 64 * 8, 4096, 60
KV_BATCH, KV_CTX, KV_DIM, KV_GROUP = 32, 4096, 5120, 16
SWEEP_DIM = 8192
MiB = 1 << 20
HANDOFF = "p2p"  # multi-GPU hand-off of config1/2 frames: "p2p" (fused into the codec) or "nccl"


def _threads(fn, n):
    """fn(0..n-1) on a host thread pool (the generators release the GIL)."""
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(n, os.cpu_count() or 1, 32))) as ex:
        return list(ex.map(fn, range(n)))


def synth(elements: int, seed: int, bf16: bool) -> bytes:
    """Host-side input generator (C++ drop-in, reference synth.cpp semantics)."""
    from paper_2604_21072_b200 import synth as S
    return S.gaussian(elements, seed, bf16)


def sd_request(r: int):
    """Request r's token tree: f32 states (exact upcast of synth fp16, seed 7 + r) + keep mask."""
    import numpy as np
    states = np.frombuffer(synth(SD_NODES * SD_DIM, 7 + r, False), dtype="<f2").astype(np.float32)
    keep = (np.random.default_rng(7000 + r).integers(0, 100, SD_NODES) < SD_KEEP_PCT).astype(np.uint8)
    return states.reshape(SD_NODES, SD_DIM), keep


def link_seconds(nbytes: int, rate_mbps: float, latency_ms: float) -> float:
    """Time a frame occupies a ShapedWriter link from idle (wire.cpp:207-242 math)."""
    from paper_2604_21072_b200.pipeline import ShapedLink
    now = [0.0]
    link = ShapedLink(rate_mbps * 1e6, latency_ms, clock=lambda: now[0],
                      sleep=lambda d: now.__setitem__(0, now[0] + d))
    link.pace(nbytes)
    return now[0]


# ---------------------------------------------------------------------------
# workloads: device state + one step (compress -> [NVLink hand-off] -> decompress)

class Workload:
    name = desc = ""
    msg_type = 0
    tokens_per_step = 0

    def frames_exchange(self, ring, cs, step_no):
        from paper_2604_21072_b200.pipeline import FLAG_BYTE_SPLIT, FLAG_COMPRESSED, build_frames, open_frames
        frames = build_frames(cs, step_no, FLAG_COMPRESSED | FLAG_BYTE_SPLIT, cs[0].device, self.msg_type)
        _, got = open_frames(ring.exchange(frames, len(cs)))
        return got


class ActWorkload(Workload):
    """configs[0] / configs[1]: micro-batch activation tensors."""

    def __init__(self, name, desc, mb, elems, bf16, tokens, seed_fn):
        self.name, self.desc, self.mb, self.elems, self.bf16 = name, desc, mb, elems, bf16
        self.tokens_per_step = mb * tokens
        self.seed_fn = seed_fn

    def host(self, rank):
        return _threads(lambda i: synth(self.elems, self.seed_fn(rank, i), self.bf16), self.mb)

    def setup(self, torch, dc, rank, world):
        self.torch, self.dc = torch, dc
        self.h = self.host(rank)
        self.raw_step = sum(len(x) for x in self.h)
        self.xs = [torch.frombuffer(bytearray(x), dtype=torch.uint8).cuda() for x in self.h]
        self.outs = [torch.empty(dc.compress_bound(x.numel()), dtype=torch.uint8, device="cuda") for x in self.xs]
        self.decs = [torch.empty(x.numel(), dtype=torch.uint8, device="cuda") for x in self.xs]
        self.rank, self.world = rank, world

    def step(self, ring, step_no):
        if ring is not None and HANDOFF == "p2p":
            # fused hand-off: the compress pipeline writes the frames into the next GPU's inbox
            from paper_2604_21072_b200.pipeline import (FLAG_BYTE_SPLIT, FLAG_COMPRESSED, PeerInbox,
                                                        open_frames)
            if getattr(self, "peer", None) is None:
                self.peer = PeerInbox([o.numel() for o in self.outs], self.xs[0].device)
            ptrs, caps = self.peer.out_ptrs(step_no)
            lens = self.dc.compress_batch_ptr(self.xs, ptrs, caps)
            frames = self.peer.post(step_no, lens, step_no, FLAG_COMPRESSED | FLAG_BYTE_SPLIT)
            _, cs = open_frames(frames)
            self.dc.decompress_batch(cs, self.decs)
            return sum(lens)
        lens = self.dc.compress_batch(self.xs, self.outs)
        cs = [o[:n] for o, n in zip(self.outs, lens)]
        if ring is not None:
            cs = self.frames_exchange(ring, cs, step_no)
        self.dc.decompress_batch(cs, self.decs)
        return sum(lens)

    def verify(self):
        if self.world > 1:  # the decoded tensors are the previous stage's activations
            prev = self.host((self.rank - 1) % self.world)
            return all(d.cpu().numpy().tobytes() == h for d, h in zip(self.decs, prev))
        return all(self.torch.equal(d, x) for d, x in zip(self.decs, self.xs))

    def e2e_buffers(self):
        t = self.torch
        pin_in = [t.frombuffer(bytearray(h), dtype=t.uint8).pin_memory() for h in self.h]
        pin_out = [t.empty(len(h), dtype=t.uint8).pin_memory() for h in self.h]
        self.e2e_bufs = (t.cuda.Stream(), [self.xs, [t.empty_like(x) for x in self.xs]],
                         [self.decs, [t.empty_like(d) for d in self.decs]],
                         [pin_out, [t.empty_like(p).pin_memory() for p in pin_out]])
        return pin_in, pin_out

    def e2e_step(self, ring, step_no, pin_in, pin_out):
        for x, p in zip(self.xs, pin_in):
            x.copy_(p, non_blocking=True)
        self.step(ring, step_no)
        for d, p in zip(self.decs, pin_out):
            p.copy_(d, non_blocking=True)
        return sum(p.numel() for p in pin_in), sum(p.numel() for p in pin_out)

    def e2e_run(self, ring, step_no, steps, pin_in, pin_out):
        """steps end-to-end steps with the copies of step k+1 (H2D) and k-1 (D2H) on a copy
        stream overlapping step k's codec work (double-buffered device tensors)."""
        t = self.torch
        comp = t.cuda.current_stream()
        copy, xin, xout, pout = self.e2e_bufs  # allocated outside the timed region
        ev_in = [t.cuda.Event(), t.cuda.Event()]
        ev_done = [t.cuda.Event(), t.cuda.Event()]
        with t.cuda.stream(copy):
            for x, p in zip(xin[0], pin_in):
                x.copy_(p, non_blocking=True)
            ev_in[0].record(copy)
        for k in range(steps):
            cur, nxt = k % 2, (k + 1) % 2
            if k + 1 < steps:
                with t.cuda.stream(copy):
                    if k >= 1:
                        copy.wait_event(ev_done[nxt])  # step k-1 no longer reads xin[nxt]
                    for x, p in zip(xin[nxt], pin_in):
                        x.copy_(p, non_blocking=True)
                    ev_in[nxt].record(copy)
            comp.wait_event(ev_in[cur])
            self.xs, self.decs = xin[cur], xout[cur]
            self.step(ring, step_no + k)
            ev_done[cur].record(comp)
            with t.cuda.stream(copy):
                copy.wait_event(ev_done[cur])
                for d, p in zip(xout[cur], pout[cur]):
                    p.copy_(d, non_blocking=True)
        copy.synchronize()
        comp.synchronize()
        self.xs, self.decs = xin[0], xout[0]
        return sum(p.numel() for p in pin_in), sum(p.numel() for p in pin_out)

    def sample_bytes(self):
        return self.h[0][: 8 * MiB]

    def ref_job(self, rank, i, cap):
        return ("synth", min(self.elems, cap // 2), self.seed_fn(rank, i % self.mb), self.bf16)


class SdWorkload(Workload):
    """configs[2]: token-tree verification payloads (PackedSd frames)."""
    name = "config3"
    desc = (f"sd token trees: {SD_REQUESTS} requests x 512 states (width 64, depth 8) x d={SD_DIM} f32, "
            f"{SD_KEEP_PCT}% kept, device pack -> encode_packed layout -> BBC1")
    msg_type = 1
    tokens_per_step = SD_REQUESTS * SD_NODES

    def setup(self, torch, dc, rank, world):
        import numpy as np
        from paper_2604_21072_b200 import specdec
        self.torch, self.dc, self.rank, self.world = torch, dc, rank, world
        self.packer = specdec.DevicePacker(torch.cuda.current_device())
        reqs = _threads(lambda r: sd_request(r + rank * SD_REQUESTS), SD_REQUESTS)
        self.h_rows = np.concatenate([s for s, _ in reqs])
        self.h_keep = np.concatenate([k for _, k in reqs])
        self.req_rows = [i * SD_NODES for i in range(SD_REQUESTS + 1)]
        self.rows = torch.from_numpy(self.h_rows).cuda()
        self.keep = torch.from_numpy(self.h_keep).cuda()
        n = self.h_rows.shape[0]
        self.pbuf = torch.empty(self.packer.bound(n, SD_DIM, SD_REQUESTS), dtype=torch.uint8, device="cuda")
        self.raw_step = int(self.packer.pack_encode(self.rows, self.keep, self.req_rows, out=self.pbuf).numel())
        self.cbuf = torch.empty(dc.compress_bound(self.raw_step), dtype=torch.uint8, device="cuda")
        self.dbuf = torch.empty(self.raw_step, dtype=torch.uint8, device="cuda")
        self.payload = None

    def step(self, ring, step_no):
        packed = self.packer.pack_encode(self.rows, self.keep, self.req_rows, out=self.pbuf)
        n = self.dc.compress_into(packed, self.cbuf)
        cs = [self.cbuf[:n]]
        if ring is not None:
            cs = self.frames_exchange(ring, cs, step_no)
        m = self.dc.decompress_into(cs[0], self.dbuf)
        self.offsets, self.payload = self.packer.open(self.dbuf[:m], SD_DIM)
        return n

    def verify(self):
        t = self.torch
        if self.world > 1:
            import numpy as np
            prev = (self.rank - 1) % self.world
            reqs = [sd_request(r + prev * SD_REQUESTS) for r in range(SD_REQUESTS)]
            want = np.concatenate([s[k.astype(bool)] for s, k in reqs])
            return self.payload.cpu().numpy().tobytes() == want.tobytes()
        return t.equal(self.payload.view(t.int32), self.rows[self.keep.bool()].view(t.int32))

    def e2e_buffers(self):
        t = self.torch
        pin_rows = t.from_numpy(self.h_rows).pin_memory()
        pin_keep = t.from_numpy(self.h_keep).pin_memory()
        return [pin_rows, pin_keep], [t.empty(self.payload.numel() * 4, dtype=t.uint8).pin_memory()]

    def e2e_step(self, ring, step_no, pin_in, pin_out):
        self.rows.copy_(pin_in[0], non_blocking=True)
        self.keep.copy_(pin_in[1], non_blocking=True)
        self.step(ring, step_no)
        pin_out[0].copy_(self.payload.reshape(-1).view(self.torch.uint8), non_blocking=True)
        return pin_in[0].numel() * 4 + pin_in[1].numel(), pin_out[0].numel()

    def sample_bytes(self):
        return self.pbuf[: min(self.raw_step, 8 * MiB)].cpu().numpy().tobytes()

    def ref_job(self, rank, i, cap):
        return ("sd", i % SD_REQUESTS + rank * SD_REQUESTS)


class KvWorkload(Workload):
    """configs[3]: LLaMA-2-13B KV-cache offload chunks (one layer per step)."""
    name = "config4"
    desc = (f"llama2-13b KV offload: layer 0, K|V x {KV_BATCH} sequences = 64 chunks of "
            f"[{KV_CTX},{KV_DIM}] fp16 (40 MiB), seeds = chunk id, {KV_GROUP} chunks per codec batch")
    tokens_per_step = KV_BATCH * KV_CTX

    def setup(self, torch, dc, rank, world):
        from paper_2604_21072_b200.kvchunk import KvChunker
        self.torch, self.dc, self.rank, self.world = torch, dc, rank, world
        self.layer = rank  # each stage offloads its own layer
        self.chunker = KvChunker(torch.cuda.current_device(), dc)
        self.k = torch.empty((KV_BATCH, KV_CTX, KV_DIM), dtype=torch.float16, device="cuda")
        self.v = torch.empty_like(self.k)
        self.chunks = self.chunker.chunks(self.k, self.v, self.layer)
        self.h = self.host(self.layer)
        for (_, view), hb in zip(self.chunks, self.h):
            view.copy_(torch.frombuffer(bytearray(hb), dtype=torch.uint8))
        self.raw_step = sum(v.numel() for _, v in self.chunks)
        self.outs = [torch.empty(dc.compress_bound(v.numel()), dtype=torch.uint8, device="cuda")
                     for _, v in self.chunks[:KV_GROUP]]
        self.decs = [torch.empty(v.numel(), dtype=torch.uint8, device="cuda") for _, v in self.chunks]

    def host(self, layer):
        from paper_2604_21072_b200.kvchunk import chunk_id
        ids = [chunk_id(layer, kind, s, KV_BATCH) for kind in (0, 1) for s in range(KV_BATCH)]
        return _threads(lambda i: synth(KV_CTX * KV_DIM, ids[i], False), len(ids))

    def step(self, ring, step_no):
        total = 0
        for g in range(0, len(self.chunks), KV_GROUP):
            part = self.chunks[g:g + KV_GROUP]
            cs = self.chunker.compress(part, self.outs[:len(part)])
            total += sum(int(c.numel()) for c in cs)
            if ring is not None:
                cs = self.frames_exchange(ring, cs, step_no)
            self.dc.decompress_batch(cs, self.decs[g:g + KV_GROUP])
        return total

    def verify(self):
        if self.world > 1:
            prev = self.host((self.rank - 1) % self.world)
            return all(d.cpu().numpy().tobytes() == h for d, h in zip(self.decs, prev))
        return all(self.torch.equal(d, v) for d, (_, v) in zip(self.decs, self.chunks))

    def e2e_buffers(self):
        t = self.torch
        return ([t.frombuffer(bytearray(h), dtype=t.uint8).pin_memory() for h in self.h],
                [t.empty(len(h), dtype=t.uint8).pin_memory() for h in self.h])

    def e2e_step(self, ring, step_no, pin_in, pin_out):
        for (_, v), p in zip(self.chunks, pin_in):
            v.copy_(p, non_blocking=True)
        self.step(ring, step_no)
        for d, p in zip(self.decs, pin_out):
            p.copy_(d, non_blocking=True)
        return sum(p.numel() for p in pin_in), sum(p.numel() for p in pin_out)

    def sample_bytes(self):
        return self.h[0][: 8 * MiB]

    def ref_job(self, rank, i, cap):
        from paper_2604_21072_b200.kvchunk import chunk_id
        return ("synth", cap // 2, chunk_id(rank, i % 2, i // 2 % KV_BATCH, KV_BATCH), False)


WORKLOADS = {
    "config2": lambda: ActWorkload("config2", "llama2-7b stage boundary: 8 micro-batches x [16,512,4096] bf16",
                                   8, 16 * 512 * 4096, True, 16 * 512, lambda rank, i: 1000 * (rank + 1) + i),
    "config1": lambda: ActWorkload("config1", "llama-7b hidden state [1,128,4096] fp16, seed 1", 1, 128 * 4096,
                                   False, 128, lambda rank, i: 1),
    "config3": SdWorkload,
    "config4": KvWorkload,
}


class Clocks:
    """nvidia-smi samples (every 200 ms: faster polling contends with the driver) kept for the timed
    region [t0, t1] (wall clock).

    The sampler is started before the warm-up so that short timed regions are covered; a region
    shorter than the sampling period reports the nearest sample and says so."""

    def __init__(self, dev: int):
        q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,power.draw")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(dev), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def stop(self, t0: float = None, t1: float = None) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        import datetime
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        rows = []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(f[1]), float(f[2]), {nm for nm, v in zip(names, f[4:8]) if v.lower() == "active"}))
            except ValueError:
                continue
        sel, nearest = rows, False
        if t0 is not None and rows:
            sel = [r for r in rows if t0 <= r[0] <= t1]
            if not sel:  # region shorter than the sampling period
                mid = 0.5 * (t0 + t1)
                sel, nearest = [min(rows, key=lambda r: abs(r[0] - mid))], True
        reasons = set().union(*[r[3] for r in sel]) if sel else set()
        res = {"sm_mhz": statistics.median(r[1] for r in sel) if sel else None,
               "sm_max_mhz": max(r[2] for r in sel) if sel else None,
               "samples": 0 if nearest else len(sel), "reasons": sorted(reasons)}
        if nearest:
            res["nearest_sample_s"] = round(min(abs(sel[0][0] - t0), abs(sel[0][0] - t1)), 3)
        return res


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# reference CPU codec (oracle/_ref = reference codec.cpp + specdec.cpp + zlib 1.3), timed on host cores

def _ref_worker(job):
    from oracle.oracle import Oracle, Reference
    ref = Reference()
    if job[0] == "sd":
        # the reference's own path for a token tree: pack -> encode_packed -> compress,
        # then decompress -> decode_packed
        states, keep = sd_request(job[1])
        per_request = [[states[i] for i in range(SD_NODES) if keep[i]]]
        t0 = time.perf_counter()
        data = ref.pack_encode(per_request)
        c = ref.compress(data, 1, True)
        t1 = time.perf_counter()
        d = ref.decompress(c)
        ref.decode_packed(d, SD_DIM)
        t2 = time.perf_counter()
    else:
        _, elems, seed, bf16 = job
        orc = Oracle()
        data = orc.synth_bf16(elems, seed) if bf16 else orc.synth_fp16(elems, seed)
        t0 = time.perf_counter()
        c = ref.compress(data, 1, True)
        t1 = time.perf_counter()
        d = ref.decompress(c)
        t2 = time.perf_counter()
    assert d == data
    return {"raw": len(data), "container": len(c), "enc_s": t1 - t0, "dec_s": t2 - t1,
            "sha256": hashlib.sha256(c).hexdigest()}


def reference_sample(jobs):
    import multiprocessing as mp
    t0 = time.perf_counter()
    if len(jobs) == 1:
        res = [_ref_worker(jobs[0])]
    else:
        with mp.get_context("fork").Pool(len(jobs)) as pool:
            res = pool.map(_ref_worker, jobs)
    return res, time.perf_counter() - t0


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    wl = WORKLOADS[args.workload]()
    from oracle.oracle import build
    build()
    procs = max(1, min(os.cpu_count() or 1, 16))
    cap = 8 * MiB  # bytes of workload data per process per step (~1 s of CPU work)
    jobs = [wl.ref_job(0, i, cap) for i in range(procs)]
    vals, total_wall, raw = [], 0.0, 0
    for step in range(args.warmup + args.steps):
        res, wall = reference_sample(jobs)
        if step >= args.warmup:
            raw = sum(r["raw"] for r in res)
            vals.append(raw / wall / 1e9)
            total_wall += wall
    value = statistics.median(vals)
    sample = f"{procs} processes x one {raw // procs} B slice of {wl.name} data per step ({wl.desc})"
    line = {
        "impl": "reference", "metric": "codec GB/s (enc+dec, bit-exact)", "value": value, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * total_wall / max(1, args.steps), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": wl.name, "description": wl.desc},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": procs, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------

def run_sweep(args, torch, dist, world, rank, dev_id):
    """configs[4]: d=8192 fp16 tensors, 1 MiB .. 1 GiB (.. 4 GiB), 100 Mbps shaped links."""
    from paper_2604_21072_b200 import _lib, codec
    dc = codec.DeviceCodec(dev_id)
    piece = 512 * MiB  # frames carry <= 1 GiB (wire.cpp:31): larger tensors are cut into pieces
    sizes = [MiB << (2 * k) for k in range(6)]
    if args.sweep_max_mib >= 4096:
        sizes.append(4096 * MiB)
    results = []
    ring = None
    if world > 1:
        from paper_2604_21072_b200.pipeline import StageRing
        ring = StageRing(ring=True, device=torch.device("cuda", dev_id))
    wl = Workload()
    clocks = Clocks(dev_id)
    launches0 = _lib.kernel_launches()
    tot_raw, tot_ms, ok_all = 0, 0.0, True
    for si, size in enumerate(sizes):
        blocks = size // MiB  # 1 MiB = 64 rows of d=8192; block b uses seed 50000 + 4096*si + b
        hb = _threads(lambda b: synth(MiB // 2, 50000 + 4096 * si + b + 1000000 * rank, False), blocks)
        x = torch.empty(size, dtype=torch.uint8, device="cuda")
        for b, h in enumerate(hb):
            x[b * MiB:(b + 1) * MiB].copy_(torch.frombuffer(bytearray(h), dtype=torch.uint8))
        del hb
        pieces = [x[o:o + piece] for o in range(0, size, piece)]
        outs = [torch.empty(dc.compress_bound(p.numel()), dtype=torch.uint8, device="cuda") for p in pieces[:2]]
        dec = torch.empty_like(x)
        decs = [dec[o:o + piece] for o in range(0, size, piece)]

        def step(step_no):
            comp = []
            for g in range(0, len(pieces), 2):  # <= 1 GiB of codec input per pipeline call
                lens = dc.compress_batch(pieces[g:g + 2], outs)
                cs = [o[:n] for o, n in zip(outs, lens)]
                comp += lens
                if ring is not None:
                    cs = wl.frames_exchange(ring, cs, step_no)
                dc.decompress_batch(cs, decs[g:g + 2])
            return comp

        steps = args.steps if size <= 256 * MiB else max(1, min(args.steps, 2))
        for w in range(max(1, args.warmup if size <= 256 * MiB else 1)):
            comp = step(w)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in range(steps):
            step(s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        ok = torch.equal(dec, x) if world == 1 else None
        ok_all = ok_all and (ok is not False)
        link_s = sum(link_seconds(n + 20, 100.0, 0.0) for n in comp)  # BBF1 header = 20 B
        raw_link_s = sum(link_seconds(p.numel() + 20, 100.0, 0.0) for p in pieces)
        comp = sum(comp)
        rows = size // (2 * SWEEP_DIM)
        results.append({"bytes": size, "rows": rows, "frames": len(pieces), "ms": ms,
                        "gbps": world * size / (ms / 1e3) / 1e9, "ratio": comp / size, "lossless": ok,
                        "link_100mbps_s": link_s, "uncompressed_link_100mbps_s": raw_link_s,
                        "pipelined_rows_per_s": rows / max(ms / 1e3, link_s)})
        tot_raw += size
        tot_ms += ms
        del x, dec, pieces, decs, outs
        torch.cuda.empty_cache()
    clk = clocks.stop()
    launches = _lib.kernel_launches() - launches0
    if rank != 0:
        return None
    big = results[-1]
    return {"metric": "codec GB/s (enc+dec, bit-exact) vs HBM roofline", "value": world * tot_raw / (tot_ms / 1e3) / 1e9,
            "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": "config5", "description": "d=8192 fp16 tensor sweep, one tensor per size per "
                       "step, 100 Mbps ShapedWriter link time computed from the frame sizes",
                       "sizes": sizes, "parallelism": f"{world} stage(s)"},
            "lossless": ok_all, "sweep": results, "largest": big, "gpu_launches": launches, "clocks": clk}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="config2", choices=sorted(list(WORKLOADS) + ["config5"]))
    ap.add_argument("--sweep-max-mib", type=int, default=1024)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--handoff", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1: frames written into the next GPU by the codec (p2p) or sent by NCCL")
    args = ap.parse_args()
    global HANDOFF
    HANDOFF = args.handoff
    world, rank, local = dist_init()
    if args.impl == "reference":
        if args.workload == "config5":
            args.workload = "config1"  # the reference CPU codec on config5 rows = the same codec on fp16 rows
        return run_reference(args, world, rank)

    import torch
    import torch.distributed as dist

    from paper_2604_21072_b200 import _lib, codec

    torch.cuda.set_device(local)
    dev_id = local
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.workload == "config5":
        line = run_sweep(args, torch, dist, world, rank, dev_id)
        if line is not None:
            print(json.dumps(line), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return 0

    wl = WORKLOADS[args.workload]()
    dc = codec.DeviceCodec(dev_id)
    wl.setup(torch, dc, rank, world)
    raw_step = wl.raw_step
    ring = None
    if world > 1:
        from paper_2604_21072_b200.pipeline import StageRing
        ring = StageRing(ring=True, device=torch.device("cuda", local))
    step_no = [0]

    def step():
        comp = wl.step(ring, step_no[0])
        step_no[0] += 1
        return comp

    comp_step = 0
    clocks = Clocks(dev_id)  # started before the warm-up; only timed-region samples are kept
    for _ in range(args.warmup):
        comp_step = step()
    torch.cuda.synchronize()
    ok = wl.verify() if args.warmup else None  # losslessness of the timed configuration, checked outside the timed region

    # timed region: device-resident inputs (> 126 MB L2 for config2/3/4: no L2 reuse between steps)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    _lib.stage_timing(True)
    _lib.stage_report(reset=True)
    launches0 = _lib.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_wall0 = time.time()
    ev0.record()
    for _ in range(args.steps):
        comp_step = step()
    ev1.record()
    torch.cuda.synchronize()
    t_wall1 = time.time()
    launches = _lib.kernel_launches() - launches0
    stages = _lib.stage_report(reset=True)
    _lib.stage_timing(False)
    clk = clocks.stop(t_wall0, t_wall1)
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = world * raw_step / (ms_step / 1e3) / 1e9

    # end to end through the public API: pinned host inputs -> device round trip -> pinned host output
    e2e = None
    if not args.no_e2e:
        pin_in, pin_out = wl.e2e_buffers()
        e_steps = max(1, min(args.steps, 8))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if hasattr(wl, "e2e_run"):  # copies of neighbouring steps overlap the codec (copy stream)
            h2d, d2h = wl.e2e_run(ring, step_no[0], e_steps, pin_in, pin_out)
            step_no[0] += e_steps
        else:
            for _ in range(e_steps):
                h2d, d2h = wl.e2e_step(ring, step_no[0], pin_in, pin_out)
                step_no[0] += 1
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        e_s = (time.perf_counter() - t0) / e_steps
        if world > 1:
            t = torch.tensor([e_s], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_s = float(t.item())
        e2e = {"value": world * raw_step / e_s / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * e_s}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"
    # dominant kernel / stage by device time
    per_launch = {k: v["ms"] / max(1, v["count"]) for k, v in stages.items()}
    dom = max(stages, key=lambda k: stages[k]["ms"]) if stages else None
    n_launch = max(1, stages[dom]["count"] // args.steps) if dom else 1
    lane_bytes = raw_step // n_launch  # deflate lanes: every raw byte is one lane position
    alg = {  # algorithmic bytes per launch ("roofline accounting")
        "deflate.hash_prev": 3 * lane_bytes,          # lane byte in, u16 link out
        "deflate.profile": 11 * lane_bytes,           # lane byte + u16 link in, 2 x u32 profile out
        "deflate.parse_spec": 9 * lane_bytes,         # profile in (8 B/pos), ~1 B/pos of symbols out
        "deflate.emit": 4 * lane_bytes + comp_step // n_launch,
        "inflate.seq": (raw_step + comp_step) // n_launch,
    }
    roof = None
    if dom:
        t_launch = per_launch[dom] / 1e3
        a_bytes = alg.get(dom, (raw_step + comp_step) // n_launch)
        achieved = a_bytes / t_launch / 1e9
        traffic = limiter = None
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                tj = json.load(f)
            traffic = tj.get(wl.name, {}).get(dom)
            limiter = tj.get("limiters", {}).get(wl.name, {}).get(dom)
        except OSError:
            pass
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic, "algorithmic_bytes_per_launch": a_bytes,
                "launch_ms": per_launch[dom], "peak_source": peak_src}
        if limiter:  # the on-chip resource the kernel actually saturates (from the committed ncu capture)
            roof["limiter"] = limiter
    codec_roof = 2 * (raw_step + comp_step) / (ms_step / 1e3) / 1e9
    # SURVEY 8(d) per-direction figures: (raw + container) / t over the device stage timers of each side
    per_dir = None
    if stages:
        t_enc = sum(v["ms"] for k, v in stages.items() if k.startswith("deflate.")) / args.steps
        t_dec = sum(v["ms"] for k, v in stages.items() if k.startswith("inflate.")) / args.steps
        if t_enc > 0 and t_dec > 0:
            per_dir = {"enc_ms": t_enc, "enc_gbs": (raw_step + comp_step) / (t_enc / 1e3) / 1e9,
                       "dec_ms": t_dec, "dec_gbs": (raw_step + comp_step) / (t_dec / 1e3) / 1e9,
                       "source": "sum of the per-stage CUDA-event timers of each direction (per GPU)"}

    cpu = None
    bit_exact = None
    if not args.no_cpu_baseline and world == 1:
        try:
            from oracle.oracle import REF_SO, build
            if not os.path.exists(REF_SO):
                build()
            res, _ = reference_sample([wl.ref_job(0, 0, 8 * MiB)])
            r = res[0]
            cpu = {"value": r["raw"] / (r["enc_s"] + r["dec_s"]) / 1e9, "unit": "GB/s", "cores": 1,
                   "kind": "reference",
                   "sample": f"{r['raw']} B of {wl.name} data (the first slice) through the reference "
                             f"compress+decompress (enc {r['enc_s']:.2f} s, dec {r['dec_s']:.2f} s)"}
            if args.workload != "config3":  # config3's slice is one request, packed by the reference
                sb = wl.sample_bytes()[: r["raw"]]
                x0 = torch.frombuffer(bytearray(sb), dtype=torch.uint8).cuda()
            else:
                from paper_2604_21072_b200 import specdec
                st, kp = sd_request(0)
                x0 = specdec.DevicePacker(dev_id).pack_encode(torch.from_numpy(st).cuda(),
                                                              torch.from_numpy(kp).cuda(), [0, SD_NODES])
            c0 = dc.compress(x0, backend=1, split=True)
            bit_exact = hashlib.sha256(c0.cpu().numpy().tobytes()).hexdigest() == r["sha256"]
        except Exception as exc:  # keep the bench line even if the host leg fails
            cpu = {"value": None, "unit": "GB/s", "cores": 1, "kind": "reference", "sample": f"failed: {exc}"}

    mb = len(getattr(wl, "xs", [])) or 1
    line = {
        "metric": "codec GB/s (enc+dec, bit-exact) vs HBM roofline", "value": value, "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": wl.name, "description": wl.desc, "micro_batches": mb,
                   "raw_bytes_per_step_per_gpu": raw_step, "container_bytes_per_step_per_gpu": comp_step,
                   "ratio": comp_step / raw_step,
                   "l2": f"inputs {raw_step / MiB:.0f} MiB/step > 126 MB L2 (no flush needed)"
                   if raw_step > 126e6 else "inputs smaller than L2",
                   "parallelism": f"{world} stage(s), one boundary per GPU"
                   + ((", BBF1 frames written into the next GPU's HBM by the codec over NVLink (CUDA IPC),"
                       " lengths by NCCL" if HANDOFF == "p2p" and isinstance(wl, ActWorkload)
                       else ", BBF1 frames over NVLink (NCCL P2P ring)") if world > 1 else "")},
        "lossless": ok, "bit_exact_vs_reference": bit_exact,
        "tokens_per_s": world * wl.tokens_per_step / (ms_step / 1e3),
        "pipeline_tokens_per_s": wl.tokens_per_step / (ms_step / 1e3),
        "pipeline_steps_per_s": 1e3 / ms_step,
        "codec_roofline": {"achieved": codec_roof, "peak": hbm, "frac": codec_roof / hbm,
                           "definition": "2*(raw+container)/(t_enc+t_dec), SURVEY 8(d)",
                           "per_direction": per_dir},
        "roofline": roof, "stages_ms_per_step": {k: v["ms"] / args.steps for k, v in stages.items()},
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
