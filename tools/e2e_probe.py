"""Where the plugin e2e's time goes (config2): 8 host threads, steps streamed, each thread one
micro-batch per step, (a) through bb_compress_host / bb_decompress_host with page-locked buffers
(the bench's e2e), (b) through the stream-ordered device calls on HBM-resident buffers (same
per-micro-batch split, no copies), (c) the batched device call over all 8 micro-batches."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_21072_b200 import codec, synth, workloads  # noqa: E402

STEPS, T = 4, int(os.environ.get("THREADS", "8"))
host = [workloads.config2_micro(synth.gaussian, 0, i) for i in range(workloads.C2_MICRO)]
dev = [torch.frombuffer(bytearray(h), dtype=torch.uint8).cuda() for h in host]
dc = codec.DeviceCodec(0)
bound = dc.compress_bound(len(host[0]))


def worker(t, nsteps):
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    out = torch.empty(bound, dtype=torch.uint8, device="cuda")
    back = torch.empty(len(host[0]), dtype=torch.uint8, device="cuda")
    with torch.cuda.stream(s):
        for _ in range(nsteps):
            for k in range(t, len(dev), T):
                n = dc.compress_into(dev[k], out, stream=s)
                dc.decompress_into(out[:n], back, stream=s)
        s.synchronize()


ex = ThreadPoolExecutor(T)
list(ex.map(worker, range(T), [1] * T))
torch.cuda.synchronize()
t0 = time.perf_counter()
list(ex.map(worker, range(T), [STEPS] * T))
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / STEPS
print(f"(b) device calls per micro-batch, {T} threads streamed: {1e3 * dt:.2f} ms/step")

t0 = time.perf_counter()
for _ in range(STEPS):
    list(ex.map(worker, range(T), [1] * T))
torch.cuda.synchronize()
print(f"(b2) the same with every step joined: {1e3 * (time.perf_counter() - t0) / STEPS:.2f} ms/step")

# (b3) per step: all compresses over the threads, join, then all decompresses, join (the
# multi-GPU step's shape: the length doorbell sits between the two phases)
cbuf = [torch.empty(bound, dtype=torch.uint8, device="cuda") for _ in dev]
dbuf = [torch.empty_like(d) for d in dev]
clen = [0] * len(dev)
sts = [torch.cuda.Stream() for _ in range(T)]


def ph_c(t):
    torch.cuda.set_device(0)
    for k in range(t, len(dev), T):
        clen[k] = dc.compress_into(dev[k], cbuf[k], stream=sts[t])
    sts[t].synchronize()


def ph_d(t):
    torch.cuda.set_device(0)
    for k in range(t, len(dev), T):
        dc.decompress_into(cbuf[k][:clen[k]], dbuf[k], stream=sts[t])
    sts[t].synchronize()


list(ex.map(ph_c, range(T)))
list(ex.map(ph_d, range(T)))
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(STEPS):
    list(ex.map(ph_c, range(T)))
    list(ex.map(ph_d, range(T)))
torch.cuda.synchronize()
print(f"(b3) compress phase then decompress phase, {T} threads each: {1e3 * (time.perf_counter() - t0) / STEPS:.2f} ms/step")

outs = [torch.empty(bound, dtype=torch.uint8, device="cuda") for _ in dev]
backs = [torch.empty_like(d) for d in dev]
lens = dc.compress_batch(dev, outs)
dc.decompress_batch([o[:n] for o, n in zip(outs, lens)], backs)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(STEPS):
    lens = dc.compress_batch(dev, outs)
    dc.decompress_batch([o[:n] for o, n in zip(outs, lens)], backs)
torch.cuda.synchronize()
print(f"(c) batched device call: {1e3 * (time.perf_counter() - t0) / STEPS:.2f} ms/step")

# (d) copies only: the plugin e2e's host traffic per step (raw in, container out, container in,
# raw out per micro-batch) from page-locked memory, 8 threads streamed, no codec
pin_raw = [torch.empty(len(h), dtype=torch.uint8).pin_memory() for h in host]
pin_c = [torch.empty(n, dtype=torch.uint8).pin_memory() for n in lens]
dev_c = [o[:n] for o, n in zip(outs, lens)]


def copier(t, nsteps):
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(nsteps):
            for k in range(t, len(dev), T):
                dev[k].copy_(pin_raw[k], non_blocking=True)
                pin_c[k].copy_(dev_c[k], non_blocking=True)
                dev_c[k].copy_(pin_c[k], non_blocking=True)
                pin_raw[k].copy_(backs[k], non_blocking=True)
                s.synchronize()
        s.synchronize()


list(ex.map(copier, range(T), [1] * T))
t0 = time.perf_counter()
list(ex.map(copier, range(T), [STEPS] * T))
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / STEPS
gb = 2 * (sum(len(h) for h in host) + sum(lens)) / 1e9
print(f"(d) copies only: {1e3 * dt:.2f} ms/step ({gb / dt:.1f} GB/s both directions)")
