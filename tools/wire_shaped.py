"""Shaped multi-GPU stage-runner measurements (profiles/r2_wire_*.json).

Runs `beeplan bench-wire --role local` (the stage API's multi-GPU runner, cpp/wire.cpp: one GPU
per role, frames in HBM, ShapedWriter-paced peer copies) over a grid of link rates, micro-batch
counts and compression on/off, at the GPU count this box has, and writes one JSON document:

    python tools/wire_shaped.py --out gpurun_out/r2_wire_2gpu.json [--payload-mib 64] [--rates 100,500]

The reference's own definition of throughput is kept (steps * 1000 / end_to_end_ms,
wire.cpp:678-679); pipelined rows/s = steps * payload / 2 / d / e2e (d = hidden size).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_2604_21072_b200", "beeplan")


def run(payload, micro, steps, stages, rate_mbps, compress, devices, compute_ms=0.0):
    cmd = [EXE, "--seed", "5", "bench-wire", "--role", "local", "--payload", str(payload), "--micro-batches",
           str(micro), "--steps", str(steps), "--stages", str(stages), "--devices", devices,
           "--compute-ms", str(compute_ms)]
    if rate_mbps:
        cmd += ["--shape", f"{rate_mbps},0"]
    if compress:
        cmd.append("--compress")
    place = os.path.join(ROOT, "gpurun_out", f"_place_{os.getpid()}.json")
    cmd += ["--placement", place]
    t0 = time.time()
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=3600)
    wall = time.time() - t0
    if r.returncode != 0:
        return {"error": r.stderr[-2000:], "cmd": " ".join(cmd)}
    doc = json.loads(r.stdout)
    where = json.load(open(place))
    os.unlink(place)
    return {"payload_bytes": payload, "micro_batches": micro, "steps": steps, "stages": stages,
            "rate_mbps": rate_mbps, "compress": compress, "compute_ms": compute_ms,
            "end_to_end_ms": doc["end_to_end_ms"], "payload_ok": doc["payload_ok"],
            "throughput_steps_per_s": doc["summary"]["throughput_tokens_per_s"],
            "hops": doc["hops"], "source_codec_ms": doc["source_codec_ms"], "sink_codec_ms": doc["sink_codec_ms"],
            "role_devices": where["role_devices"], "hop_bytes": where["hop_bytes"], "hop_peer": where["hop_peer"],
            "wall_s": round(wall, 2)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--payload-mib", type=int, default=64)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--rates", default="100")
    ap.add_argument("--micro", default="1,8")
    ap.add_argument("--hidden", type=int, default=8192)
    ap.add_argument("--sizes-mib", default="",
                    help="config5 sweep: payload sizes (MiB, d=8192 fp16 rows), run at --micro[0] compressed "
                         "and uncompressed, one step each")
    args = ap.parse_args()
    import torch
    g = torch.cuda.device_count()
    devices = ",".join(str(d) for d in range(g))
    stages = max(0, g - 2)  # source + stages + sink = one role per GPU
    res = {"gpus": g, "devices": devices, "stages": stages, "runs": []}
    if args.sizes_mib:
        micro = int(args.micro.split(",")[-1])
        for mib in [int(x) for x in args.sizes_mib.split(",")]:
            for compress in (False, True):
                r = run(mib << 20, micro, 1, stages, float(args.rates.split(",")[0]), compress, devices)
                if "end_to_end_ms" in r:
                    r["pipelined_rows_per_s"] = r["payload_bytes"] / 2 / args.hidden / (r["end_to_end_ms"] / 1e3)
                res["runs"].append(r)
                print(json.dumps({k: r.get(k) for k in ("payload_bytes", "compress", "end_to_end_ms", "payload_ok",
                                                        "error")}), flush=True)
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)
        return 0
    for rate in [float(x) for x in args.rates.split(",")]:
        for micro in [int(x) for x in args.micro.split(",")]:
            for compress in (False, True):
                r = run(args.payload_mib << 20, micro, args.steps, stages, rate, compress, devices)
                if "end_to_end_ms" in r:
                    r["pipelined_rows_per_s"] = args.steps * r["payload_bytes"] / 2 / args.hidden / (
                        r["end_to_end_ms"] / 1e3)
                res["runs"].append(r)
                print(json.dumps({k: r.get(k) for k in ("rate_mbps", "micro_batches", "compress", "end_to_end_ms",
                                                        "payload_ok", "error")}), flush=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
    return 0


if __name__ == "__main__":
    sys.exit(main())
