"""Generate tests/golden/codec_golden.json from the REFERENCE itself.

Run in the build container (needs /root/reference):
    make -C oracle && python tests/golden/make_golden.py

Every entry is the unmodified reference codec (oracle/_ref/libbeeplan_ref.so,
compiled from /root/reference/proj/src/{codec,synth}.cpp against the pinned
system zlib 1.3) applied to a recipe input (tests/golden/inputs.py):
    container = serialize_container(compress(input, backend, split))
The fixture stores the container's length, SHA-256 and lane blob lengths, plus
the raw bytes of containers up to 256 B (the known-answer tests).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from inputs import make_input  # noqa: E402
from oracle.oracle import Oracle, Reference  # noqa: E402

SPECS = [
    # reference KAT shapes (test_codec.cpp:22-28,76-97,107-112)
    "const:0:0", "rand:2:1", "rand:4:2", "const:65536:66", "const:4096:0",
    # config 1: LLaMA-7B hidden state 1x128x4096 fp16 (BASELINE.json configs[0])
    "fp16:524288:1",
    # config 1 shape in bf16, config 3 tree (512x4096 fp16, seed 7)
    "bf16:524288:1", "fp16:2097152:7",
    # reference test_codec Gaussian case (seed 2024, 2^20 elements)
    "fp16:1048576:2024",
    # edge lengths around zlib's window / block boundaries
    "rand:258:3", "rand:262:4", "rand:4096:5", "rand:32506:6", "rand:32768:7",
    "rand:65274:8", "rand:65536:9", "rand:65538:10", "rand:131074:11",
    "skew:65274:12:3", "skew:65536:13:5", "skew:98304:14:17", "skew:200000:15:2",
    "period:100000:16:7", "period:70000:17:300", "runs:150000:18", "const:300000:0",
    "fp16:40000:3", "bf16:40000:4", "bf16:300000:5", "fp16:300001:6",
]


def entry(ref: Reference, spec: str, backend: int, split: bool, data: bytes) -> dict:
    c = ref.compress(data, backend, split)
    hl = int.from_bytes(c[15:23], "little")
    ll = int.from_bytes(c[23:31], "little")
    e = {"spec": spec, "backend": backend, "split": split, "len": len(c),
         "sha256": hashlib.sha256(c).hexdigest(), "high_len": hl, "low_len": ll}
    if len(c) <= 256:
        e["hex"] = c.hex()
    return e


def main() -> None:
    ref = Reference()
    orc = Oracle()
    out = {"generator": "tests/golden/make_golden.py",
           "reference": "/root/reference/proj/src/codec.cpp via oracle/_ref/libbeeplan_ref.so",
           "zlib": "system zlib 1.3 (zlib1g 1:1.3.dfsg-3.1ubuntu2.2)",
           "entries": [], "kat": {}}
    for spec in SPECS:
        data = make_input(spec, orc)
        if len(data) % 2:
            data = data[:-1]
        for backend in (0, 1):
            for split in (True, False):
                if backend == 0 and len(data) > 4096 and not split:
                    continue
                out["entries"].append(entry(ref, spec, backend, split, data))
        print(spec, "done", flush=True)
    # backend-level KATs (lane blobs)
    out["kat"]["deflate_empty"] = ref.encode(1, b"").hex()
    out["kat"]["deflate_hello_world"] = ref.encode(1, b"hello world").hex()
    out["kat"]["deflate_0x12"] = ref.encode(1, b"\x12").hex()
    out["kat"]["deflate_0x34"] = ref.encode(1, b"\x34").hex()
    # synth pinning: sha256 of the reference generator's bytes
    out["kat"]["synth_fp16_524288_1_sha256"] = hashlib.sha256(ref.synth_fp16(524288, 1)).hexdigest()
    out["kat"]["synth_fp16_1000000_424242_sha256"] = hashlib.sha256(
        ref.synth_fp16(1000000, 424242)).hexdigest()
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "codec_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path, len(out["entries"]), "entries")


if __name__ == "__main__":
    main()
