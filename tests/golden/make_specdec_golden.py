"""Generate tests/golden/specdec_golden.json from the REFERENCE itself.

Run in the build container (needs /root/reference):
    make -C oracle && python tests/golden/make_specdec_golden.py

Entries: the unmodified reference (oracle/_ref/libbeeplan_ref.so, compiled from
/root/reference/proj/src/specdec.cpp + codec.cpp) applied to token-tree batches
rebuilt from spec strings (tests/golden/inputs.py:sd_tree):
    packed    = encode_packed(pack(kept rows per request))      specdec.cpp:153-165,192-198
    container = serialize_container(compress(packed, deflate, split))
plus decode_packed error cases (status + message, specdec.cpp:200-220) and the
reference's own test_specdec.cpp pack/unpack cases.
"""
from __future__ import annotations

import hashlib
import json
import os
import struct
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from inputs import sd_tree  # noqa: E402
from oracle.oracle import OracleError, Reference  # noqa: E402

SPECS = [
    "sdtree:1:1:1:1:100:f32", "sdtree:3:4:3:2:70:f32", "sdtree:5:6:1:3:50:f32",
    "sdtree:4:16:64:4:60:special", "sdtree:2:64:4096:5:60:bf16up", "sdtree:8:40:257:6:30:f32",
    "sdtree:16:3:8:7:0:f32", "sdtree:4:9:5:8:100:special",
    # config 3: tree width 64 x depth 8 = 512 nodes, d = 4096, two requests
    "sdtree:2:512:4096:9:60:bf16up",
]


def err(ref, data, dim):
    try:
        ref.decode_packed(data, dim)
        return {"status": 0}
    except OracleError as e:
        return {"status": e.status, "message": str(e).split(": ", 1)[1]}


def main() -> None:
    ref = Reference()
    out = {"generator": "tests/golden/make_specdec_golden.py",
           "reference": "/root/reference/proj/src/specdec.cpp via oracle/_ref/libbeeplan_ref.so",
           "entries": [], "decode_cases": []}
    for spec in SPECS:
        rows, keep, request_rows, per_request = sd_tree(spec)
        packed = ref.pack_encode(per_request)
        c = ref.compress(packed, 1, True)
        e = {"spec": spec, "packed_len": len(packed), "packed_sha256": hashlib.sha256(packed).hexdigest(),
             "container_len": len(c), "container_sha256": hashlib.sha256(c).hexdigest()}
        if len(packed) <= 256:
            e["packed_hex"] = packed.hex()
        out["entries"].append(e)
        print(spec, len(packed), len(c), flush=True)
    # decode_packed error parity (specdec.cpp:200-220) on hand-made images
    u32 = lambda *v: struct.pack(f"<{len(v)}I", *v)  # noqa: E731
    f32 = lambda *v: struct.pack(f"<{len(v)}f", *v)  # noqa: E731
    cases = [
        ("empty", b"", 2), ("short_count", b"\x01\x00\x00", 2), ("zero_count", u32(0), 2),
        ("truncated_offsets", u32(3, 0, 1), 2), ("ok_empty_batch", u32(1, 0), 2),
        ("ok_two", u32(3, 0, 1, 2) + f32(1, 2, 3, 4), 2), ("payload_short", u32(3, 0, 1, 2) + f32(1, 2, 3), 2),
        ("payload_odd_bytes", u32(2, 0, 1) + f32(1, 2) + b"\x00", 2), ("nonzero_start", u32(2, 1, 1) + f32(1, 2), 2),
        ("decreasing", u32(3, 0, 2, 1) + f32(1, 2), 2), ("dim0_ok", u32(2, 0, 5), 0),
        ("dim0_payload", u32(2, 0, 5) + f32(1), 0), ("big_count", u32(0xFFFFFFFF, 0), 1),
        ("ok_ragged", u32(4, 0, 0, 3, 3) + f32(*range(9)), 3),
    ]
    for name, data, dim in cases:
        out["decode_cases"].append({"name": name, "hex": data.hex(), "hidden_dim": dim, **err(ref, data, dim)})
    # test_specdec.cpp pack/unpack cases
    out["pack_offsets_0346"] = ref.pack_encode([[[1.0, 2.0]] * 3, [[3.0, 4.0]], [[5.0, 6.0]] * 2]).hex()
    try:
        ref.pack_encode([[[1.0, 2.0]], [[1.0, 2.0, 3.0]]])
        out["pack_ragged_status"] = 0
    except OracleError as e:
        out["pack_ragged_status"] = e.status
        out["pack_ragged_message"] = str(e).split(": ", 1)[1]
    out["unpack_checks"] = [{"offsets": o, "hidden_dim": d, "payload": p, "status": ref.unpack_check(o, d, p)}
                            for o, d, p in [([0, 1, 3], 2, 6), ([1, 3], 2, 4), ([0, 3, 2], 1, 3), ([0, 2], 2, 3),
                                            ([], 1, 0), ([0, 4], 0, 0), ([0, 4], 0, 1), ([0], 7, 0)]]
    with open(os.path.join(ROOT, "tests", "golden", "specdec_golden.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
