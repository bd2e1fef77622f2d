"""Generate tests/golden/fullsize_golden.json: the REFERENCE's containers at the full
BASELINE.json config sizes (TEST INFRASTRUCTURE; needs /root/reference, run here).

    make -C oracle && python tests/golden/make_fullsize_golden.py [-j 8]

Every entry is serialize_container(compress(input, kBackendDeflate, split=true)) of the
unmodified reference codec (oracle/_ref/libbeeplan_ref.so = /root/reference/proj/src/
codec.cpp:163-179 + zlib 1.3 compress2 level 6, codec.cpp:17-25) on the exact bytes the
bench times (paper_2604_21072_b200/workloads.py), generated here with the ORACLE's synth
(pinned to the reference generator).  For config3 the packed image itself is the
reference's encode_packed(pack(...)) (specdec.cpp:153-198).  The fixture keeps
SHA-256 + sizes only; the GPU tests rebuild the inputs on the box and compare.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_2604_21072_b200 import workloads as W  # noqa: E402


def _synth():
    from oracle.oracle import Oracle
    orc = Oracle()
    return lambda n, seed, bf16: orc.synth_bf16(n, seed) if bf16 else orc.synth_fp16(n, seed)


def _input(job):
    synth = _synth()
    kind = job["config"]
    if kind == "config2":
        return W.config2_micro(synth, job["rank"], job["index"])
    if kind == "config4":
        return W.kv_chunk(synth, job["chunk_id"])
    if kind == "config5":
        data = W.sweep_tensor(synth, job["size_index"], job["tensor_bytes"], job.get("rank", 0))
        o = job["offset"]
        return data[o:o + job["piece_bytes"]]
    if kind == "config3":
        from oracle.oracle import Reference
        ref = Reference()
        per = []
        for r in range(job["first_request"], job["first_request"] + job["requests"]):
            st, kp = W.sd_request(synth, r)
            per.append([st[i] for i in range(st.shape[0]) if kp[i]])
        return ref.pack_encode(per)
    if kind == "config1":
        return synth(W.C1_ELEMS, 1, False)
    raise ValueError(kind)


def _run(job):
    from oracle.oracle import Reference
    ref = Reference()
    data = _input(job)
    t0 = time.perf_counter()
    c = ref.compress(data, 1, True)
    t1 = time.perf_counter()
    e = dict(job)
    e.update({"raw_len": len(data), "raw_sha256": hashlib.sha256(data).hexdigest(),
              "len": len(c), "sha256": hashlib.sha256(c).hexdigest(),
              "high_len": int.from_bytes(c[15:23], "little"), "low_len": int.from_bytes(c[23:31], "little"),
              "ref_compress_s": round(t1 - t0, 2)})
    print(f"{job['name']}: {len(data)} -> {len(c)} B in {t1 - t0:.1f} s", flush=True)
    return e


def jobs():
    out = [{"config": "config1", "name": "config1 [1,128,4096] fp16 seed 1"}]
    for i in range(W.C2_MICRO):
        out.append({"config": "config2", "name": f"config2 stage 0 micro-batch {i} (seed {W.config2_seed(0, i)})",
                    "rank": 0, "index": i})
    for cid in W.kv_layer_ids(0):
        out.append({"config": "config4", "name": f"config4 layer 0 chunk {cid}", "chunk_id": cid})
    out.append({"config": "config3", "name": "config3 32-request packed token-tree step",
                "first_request": 0, "requests": W.SD_REQUESTS})
    for si, size in enumerate(W.sweep_sizes(1024)):
        for o in range(0, size, W.SWEEP_PIECE):
            piece = min(W.SWEEP_PIECE, size - o)
            out.append({"config": "config5", "name": f"config5 {size // W.MiB} MiB tensor, piece at {o}",
                        "size_index": si, "tensor_bytes": size, "offset": o, "piece_bytes": piece})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    js = jobs()
    order = sorted(range(len(js)), key=lambda k: -js[k].get("piece_bytes", 64 * W.MiB))  # big first
    with mp.get_context("fork").Pool(args.j, maxtasksperchild=1) as pool:
        res = pool.map(_run, [js[k] for k in order], chunksize=1)
    back = [None] * len(js)
    for k, r in zip(order, res):
        back[k] = r
    doc = {"generator": "tests/golden/make_fullsize_golden.py",
           "reference": "/root/reference/proj/src/codec.cpp (+ specdec.cpp for config3) via oracle/_ref",
           "zlib": "system zlib 1.3 (zlib1g 1:1.3.dfsg-3.1ubuntu2.2), compress2 level 6",
           "inputs": "paper_2604_21072_b200/workloads.py recipes, oracle synth",
           "entries": back}
    path = os.path.join(HERE, "fullsize_golden.json")
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
    print("wrote", path, len(back), "entries")


if __name__ == "__main__":
    main()
