"""The workload recipes shared by bench.py, the GPU parity tests and the full-size golden generator
(paper_2604_21072_b200/workloads.py) against the BASELINE.json configs and the committed fixture."""
import json
import os

from paper_2604_21072_b200 import workloads as W

HERE = os.path.dirname(os.path.abspath(__file__))


def test_shapes_match_baseline_configs():
    assert W.C1_ELEMS * 2 == 1 << 20                         # [1,128,4096] fp16
    assert W.C2_MICRO == 8 and W.C2_ELEMS * 2 == 64 << 20     # 8 x [16,512,4096] bf16
    assert W.SD_NODES == 64 * 8 and W.SD_DIM == 4096          # tree width 64, depth 8, d=4096
    assert W.KV_CTX * W.KV_DIM * 2 == 40 << 20                # 13B KV chunk [4096, 5120] fp16
    assert W.sweep_sizes(4096)[0] == 1 << 20 and W.sweep_sizes(4096)[-1] == 4 << 30
    assert W.kv_layer_ids(0) == list(range(64)) and W.kv_layer_ids(1)[0] == 64


def test_fixture_covers_every_timed_container():
    gold = json.load(open(os.path.join(HERE, "golden", "fullsize_golden.json")))["entries"]
    by = {}
    for e in gold:
        by.setdefault(e["config"], []).append(e)
    assert [e["index"] for e in by["config2"]] == list(range(8))
    assert all(e["raw_len"] == 64 << 20 for e in by["config2"])
    assert [e["chunk_id"] for e in by["config4"]] == W.kv_layer_ids(0)
    assert by["config3"][0]["requests"] == W.SD_REQUESTS
    sizes = sorted({e["tensor_bytes"] for e in by["config5"]})
    assert sizes == W.sweep_sizes(1024)
    assert sum(e["piece_bytes"] for e in by["config5"] if e["tensor_bytes"] == 1 << 30) == 1 << 30


def test_small_recipes_are_deterministic():
    calls = []

    def synth(n, seed, bf16):
        calls.append((n, seed, bf16))
        return bytes(2 * n)

    W.config2_micro(synth, 1, 3)
    W.kv_chunk(synth, 65)
    W.sweep_tensor(synth, 2, 2 << 20, rank=1)
    assert calls == [(W.C2_ELEMS, 2003, True), (W.KV_CTX * W.KV_DIM, 65, False),
                     (1 << 19, 50000 + 8192 + 0 + 1000000, False), (1 << 19, 50000 + 8192 + 1 + 1000000, False)]


def test_module_level_codec_device_follows_env(monkeypatch):
    from paper_2604_21072_b200 import codec
    monkeypatch.setenv("BEEPLAN_CUDA_DEVICE", "3")
    assert codec._device() == 3
    monkeypatch.delenv("BEEPLAN_CUDA_DEVICE")
    assert codec._device() == 0  # torch has not initialised CUDA in the CPU suite
