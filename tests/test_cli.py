"""The `beeplan` CLI (codec + bench-wire subcommands) against the reference's
cli_tests.sh:74-104 checks and exit-code contract (beeplan_main.cpp:326-351)."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2604_21072_b200", "beeplan")


def run(*args, **kw):
    return subprocess.run([BIN, *map(str, args)], capture_output=True, text=kw.pop("text", True), timeout=600, **kw)


@pytest.fixture(scope="module", autouse=True)
def binary():
    if not os.path.exists(BIN):
        pytest.skip("beeplan CLI not built (run __graft_entry__.build())")


def test_usage_errors_exit_2():
    assert run("--help").returncode == 0
    assert run().returncode == 2
    assert run("compress").returncode == 2                  # missing positionals
    assert run("--bogus", "entropy", "x").returncode == 2   # unknown option
    assert run("--format", "xml", "entropy", "x").returncode == 2
    assert run("entropy", "--seed").returncode == 2         # option without its value


def test_domain_errors_exit_1_with_json_line(tmp_path):
    r = run("compress", tmp_path / "missing.fp16", tmp_path / "out.bbc")
    assert r.returncode == 1
    assert json.loads(r.stderr.strip().splitlines()[-1]) == {"error": f"cannot open file: {tmp_path / 'missing.fp16'}"}
    r = run("bench-wire", "--role", "source")
    assert r.returncode == 1 and "error" in json.loads(r.stderr.strip().splitlines()[-1])
    r = run("bench-wire", "--role", "nope")
    assert r.returncode == 1
    assert json.loads(r.stderr.strip())["error"] == "--role: expected source|stage|sink|local"


@pytest.mark.gpu
def test_cli_codec_matches_cli_tests_sh(tmp_path, reference):
    zero = tmp_path / "zero.fp16"
    zero.write_bytes(bytes(8192))
    r = run("entropy", zero)
    assert r.returncode == 0 and '"raw_entropy": 0.0' in r.stdout
    act = tmp_path / "act.fp16"
    data = np.random.default_rng(5).bytes(131072)
    act.write_bytes(data)
    assert run("compress", act, tmp_path / "act.bbc").returncode == 0
    assert (tmp_path / "act.bbc").read_bytes() == reference.compress(data, 1, True)  # bit-exact container
    assert run("decompress", tmp_path / "act.bbc", tmp_path / "act.out").returncode == 0
    assert (tmp_path / "act.out").read_bytes() == data
    assert run("compress", "--backend", "identity", "--no-split", act, tmp_path / "act.id").returncode == 0
    assert os.path.getsize(tmp_path / "act.id") == 131072 + 31
    # corrupt container -> CorruptContainer, exit 1
    bad = bytearray((tmp_path / "act.bbc").read_bytes())
    bad[0] ^= 0xff
    (tmp_path / "bad.bbc").write_bytes(bytes(bad))
    r = run("decompress", tmp_path / "bad.bbc", tmp_path / "x")
    assert r.returncode == 1 and json.loads(r.stderr.strip())["error"] == "container: bad magic"


@pytest.mark.gpu
def test_cli_entropy_document(tmp_path):
    from paper_2604_21072_b200 import codec, synth
    raw = synth.gaussian(65536, 3)
    f = tmp_path / "g.fp16"
    f.write_bytes(raw)
    r = run("--output", tmp_path / "e.json", "entropy", f)
    assert r.returncode == 0
    doc = json.loads((tmp_path / "e.json").read_text())
    rep = codec.analyze(raw, 1)
    assert doc["raw_size"] == rep.raw_size and doc["split_mode_compressed"] == rep.split_mode_compressed
    assert sorted(doc) == sorted(["raw_entropy", "high_entropy", "low_entropy", "raw_size", "lane_size",
                                  "raw_mode_compressed", "high_lane_compressed", "low_lane_compressed",
                                  "split_mode_compressed", "ratio"])


@pytest.mark.gpu
def test_cli_bench_wire_local_lossless(tmp_path):
    r = run("--seed", "7", "bench-wire", "--role", "local", "--payload", "65536", "--micro-batches", "2",
            "--steps", "1", "--shape", "200,0", "--compute-ms", "1", "--stages", "1")
    assert r.returncode == 0, r.stderr
    assert '"payload_ok": true' in r.stdout
    doc = json.loads(r.stdout)
    assert sorted(doc) == ["end_to_end_ms", "hops", "payload_ok", "sink_codec_ms", "source_codec_ms", "summary"]
    assert sorted(doc["summary"]) == ["completion_ms", "hops", "stages", "step_ms", "throughput_tokens_per_s"]
    assert [h["frames"] for h in doc["hops"]] == [2, 2]
    # compressed hand-off through two relay stages, shaped to 20 Mbps
    r = run("bench-wire", "--role", "local", "--payload", "416400", "--micro-batches", "4", "--steps", "2",
            "--shape", "20,1", "--compress", "--stages", "2")
    assert r.returncode == 0, r.stderr
    doc = json.loads(r.stdout)
    assert doc["payload_ok"] is True and doc["source_codec_ms"] > 0 and doc["sink_codec_ms"] > 0
    assert len(doc["summary"]["stages"]) == 2 and [h["frames"] for h in doc["hops"]] == [8, 8, 8]
