"""Multi-GPU stage hand-off, skipped on boxes with fewer than two GPUs.

* bench.py under torchrun, two ranks = two pipeline stages: the fused hand-off (the codec writes
  the frames into the next GPU's HBM through CUDA IPC, acked back-pressure on the inbox slots) and
  the NCCL frame hand-off; every rank checks the decoded frames against the previous rank's
  regenerated activations, after the timed steps and again after each of --verify-steps steps.
* the stage API's multi-GPU runner (beeplan::run_wire_local, cpp/wire.cpp) with its roles spread
  over two GPUs: frames cross GPUs as paced peer copies, sink reassembly bit-exact.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    import torch
    return torch.cuda.device_count()


def _bench(handoff, workload, port, extra=()):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "1",
           "--workload", workload, "--no-cpu-baseline", "--no-e2e", "--handoff", handoff, *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("handoff", ["p2p", "nccl"])
def test_two_stage_handoff_lossless(handoff):
    if _gpus() < 2:
        pytest.skip("needs two GPUs")
    line = _bench(handoff, "config1", 29611 + (handoff == "nccl"), ["--verify-steps", "3"])
    assert line["n_gpus"] == 2 and line["lossless"] is True
    assert line["verified_steps"] == 3


def test_two_stage_config2_fused_handoff_every_step_verified():
    """The headline workload across two GPUs: 8 x 64 MiB micro-batches per step through the fused
    IPC hand-off; stage 1 holds stage 0's containers, which must equal the reference's."""
    if _gpus() < 2:
        pytest.skip("needs two GPUs")
    line = _bench("p2p", "config2", 29613, ["--verify-steps", "3"])
    assert line["lossless"] is True and line["verified_steps"] == 3
    assert line["bit_exact_timed_step"]["match"] is True


def test_wire_runner_across_two_gpus():
    if _gpus() < 2:
        pytest.skip("needs two GPUs")
    exe = os.path.join(ROOT, "paper_2604_21072_b200", "beeplan")
    place = os.path.join(ROOT, "gpurun_out", "_placement_test.json")
    os.makedirs(os.path.dirname(place), exist_ok=True)
    r = subprocess.run([exe, "bench-wire", "--role", "local", "--stages", "2", "--payload", str(8 << 20),
                        "--micro-batches", "4", "--steps", "2", "--compress", "--devices", "0,1",
                        "--placement", place], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    doc = json.loads(r.stdout)
    assert doc["payload_ok"] is True and len(doc["hops"]) == 3
    where = json.load(open(place))
    assert where["role_devices"] == [0, 1, 0, 1] and all(where["hop_peer"])
