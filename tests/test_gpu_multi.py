"""Multi-GPU stage hand-off: two ranks on two GPUs, each a pipeline stage.
Runs bench.py under torchrun with the fused hand-off (codec writes the frames into the next
GPU's HBM via CUDA IPC) and the NCCL frame hand-off; both must be lossless (every rank checks
the decoded frames against the previous rank's regenerated activations).  Skipped on boxes
with fewer than two GPUs."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("handoff", ["p2p", "nccl"])
def test_two_stage_handoff_lossless(handoff):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29" + str(611 + (handoff == "nccl")),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "1",
           "--workload", "config1", "--no-cpu-baseline", "--no-e2e", "--handoff", handoff]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["lossless"] is True
