"""bench.py's GPU arm end to end on one B200: the timed config2 step (its micro-batches over
streams, or one batched call) reproduces the reference's containers and round-trips losslessly,
and the line carries the contract's keys."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("streams", [8, 1])
def test_bench_config2_step_bit_exact(streams):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "2", "--warmup", "1",
                        "--no-cpu-baseline", "--no-e2e", "--streams", str(streams)],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks",
              "stages_ms_per_step", "stages_source"):
        assert k in line, k
    assert line["lossless"] is True
    assert line["bit_exact_timed_step"]["match"] is True and line["bit_exact_timed_step"]["checked"] == 8
    assert line["gpu_launches"] > 0 and line["value"] > 0
    assert ("streams" in line["config"]["parallelism"]) == (streams > 1)
    assert line["roofline"]["kernel"].startswith("deflate.")
