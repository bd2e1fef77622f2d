"""The reference's own codec test cases (tests/cpp/test_codec.cpp, ported from
/root/reference/proj/tests/test_codec.cpp) run against the C++ drop-in
(libbeeplan_b200.so -> libbbcodec.so) on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_codec")


def test_dropin_binary_links_the_c_abi():
    assert os.path.exists(BIN), "run __graft_entry__.build()"
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libbeeplan_b200.so" in out and "libbbcodec.so" in out


@pytest.mark.gpu
def test_reference_codec_suite_on_b200():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
