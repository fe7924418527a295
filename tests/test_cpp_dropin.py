"""The C++ host API (include/riffle_b200.hpp) as a drop-in for the reference's
riffle:: loader / pre-shuffle API: tests/cpp/test_dropin.cpp drives both
libraries side by side (oracle/_ref/test_dropin, built by `make -C oracle
dropin` where /root/reference exists; the binary travels to the GPU box)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "oracle" / "_ref" / "test_dropin"


def _run(*args):
    if not BIN.exists():
        pytest.skip("oracle/_ref/test_dropin not built (needs /root/reference at build time)")
    p = subprocess.run([str(BIN), *args], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "0 failures" in p.stdout
    return p.stdout


def test_cpp_dropin_host():
    out = _run()
    assert "[pass] plan_epoch" in out


@pytest.mark.gpu
def test_cpp_dropin_device():
    out = _run("--gpu")
    assert "[pass] BatchIterator" in out and "[pass] run_shuffle" in out
