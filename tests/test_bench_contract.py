"""bench.py's JSON contract on the CPU: the reference arm (`--impl reference`)
runs the compiled reference here, so its line can be checked end to end.
The GPU arm's line is exercised by the driver on a B200."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(not (ROOT / "oracle" / "_ref" / "libriffle_ref.so").exists(), reason="reference not built")
def test_reference_arm_preshuffle_line(tmp_path):
    env = dict(os.environ, RIFFLE_BENCH_DIR=str(tmp_path), RIFFLE_CFG5_REF_ROWS="1500")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--workload", "cfg5",
                          "--steps", "4", "--warmup", "3"], env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["metric"] == "preshuffle GB/s" and d["unit"] == "GB/s"
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_bench_help_lists_workloads():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--help"], capture_output=True, text=True,
                         timeout=120)
    assert out.returncode == 0
    for w in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
        assert w in out.stdout
