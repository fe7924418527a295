import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (run on the B200 box)")


@pytest.fixture(scope="session")
def golden():
    return json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())


@pytest.fixture(scope="session")
def golden_stores(golden, tmp_path_factory):
    """The golden stores, regenerated with the product's synth_store (byte-identical
    to the reference's, see test_host.py::test_synth_byte_identical)."""
    import paper_2604_01949_b200 as R
    d = tmp_path_factory.mktemp("golden_stores")
    out = {}
    for name, c in golden["stores"].items():
        R.synth_store(d / name, R.SynthConfig(c["n_obs"], c["n_var"], c["layout"], c["value_dtype"],
                                              c.get("index_dtype", "u32"), c["density"], c["seed"],
                                              c["chunk_rows"], c["cps"]))
        out[name] = d / name
    return out


def fnv(arrs, h=0xCBF29CE484222325):
    from oracle.oracle import Orc
    import numpy as np
    for a in arrs:
        h = Orc.fnv1a64(np.ascontiguousarray(a), h)
    return h
