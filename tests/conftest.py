import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def pytest_collection_modifyitems(config, items):
    import torch
    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def orc():
    from oracle import c_oracle
    return c_oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle import ref_lib
    r = ref_lib()
    if r is None:
        pytest.skip("reference library (oracle/_ref/libjenga_ref.so) not built on this machine")
    return r


def load_golden(name):
    import json
    with open(GOLDEN / name) as f:
        return json.load(f)
