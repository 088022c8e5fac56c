import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def orc():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def golden():
    import json
    import numpy as np
    g = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(g, "protocol.json")) as f:
        rec = json.load(f)
    rec["final_params"] = np.fromfile(os.path.join(g, "final_params.f32"), np.float32)
    rec["test_pred"] = np.fromfile(os.path.join(g, "test_pred.u8"), np.uint8).astype(np.int32)
    rec["cells"] = np.fromfile(os.path.join(g, "cells.f32"), np.float32).reshape(8, 3899)
    with open(os.path.join(g, "ops.json")) as f:
        rec["ops"] = json.load(f)
    return rec


@pytest.fixture(scope="session")
def zhang_sets(orc):
    tr = orc.make_set(10000, 1)
    te = orc.make_set(10000, 2)
    return tr, te
