import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a); run with -m gpu")
    config.addinivalue_line("markers", "slow: large-config checks (minutes)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import Oracle
    return Oracle(threads=0)


@pytest.fixture(scope="session")
def golden():
    import json
    import numpy as np
    g = {}
    for name in ("refkat", "trials", "configs", "with_plan"):
        with open(os.path.join(GOLDEN, f"{name}.json")) as f:
            g[name] = json.load(f)
    g["cfg1"] = dict(np.load(os.path.join(GOLDEN, "cfg1.npz")))
    return g
