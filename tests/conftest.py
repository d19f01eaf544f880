import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(ROOT, "tests", "golden", "paper_fixtures.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def cascade():
    import oracle
    from synth import arch, weights
    return oracle.Cascade(arch.NETS, weights.make_cascade_weights())
