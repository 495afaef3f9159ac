import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden_arrays():
    return np.load(os.path.join(GOLDEN, "golden_arrays.npz"))


@pytest.fixture(scope="session")
def golden_cases():
    with open(os.path.join(GOLDEN, "golden_cases.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def trace_golden():
    """Reference stability reports / classifications / load errors on the
    committed FXTK fixtures (tests/golden/make_golden_trace.py)."""
    with open(os.path.join(GOLDEN, "trace_golden.json")) as fh:
        return json.load(fh)


def golden_blob(name):
    with open(os.path.join(GOLDEN, name), "rb") as fh:
        return fh.read()
