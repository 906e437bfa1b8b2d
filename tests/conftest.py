import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def load_cases(stem):
    """Golden cases written by tests/golden/make_golden.py (reference outputs)."""
    with open(os.path.join(GOLDEN, stem + ".json")) as fh:
        metas = json.load(fh)
    data = np.load(os.path.join(GOLDEN, stem + ".npz"))
    shared = {}
    cases = []
    for i, meta in enumerate(metas):
        arrays = {k.split("_", 1)[1]: data[k] for k in data.files if k.startswith(f"c{i}_")}
        if "inputs" in meta:
            if "a" in arrays:
                shared[meta["inputs"]] = (arrays["a"], arrays["b"])
            arrays["a"], arrays["b"] = shared[meta["inputs"]]
        if "output" in meta:
            if "out" in arrays:
                shared[meta["output"]] = arrays["out"]
            arrays["out"] = shared[meta["output"]]
        cases.append((meta, arrays))
    return cases


@pytest.fixture(scope="session")
def execute_cases():
    return load_cases("execute_cases")


@pytest.fixture(scope="session")
def pipeline_cases():
    return load_cases("pipeline_cases")
