import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(GOLDEN_DIR, "golden.npz"))


@pytest.fixture(scope="session")
def golden_meta():
    import json

    with open(os.path.join(GOLDEN_DIR, "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_alg2():
    return np.load(os.path.join(GOLDEN_DIR, "golden_alg2.npz"))


ALG2_TAGS = ["m8_b2", "m32_b2", "m8_default", "dup_col", "zero_col", "with_b", "with_x0", "m96_b16"]
ALG2_KW = {"m8_b2": dict(block_width=2), "m32_b2": dict(block_width=2), "m8_default": {},
           "dup_col": dict(block_width=2), "zero_col": dict(block_width=3), "with_b": {},
           "with_x0": dict(block_width=5), "m96_b16": dict(block_width=16)}
