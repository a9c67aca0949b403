import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
PIPELINE_CASES = ("blobs_d64", "gauss_d64", "gauss_d128", "dups_d64", "tiny_d16")
GPU_PIPELINE_CASES = ("blobs_d64", "gauss_d64", "gauss_d128", "dups_d64")  # d in {64,128}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


@pytest.fixture(scope="session")
def golden():
    return load_golden
