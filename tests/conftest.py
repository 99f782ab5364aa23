import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    _ensure_library()


def _ensure_library():
    """Build libkbe200.so (nvcc, sm_100a) when it is missing or older than its sources, so a
    fresh checkout runs the suite; on a GPU box the prebuilt library travels in-tree."""
    pkg = os.path.join(ROOT, "paper_2505_19467_b200")
    lib = os.path.join(pkg, "libkbe200.so")
    srcs = [os.path.join(pkg, "csrc", "kbe200.cu"), os.path.join(ROOT, "include", "kbe200.h")]
    if os.path.exists(lib) and all(os.path.getmtime(lib) >= os.path.getmtime(x) for x in srcs):
        return
    import shutil
    if shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"):
        return   # nothing to build with: the ABI checks will report the missing library
    import __graft_entry__
    __graft_entry__.build()


def rel_err(a, b):
    """max|a-b| / max|b|, the reference's tolerance helper (test_selfenergy.py:101-103)."""
    a = np.asarray(a)
    b = np.asarray(b)
    scale = max(float(np.abs(b).max(initial=0.0)), 1e-300)
    return float(np.abs(a - b).max(initial=0.0)) / scale


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture
def golden():
    return load_golden
