import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    data = np.load(os.path.join(GOLDEN_DIR, "bump40.npz"))
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as f:
        meta = json.load(f)
    return {k: data[k] for k in data.files}, meta


@pytest.fixture(scope="session")
def bump_cloud_arrays(golden):
    """The reference's canonical bump fixture (tests/support.hpp:45-70) as arrays."""
    import pyoracle as P
    g, _ = golden
    c = P.Cloud(g["x"], g["y"], g["kind"], g["nx"], g["ny"], g["off"], g["nbr"])
    return c, g["prim0"]


def rel_err(got, want):
    """Scale-aware error (reference tests/acceptance.cpp:56-62 vec_err): relative
    to the largest |component| per row, absolute once everything is below one."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    scale = np.maximum(np.abs(want).max(axis=-1, keepdims=True), 1.0) if want.ndim else max(abs(want), 1.0)
    return float(np.max(np.abs(got - want) / scale))
