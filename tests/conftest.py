"""Shared fixtures.  `-m gpu` tests need a B200 and the built librsr_b200.so;
everything else runs on CPU (oracle vs golden vectors, host logic, ABI exports)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and librsr_b200.so")


def load_golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name)) as z:
        return {k: z[k] for k in z.files}


def unpack_index(g: dict, prefix: str):
    """(perms [NB, n] u32, list of seg arrays (2^w + 1 each), buckets [NB, n]) from a golden index."""
    perms = g[prefix + "perms"]
    segs_flat, starts, widths = g[prefix + "segs"], g[prefix + "seg_starts"], g[prefix + "widths"]
    segs = [segs_flat[int(s): int(s) + (1 << int(w)) + 1] for s, w in zip(starts, widths)]
    return perms, segs, g[prefix + "buckets"]


@pytest.fixture(scope="session")
def worked():
    return load_golden("worked_example.npz")


@pytest.fixture(scope="session")
def fuzz():
    return load_golden("fuzz_small.npz")


@pytest.fixture(scope="session")
def medium():
    return load_golden("medium.npz")


@pytest.fixture(scope="session")
def folds():
    return load_golden("folds.npz")


@pytest.fixture(scope="session")
def tuner():
    return load_golden("tuner.npz")


@pytest.fixture(scope="session")
def rsr():
    """The product package (import requires only the library file, not a GPU)."""
    import paper_2411_06360_b200 as pkg
    return pkg


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")
