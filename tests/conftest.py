"""Shared fixtures.  `-m gpu` tests need a CUDA device (B200); everything
else runs on CPU.  Only tests/ (plus smoke() and bench.py's baseline leg)
may import the oracle, and only as the checker."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture
def rng():
    return np.random.default_rng(0x5EED)


def smooth_field(rng, shape):
    """Sum of a few low-frequency sinusoids per axis (float64 -> float32)."""
    axes = np.indices(shape).astype(np.float64)
    out = np.zeros(shape)
    for ax, coord in enumerate(axes):
        for _ in range(int(rng.integers(1, 4))):
            freq = rng.uniform(0.5, 3.0) / max(shape[ax], 2)
            out += rng.uniform(0.3, 1.0) * np.sin(2 * np.pi * freq * coord + rng.uniform(0, 6.283))
    return out.astype(np.float32)


def noisy_field(rng, shape):
    return (smooth_field(rng, shape).astype(np.float64) + rng.normal(0, 0.2, shape)).astype(
        np.float32)


def constant_field(rng, shape):
    return np.full(shape, np.float32(rng.uniform(-5, 5)), dtype=np.float32)


def affine_field(rng, shape):
    axes = np.indices(shape).astype(np.float64)
    out = np.full(shape, rng.uniform(-1, 1))
    for c in axes:
        out = out + rng.uniform(-0.5, 0.5) * c
    return out.astype(np.float32)


KINDS = (smooth_field, noisy_field, constant_field, affine_field)
