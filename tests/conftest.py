import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box with -m gpu)")


@pytest.fixture(scope="session")
def oracle():
    from oracle import load_oracle

    return load_oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle import load_reference, reference_available

    if not reference_available():
        pytest.skip("oracle/_ref/liblmshoot_ref.so not built (needs /root/reference at build time)")
    return load_reference()


@pytest.fixture(scope="session")
def golden_hotpath():
    return dict(np.load(os.path.join(GOLDEN, "hotpath_golden.npz")))


@pytest.fixture(scope="session")
def golden_optimiser():
    return dict(np.load(os.path.join(GOLDEN, "optimiser_golden.npz")))


@pytest.fixture(scope="session")
def golden_rng():
    return dict(np.load(os.path.join(GOLDEN, "rng_golden.npz")))


def synth_case(n, dim, seed, spread=4.0):
    """Seeded inputs independent of the golden files (numpy Generator streams are stable)."""
    rng = np.random.default_rng(seed)
    q = rng.uniform(-spread, spread, (n, dim))
    p = 0.75 * rng.normal(size=(n, dim))
    target = q + 0.5 * rng.normal(size=(n, dim))
    alpha = rng.normal(size=(n, dim))
    beta = rng.normal(size=(n, dim))
    return q, p, target, alpha, beta


def rel_inf(a, b):
    """||a - b||_inf / ||b||_inf (the metric BASELINE.md §4 states the tolerances in)."""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    scale = np.abs(b).max() if b.size else 0.0
    if scale == 0.0:
        return float(np.abs(a - b).max()) if a.size else 0.0
    return float(np.abs(a - b).max() / scale)
