"""CPU tests of the C-ABI library: it loads, exports every symbol include/lmshoot_b200.h declares,
fails loudly without a device, and its host-only entry points (RNG, synthetic template) agree with the
reference streams."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "lmshoot_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lms_[a-z0-9_]+)\s*\(", text)) - {"lms_objective_fn"})


def test_library_exports_every_declared_symbol():
    from paper_1907_04839_b200 import _lib

    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 30
    for name in names:
        assert hasattr(lib, name), f"{name} declared in include/lmshoot_b200.h but not exported"
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_no_oracle_or_cpu_fallback_in_product():
    """The product package must not import, link or execute anything under oracle/."""
    pkg = os.path.join(ROOT, "paper_1907_04839_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in text.lower(), (dirpath, f)
    import subprocess

    out = subprocess.run(["ldd", os.path.join(pkg, "liblmshoot_b200.so")], capture_output=True, text=True).stdout
    assert "oracle" not in out and "lmshoot_ref" not in out


def test_create_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1907_04839_b200 import CudaError, HamiltonianSystem

    with pytest.raises(CudaError):
        HamiltonianSystem(1.5, 10)


def test_argument_validation_precedes_device_use():
    from paper_1907_04839_b200 import HamiltonianSystem, ShapeError, ShootingConfig

    with pytest.raises(ShapeError):
        HamiltonianSystem(1.5, 10, dim=4)  # shooting.hpp:358
    with pytest.raises(ValueError):
        HamiltonianSystem(-1.0, 10)  # shooting.hpp:113
    with pytest.raises(ValueError):
        ShootingConfig(timesteps=0).validate()
    with pytest.raises(ValueError):
        ShootingConfig(lam=-1).validate()


def test_host_rng_and_template_match_reference_streams(oracle, golden_rng):
    from paper_1907_04839_b200 import make_template_points, rng_normals, rng_uniforms

    for key, want in golden_rng.items():
        kind, seed = key.split("_")
        got = (rng_normals if kind == "normals" else rng_uniforms)(int(seed), want.size)
        assert np.array_equal(got, want)
    assert np.array_equal(rng_normals(5, 1000), oracle.rng_normals(5, 1000))
    pts = make_template_points(1847, 40.0)
    assert np.allclose(np.linalg.norm(pts, axis=1), 20.0, rtol=1e-12)
    assert abs(pts.mean(axis=0)).max() < 0.05


def test_status_strings():
    from paper_1907_04839_b200 import _lib

    lib = _lib.load()
    assert lib.lms_status_string(0) == b"ok"
    assert b"DivergedError" in lib.lms_status_string(2)
    assert lib.lms_variant_name(0, 0).startswith(b"fwd_f32x2") and lib.lms_variant_name(0, 1) == b"fwd_f32_r4_j4"
