"""Synthetic template/target generation (synth.hpp:15-43; the reference ships declarations only).

Template: Fibonacci sphere of diameter ``extent`` (the formula is this build's choice).
Ground-truth momenta: ``Rng(seed)`` row-major ``momentum_scale * normal()`` (rng.hpp:27-41).
Target: the template flowed under those momenta in 64-bit on the device (synth.hpp:40-43).
"""
from __future__ import annotations

import ctypes
from ctypes import POINTER, c_double

import numpy as np

from . import _lib


def rng_normals(seed, count):
    lib = _lib.load()
    out = np.empty(count)
    lib.lms_rng_normals(seed, count, out.ctypes.data_as(POINTER(c_double)))
    return out


def rng_uniforms(seed, count):
    lib = _lib.load()
    out = np.empty(count)
    lib.lms_rng_uniforms(seed, count, out.ctypes.data_as(POINTER(c_double)))
    return out


def make_template_points(count, extent=40.0):
    lib = _lib.load()
    out = np.empty((count, 3))
    lib.lms_synth_sphere(count, extent, out.ctypes.data_as(POINTER(c_double)))
    return out


def make_synthetic_pair(count, sigma, timesteps, extent=40.0, momentum_scale=0.75, seed=0, device=0,
                        density_scaled=False):
    """Returns (template q0, target, ground-truth momenta).  ``density_scaled`` grows the sphere radius
    with sqrt(count / 1847) so that point density stays that of the reference's default problem."""
    from .shooting import HamiltonianSystem

    if density_scaled:
        extent = extent * float(np.sqrt(count / 1847.0))
    q0 = make_template_points(count, extent)
    momenta = (momentum_scale * rng_normals(seed, count * 3)).reshape(count, 3)
    system = HamiltonianSystem(sigma, count, 3, "f64", device=device, max_timesteps=timesteps)
    try:
        traj_q, _ = system.integrate_forward(q0, momenta, timesteps)
    finally:
        system.close()
    return q0, np.ascontiguousarray(traj_q[-1]), momenta
