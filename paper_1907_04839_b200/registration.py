"""The registration core (registration.cpp:22-100) on the device objective.

Only what surrounds the hot path: p0 initialisation x0 = (target - q0)/T (:47-52), the objective
closure (:58-74), minimize (:79), and the warped landmarks / distance metrics (:85-96).  Procrustes
alignment, landmark file I/O and the JSON result document are out of scope."""
from __future__ import annotations

import ctypes
from ctypes import POINTER, c_double
from dataclasses import dataclass

import numpy as np

from . import _lib
from .lbfgs import STOP_REASONS, LbfgsParams
from .shooting import HamiltonianSystem, ShootingConfig


@dataclass
class RegistrationResult:
    momenta: np.ndarray
    warped: np.ndarray
    final_loss: float
    initial_loss: float
    evaluations: int
    iterations: int
    reason: str
    hist_loss: np.ndarray
    avg_before: float
    max_before: float
    avg_after: float
    max_after: float


def average_dist(a, b):
    """landmarks.cpp:164-171 on the host (numpy), for callers without a device handle; register_landmarks itself
    takes the metrics from the device (lms_registration_metrics)."""
    return float(np.mean(np.linalg.norm(np.asarray(a) - np.asarray(b), axis=1))) if len(a) else 0.0


def max_dist(a, b):
    """landmarks.cpp:173-179."""
    return float(np.max(np.linalg.norm(np.asarray(a) - np.asarray(b), axis=1))) if len(a) else 0.0


def register_landmarks(template, target, config: ShootingConfig | None = None, grad_tol=1e-6, device=0,
                       system: HamiltonianSystem | None = None, device_vectors=False,
                       already_bound=False) -> RegistrationResult:
    """register_landmarks (registration.hpp:48-50) without Procrustes: runs wholly through the C ABI
    (lms_register): device objective + the library's host L-BFGS driver; ``device_vectors=True`` keeps the
    optimiser's vectors in HBM as well (lms_register_device)."""
    config = config or ShootingConfig()
    config.validate()
    template = np.ascontiguousarray(np.asarray(template, dtype=np.float64))
    target = np.ascontiguousarray(np.asarray(target, dtype=np.float64))
    if template.shape != target.shape or template.ndim != 2:
        from .errors import ShapeError

        raise ShapeError("template and target must have equal count and dimension")  # registration.cpp:148-150
    n, dim = template.shape
    own = system is None
    if own:
        system = HamiltonianSystem(config.sigma, n, dim, config.precision, device=device,
                                   max_timesteps=config.timesteps)
    try:
        if not already_bound:  # binding uploads q0/target and captures the evaluation graph (a few ms)
            system.bind_registration(template, target, config.lam, config.timesteps)
        lib = system.lib
        params = LbfgsParams(max_iter=config.max_iter, grad_tol=grad_tol).to_c()
        dp = POINTER(c_double)
        momenta, warped = np.empty((n, dim)), np.empty((n, dim))
        hist = np.zeros(config.max_iter)
        res = _lib.LmsMinimizeResult()
        entry = lib.lms_register_device if device_vectors else lib.lms_register
        _lib.check(entry(system.handle, ctypes.byref(params), momenta.ctypes.data_as(dp),
                                    warped.ctypes.data_as(dp), ctypes.byref(res), hist.ctypes.data_as(dp)),
                   system.handle)
        # avg / max landmark distance before and after (registration.cpp:39-40,95-96), computed on the device from
        # the bound sets and the resident q(1)
        metrics = np.zeros(4)
        _lib.check(lib.lms_registration_metrics(system.handle, metrics.ctypes.data_as(dp)), system.handle)
    finally:
        if own:
            system.close()
    return RegistrationResult(
        momenta=momenta, warped=warped, final_loss=res.loss, initial_loss=res.initial_loss,
        evaluations=res.evaluations, iterations=res.iterations, reason=STOP_REASONS[res.reason],
        hist_loss=hist[: res.iterations].copy(),
        avg_before=float(metrics[0]), max_before=float(metrics[1]),
        avg_after=float(metrics[2]), max_after=float(metrics[3]),
    )
