"""L-BFGS + strong-Wolfe driver (lbfgs.hpp) over the library's own host implementation
(csrc/lbfgs_driver.cpp).  Same parameter names, defaults, stop reasons and history records."""
from __future__ import annotations

import ctypes
from ctypes import POINTER, c_double, c_int
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import NumericalError

STOP_REASONS = ("gradient-tolerance", "max-iterations", "line-search-failure")  # lbfgs.cpp:11-19


@dataclass
class LbfgsParams:
    """LbfgsParams (lbfgs.hpp:11-27)."""

    memory: int = 10
    max_iter: int = 100
    grad_tol: float = 1e-6
    c1: float = 1e-4
    c2: float = 0.9
    max_line_search: int = 20

    def validate(self):
        if self.memory < 1:
            raise ValueError("memory must be >= 1")
        if self.max_iter < 1:
            raise ValueError("max_iter must be >= 1")
        if not (0 < self.c1 < self.c2 < 1):
            raise ValueError("need 0 < c1 < c2 < 1")
        if self.max_line_search < 1:
            raise ValueError("max_line_search must be >= 1")

    def to_c(self):
        return _lib.LmsLbfgsParams(self.memory, self.max_iter, self.grad_tol, self.c1, self.c2, self.max_line_search)


@dataclass
class MinimizeResult:
    """MinimizeResult + OptimHistory (lbfgs.hpp:33-46,71-76)."""

    x: np.ndarray
    loss: float
    grad: np.ndarray
    initial_loss: float
    initial_grad_inf_norm: float
    evaluations: int
    reason: str
    iterations: list = field(default_factory=list)  # (loss, grad_inf_norm, step, evals) per accepted iterate


def minimize(objective, x0, params: LbfgsParams | None = None) -> MinimizeResult:
    """minimize (lbfgs.hpp:81-82).  ``objective(x) -> (loss, grad)`` with x, grad flat float64."""
    params = params or LbfgsParams()
    params.validate()
    lib = _lib.load()
    x0 = np.ascontiguousarray(np.asarray(x0, dtype=np.float64)).ravel()
    n = x0.size
    dp = POINTER(c_double)
    raised = []

    def trampoline(_user, xp, gp, nn):
        try:
            x = np.ctypeslib.as_array(xp, shape=(nn,)) if nn else np.empty(0)
            loss, g = objective(x.copy())
            if nn:
                np.ctypeslib.as_array(gp, shape=(nn,))[:] = np.asarray(g, dtype=np.float64).ravel()
            return float(loss)
        except Exception as e:  # an objective error (e.g. DivergedError) aborts the run, as in the reference
            raised.append(e)
            return float("nan")

    cb = _lib.OBJECTIVE_FN(trampoline)
    x_out, g_out = np.empty(max(n, 1)), np.empty(max(n, 1))
    res = _lib.LmsMinimizeResult()
    k = params.max_iter
    hl, hg, hs = np.zeros(k), np.zeros(k), np.zeros(k)
    he = np.zeros(k, dtype=np.int32)
    cparams = params.to_c()
    rc = lib.lms_minimize(cb, None, n, x0.ctypes.data_as(dp), ctypes.byref(cparams), x_out.ctypes.data_as(dp),
                          g_out.ctypes.data_as(dp), ctypes.byref(res), hl.ctypes.data_as(dp), hg.ctypes.data_as(dp),
                          hs.ctypes.data_as(dp), he.ctypes.data_as(POINTER(c_int)))
    if raised:
        raise raised[0]
    if rc == _lib.LMS_ERR_NUMERICAL:
        raise NumericalError("objective non-finite at starting point")
    _lib.check(rc)
    it = res.iterations
    return MinimizeResult(
        x=x_out[:n].copy(), loss=res.loss, grad=g_out[:n].copy(), initial_loss=res.initial_loss,
        initial_grad_inf_norm=res.initial_grad_inf_norm, evaluations=res.evaluations,
        reason=STOP_REASONS[res.reason],
        iterations=[(hl[i], hg[i], hs[i], int(he[i])) for i in range(it)],
    )
