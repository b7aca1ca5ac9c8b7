"""Population studies: a batch of independent registrations evaluated together (BASELINE configs[3]).

Each problem is a separate instance of the reference's registration (registration.cpp:22-100) with its own
L-BFGS run; the library coalesces the concurrent objective calls of all problems into one batched device
evaluation per round, so problems of N ~ 2000 landmarks fill a B200 that one of them alone cannot."""
from __future__ import annotations

import ctypes
from ctypes import POINTER, c_double, c_int, c_void_p
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ShapeError
from .lbfgs import STOP_REASONS, LbfgsParams
from .shooting import PRECISION

_dp = POINTER(c_double)


def _ptr(a):
    return a.ctypes.data_as(_dp)


@dataclass
class BatchRegistrationResult:
    momenta: np.ndarray      # batch x n x dim
    warped: np.ndarray       # batch x n x dim
    final_loss: np.ndarray   # batch
    initial_loss: np.ndarray
    evaluations: np.ndarray
    iterations: np.ndarray
    reasons: list
    status: np.ndarray       # per problem C-ABI status (0 ok, 2 diverged, 4 numerical)
    rounds: int              # batched device evaluations performed


class BatchedRegistrations:
    """`batch` registrations of n landmarks each on one GPU (lms_batch_* in include/lmshoot_b200.h)."""

    def __init__(self, sigma, n, batch, dim=3, precision="f32", device=0, max_timesteps=10, variant=0):
        if dim not in (2, 3):
            raise ShapeError("dimension must be 2 or 3")
        self.lib = _lib.load()
        self.n, self.batch, self.dim, self.precision = int(n), int(batch), int(dim), precision
        cfg = _lib.LmsConfig(PRECISION[precision], dim, n, sigma, max_timesteps, device, variant, 0)
        handle = c_void_p()
        _lib.check(self.lib.lms_batch_create(ctypes.byref(cfg), batch, ctypes.byref(handle)))
        self.handle = handle

    def close(self):
        if getattr(self, "handle", None):
            self.lib.lms_system_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _batch_array(self, a, name):
        a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
        if a.shape != (self.batch, self.n, self.dim):
            raise ShapeError(f"{name}: expected shape {(self.batch, self.n, self.dim)}, got {a.shape}")
        return a

    def bind(self, templates, targets, lam, timesteps):
        q0, tg = self._batch_array(templates, "templates"), self._batch_array(targets, "targets")
        _lib.check(self.lib.lms_bind_registration(self.handle, _ptr(q0), _ptr(tg), lam, timesteps), self.handle)

    def evaluate(self, x, ids=None):
        """One objective evaluation for the problems in ids (default all): returns (scalars batch x 3, grad,
        diverged_step batch); entries of problems not listed are left zero / -1."""
        x = self._batch_array(x, "x")
        grad = np.zeros_like(x)
        scalars = np.zeros((self.batch, 3))
        div = np.full(self.batch, -1, dtype=np.int32)
        if ids is None:
            idp, count = None, self.batch
        else:
            ids = np.ascontiguousarray(ids, dtype=np.int32)
            idp, count = ids.ctypes.data_as(POINTER(c_int)), ids.size
        _lib.check(self.lib.lms_batch_eval(self.handle, count, idp, _ptr(x), _ptr(grad), _ptr(scalars),
                                           div.ctypes.data_as(POINTER(c_int))), self.handle)
        return scalars, grad, div

    def evaluate_ptrs(self, x_ptr: int, grad_ptr: int, scalars_ptr: int, diverged_ptr: int = 0):
        """The same evaluation of all problems on caller-owned host buffers given as addresses (x, grad: batch x n x
        dim float64; scalars: batch x 3 float64; diverged: batch int32 or 0) -- e.g. pinned memory, no allocation."""
        from ctypes import c_void_p, cast

        dp = POINTER(ctypes.c_double)
        _lib.check(self.lib.lms_batch_eval(self.handle, self.batch, None, cast(c_void_p(x_ptr), dp),
                                           cast(c_void_p(grad_ptr), dp), cast(c_void_p(scalars_ptr), dp),
                                           cast(c_void_p(diverged_ptr), POINTER(c_int)) if diverged_ptr else None),
                   self.handle)

    def final_q(self):
        out = np.empty((self.batch, self.n, self.dim))
        _lib.check(self.lib.lms_batch_final_q(self.handle, _ptr(out)), self.handle)
        return out

    def last_eval_device_ms(self):
        return self.lib.lms_last_eval_device_ms(self.handle)

    def register(self, params: LbfgsParams | None = None) -> BatchRegistrationResult:
        params = params or LbfgsParams()
        params.validate()
        cparams = params.to_c()
        momenta = np.zeros((self.batch, self.n, self.dim))
        warped = np.zeros((self.batch, self.n, self.dim))
        results = (_lib.LmsMinimizeResult * self.batch)()
        status = np.zeros(self.batch, dtype=np.int32)
        rounds = c_int()
        _lib.check(self.lib.lms_batch_register(self.handle, ctypes.byref(cparams), _ptr(momenta), _ptr(warped), results,
                                               status.ctypes.data_as(POINTER(c_int)), ctypes.byref(rounds)),
                   self.handle)
        return BatchRegistrationResult(
            momenta=momenta, warped=warped,
            final_loss=np.array([r.loss for r in results]), initial_loss=np.array([r.initial_loss for r in results]),
            evaluations=np.array([r.evaluations for r in results]), iterations=np.array([r.iterations for r in results]),
            reasons=[STOP_REASONS[r.reason] for r in results], status=status, rounds=rounds.value)
