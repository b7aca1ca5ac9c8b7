"""Host-side mirror of the reference's shooting interface (shooting.hpp) over the CUDA C ABI.

Same names, argument meaning and error behaviour as ``lmshoot::HamiltonianSystem<T, D>`` so that the
parity tests read like tests of the reference.  All arrays are (n, dim) float64 on entry and exit;
the working precision T lives on the device.
"""
from __future__ import annotations

import ctypes
from ctypes import c_double, c_void_p
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ShapeError

PRECISION = {"f32": 0, "f64": 1}


@dataclass
class ShootingConfig:
    """ShootingConfig (shooting.hpp:25-50); the CPU-only fields (backend, block_size, threads,
    memory_budget) have no GPU counterpart and are omitted."""

    sigma: float = 1.5
    timesteps: int = 40
    lam: float = 500000.0
    max_iter: int = 400
    precision: str = "f64"

    def validate(self):
        if not self.sigma > 0:
            raise ValueError("sigma must be positive")
        if self.timesteps < 1:
            raise ValueError("timesteps must be >= 1")
        if self.lam < 0:
            raise ValueError("lambda must be >= 0")
        if self.max_iter < 1:
            raise ValueError("max_iter must be >= 1")
        if self.precision not in PRECISION:
            raise ValueError("bad precision")


@dataclass
class GradientResult:
    """GradientResult (shooting.hpp:91-97)."""

    loss: float
    kinetic: float
    mismatch: float
    grad: np.ndarray


def _points(a, name="points"):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if a.ndim != 2:
        raise ShapeError(f"{name}: expected an (n, dim) array")
    return a


def _ptr(a):
    return a.ctypes.data_as(ctypes.POINTER(c_double))


class HamiltonianSystem:
    """``HamiltonianSystem<T, D>`` (shooting.hpp:104-344) bound to n landmarks on one B200.

    The device handle owns the trajectory (``max_timesteps`` + 1 snapshots), the adjoint state and all
    scratch; nothing O(N^2) is ever allocated (K is never materialised).
    """

    def __init__(self, sigma, n, dim=3, precision="f64", device=0, max_timesteps=40, variant=0, tiled_only=False):
        if dim not in (2, 3):
            raise ShapeError("dimension must be 2 or 3")  # shooting.hpp:358
        if not sigma > 0:
            raise ValueError("sigma must be positive")  # shooting.hpp:113
        if precision not in PRECISION:
            raise ValueError("bad precision")
        self.lib = _lib.load()
        self.sigma, self.n, self.dim, self.precision = float(sigma), int(n), int(dim), precision
        self.device, self.max_timesteps, self.variant = int(device), int(max_timesteps), int(variant)
        # tiled_only: LMS_FLAG_TILED_ONLY, pins the multi-launch tiled path (small problems otherwise run the whole
        # evaluation as one persistent kernel)
        cfg = _lib.LmsConfig(PRECISION[precision], dim, n, sigma, max_timesteps, device, variant, 1 if tiled_only else 0)
        handle = c_void_p()
        _lib.check(self.lib.lms_system_create(ctypes.byref(cfg), ctypes.byref(handle)))
        self.handle = handle
        self._bound = None

    def close(self):
        if getattr(self, "handle", None):
            self.lib.lms_system_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- helpers --------------------------------------------------------------------------------------
    def _same(self, op, *arrays):
        out = []
        for a in arrays:
            a = _points(a)
            if a.shape[1] != self.dim:
                raise ShapeError(f"{op}: dimension {a.shape[1]} != {self.dim}")
            out.append(a)
        n0 = out[0].shape[0]
        for a in out[1:]:
            if a.shape[0] != n0:  # require_same, shooting.hpp:332-338
                raise ShapeError(f"{op}: mismatched landmark counts ({n0} vs {a.shape[0]})")
        if n0 != self.n:
            raise ShapeError(f"{op}: system was created for {self.n} landmarks, got {n0}")
        return out

    def _check(self, status):
        _lib.check(status, self.handle)

    # -- HamiltonianSystem members --------------------------------------------------------------------------
    def hamiltonian(self, q, p):
        """shooting.hpp:123-142."""
        q, p = self._same("hamiltonian", q, p)
        out = c_double()
        self._check(self.lib.lms_hamiltonian(self.handle, _ptr(q), _ptr(p), ctypes.byref(out)))
        return out.value

    def derivatives(self, q, p):
        """shooting.hpp:147-176 -> (hq, hp)."""
        q, p = self._same("derivatives", q, p)
        hq, hp = np.empty_like(q), np.empty_like(q)
        self._check(self.lib.lms_derivatives(self.handle, _ptr(q), _ptr(p), _ptr(hq), _ptr(hp)))
        return hq, hp

    def integrate_forward(self, q0, p0, timesteps):
        """shooting.hpp:180-214 -> (traj_q, traj_p), each (timesteps + 1, n, dim)."""
        q0, p0 = self._same("integrate_forward", q0, p0)
        if timesteps < 1:
            raise ValueError("timesteps must be >= 1")
        tq = np.empty((timesteps + 1, self.n, self.dim))
        tp = np.empty((timesteps + 1, self.n, self.dim))
        self._check(self.lib.lms_integrate_forward(self.handle, _ptr(q0), _ptr(p0), timesteps, _ptr(tq), _ptr(tp)))
        return tq, tp

    def adjoint_step(self, q, p, alpha, beta):
        """shooting.hpp:233-271 -> (d_alpha, d_beta)."""
        q, p, alpha, beta = self._same("adjoint_step", q, p, alpha, beta)
        da, db = np.empty_like(q), np.empty_like(q)
        self._check(self.lib.lms_adjoint_step(self.handle, _ptr(q), _ptr(p), _ptr(alpha), _ptr(beta), _ptr(da),
                                              _ptr(db)))
        return da, db

    def mismatch_sq(self, a, b):
        """shooting.hpp:318-329."""
        a, b = self._same("mismatch_sq", a, b)
        out = c_double()
        self._check(self.lib.lms_mismatch_sq(self.handle, _ptr(a), _ptr(b), ctypes.byref(out)))
        return out.value

    def compute_gradient(self, q0, p0, target, lam, timesteps):
        """shooting.hpp:277-315 -> GradientResult."""
        q0, p0, target = self._same("compute_gradient", q0, p0, target)
        sc = np.empty(3)
        grad = np.empty_like(q0)
        self._check(self.lib.lms_compute_gradient(self.handle, _ptr(q0), _ptr(p0), _ptr(target), lam, timesteps,
                                                  _ptr(sc), _ptr(grad)))
        self._bound = (lam, timesteps)
        return GradientResult(sc[0], sc[1], sc[2], grad)

    # -- the objective closure (registration.cpp:58-74) ----------------------------------------------------------
    def bind_registration(self, q0, target, lam, timesteps):
        q0, target = self._same("register", q0, target)
        self._check(self.lib.lms_bind_registration(self.handle, _ptr(q0), _ptr(target), lam, timesteps))
        self._bound = (lam, timesteps)

    def objective(self, x, grad=None):
        """One call of the reference's ``Objective`` (lbfgs.hpp:48-50): flat p0 -> (loss, grad).
        ``self.last_kinetic`` / ``self.last_mismatch`` carry the verbose line's extras."""
        x = np.ascontiguousarray(np.asarray(x, dtype=np.float64)).ravel()
        if x.size != self.n * self.dim:
            raise ShapeError(f"objective: expected {self.n * self.dim} values, got {x.size}")
        if grad is None:
            grad = np.empty(self.n * self.dim)
        loss, kin, mm = c_double(), c_double(), c_double()
        self._check(self.lib.lms_objective_eval(self.handle, _ptr(x), _ptr(grad), ctypes.byref(loss),
                                                ctypes.byref(kin), ctypes.byref(mm)))
        self.last_kinetic, self.last_mismatch = kin.value, mm.value
        return loss.value, grad

    def objective_ptrs(self, x_ptr, grad_ptr, device=False):
        """Pointer-level evaluation for benchmarks: host (pinned) or device float64 buffers."""
        sc = (c_double * 3)()
        if device:
            self._check(self.lib.lms_objective_eval_device(self.handle, c_void_p(x_ptr), c_void_p(grad_ptr), sc))
        else:
            self._check(self.lib.lms_objective_eval(
                self.handle, ctypes.cast(c_void_p(x_ptr), ctypes.POINTER(c_double)),
                ctypes.cast(c_void_p(grad_ptr), ctypes.POINTER(c_double)),
                ctypes.cast(sc, ctypes.POINTER(c_double)),
                ctypes.cast(ctypes.addressof(sc) + 8, ctypes.POINTER(c_double)),
                ctypes.cast(ctypes.addressof(sc) + 16, ctypes.POINTER(c_double))))
        return sc[0], sc[1], sc[2]

    def final_q(self):
        out = np.empty((self.n, self.dim))
        self._check(self.lib.lms_objective_final_q(self.handle, _ptr(out)))
        return out

    # -- measurement hooks -------------------------------------------------------------------------------------------
    def last_eval_device_ms(self):
        return self.lib.lms_last_eval_device_ms(self.handle)

    def last_eval_kernel_launches(self):
        return self.lib.lms_last_eval_kernel_launches(self.handle)

    def set_kernel_timing(self, enabled):
        self._check(self.lib.lms_set_kernel_timing(self.handle, int(bool(enabled))))

    def last_kernel_ms(self, which):
        return self.lib.lms_last_kernel_ms(self.handle, {"forward": 0, "adjoint": 1}.get(which, which))

    # -- flow (flow.hpp) ----------------------------------------------------------------------------------------------
    def velocities_at_step(self, q, p, points):
        """detail::velocities_at_step (flow.hpp:26-48) against one snapshot (q, p)."""
        q, p = self._same("velocities", q, p)
        points = _points(points)
        if points.shape[1] != self.dim:
            raise ShapeError("velocities: point dimension mismatch")
        out = np.empty_like(points)
        self._check(self.lib.lms_velocities(self.handle, _ptr(q), _ptr(p), points.shape[0], _ptr(points), _ptr(out)))
        return out

    def warp_points(self, points):
        """warp_points (flow.hpp:66-81) through the trajectory stored by the last integrate/evaluate."""
        points = _points(points)
        if points.shape[1] != self.dim:
            raise ShapeError("warp_points: point dimension mismatch")
        out = np.empty_like(points)
        self._check(self.lib.lms_warp_points_stored(self.handle, points.shape[0], _ptr(points), _ptr(out)))
        return out

    # -- multi-GPU row partition ------------------------------------------------------------------------------------------
    def join_local_group(self, group, rank: int):
        """Row partition over the in-process loopback transport (see LocalGroup)."""
        self._check(self.lib.lms_system_join_local_group(self.handle, group.handle, rank))

    def comm_init(self, unique_id: bytes, rank: int, world: int):
        buf = (ctypes.c_ubyte * 128).from_buffer_copy(unique_id)
        self._check(self.lib.lms_system_comm_init(self.handle, buf, rank, world))

    def p2p_export(self, rank: int, world: int) -> bytes:
        """Row partition over the peer-push transport, step 1: lay this handle out as `rank` of `world` and
        describe its exchange arena (128 bytes to all-gather among the ranks)."""
        buf = (ctypes.c_ubyte * 128)()
        self._check(self.lib.lms_p2p_export(self.handle, rank, world, buf))
        return bytes(buf)

    def p2p_connect(self, blobs):
        """Step 2: map every peer's arena (`blobs`: the `world` exported blobs in rank order)."""
        joined = b"".join(blobs)
        buf = (ctypes.c_ubyte * len(joined)).from_buffer_copy(joined)
        self._check(self.lib.lms_p2p_connect(self.handle, buf))


def gaussian_kernel(r_sq, sigma):
    """gaussian_kernel (shooting.hpp:55-59) in float64; the device evaluates exp(r2 * kernel_scale)."""
    return float(np.exp(-r_sq / (2.0 * sigma * sigma)))


def kernel_scale(sigma, precision="f64"):
    """kernel_scale<T> (shooting.hpp:63-68): rounded in T exactly as the reference rounds it."""
    t = np.float32 if precision == "f32" else np.float64
    inv_sig2 = t(1) / (t(sigma) * t(sigma))
    return float(t(-0.5) * inv_sig2)


def comm_unique_id() -> bytes:
    lib = _lib.load()
    buf = (ctypes.c_ubyte * 128)()
    _lib.check(lib.lms_comm_unique_id(buf))
    return bytes(buf)


def row_partition(n, world, rank):
    """The row partition of the multi-GPU path (lms_row_partition): returns (slice, stride, row_begin, row_end).
    Host arithmetic only; usable without a device."""
    from ctypes import c_longlong

    lib = _lib.load()
    vals = [c_longlong() for _ in range(4)]
    _lib.check(lib.lms_row_partition(n, world, rank, *[ctypes.byref(v) for v in vals]))
    return tuple(v.value for v in vals)


class LocalGroup:
    """`world` ranks as handles in one process (lms_local_group_*): the row partition's loopback transport."""

    def __init__(self, world):
        self.lib = _lib.load()
        self.world = int(world)
        handle = c_void_p()
        _lib.check(self.lib.lms_local_group_create(self.world, ctypes.byref(handle)))
        self.handle = handle

    def close(self):
        if getattr(self, "handle", None):
            self.lib.lms_local_group_destroy(self.handle)
            self.handle = None
