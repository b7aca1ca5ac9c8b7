"""TEST INFRASTRUCTURE ONLY: ctypes bindings for the CPU oracle libraries (see oracle/__init__.py)."""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_size_t, c_ubyte, c_uint, c_ulonglong, c_void_p

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ORACLE_SO = os.path.join(_HERE, "liblmshoot_oracle.so")
_REF_SO = os.path.join(_HERE, "_ref", "liblmshoot_ref.so")

_dp = POINTER(c_double)

STRATEGY = {"sequential": 0, "precompute_matrix": 1, "blocked_tree": 2}
PREC = {"f32": 0, "f64": 1}


class OracleError(RuntimeError):
    def __init__(self, code, step=-1):
        names = {1: "shape", 2: "diverged", 3: "invalid argument", 4: "numerical", 5: "other"}
        super().__init__(f"oracle error {code} ({names.get(code, '?')}), timestep {step}")
        self.code = code
        self.timestep = step


def _arr(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a):
    return a.ctypes.data_as(_dp)


class RefMinimizeOut(ctypes.Structure):
    _fields_ = [
        ("loss", c_double),
        ("evaluations", c_int),
        ("iterations", c_int),
        ("reason", c_int),
        ("initial_loss", c_double),
        ("initial_grad_inf_norm", c_double),
    ]


OBJECTIVE_FN = ctypes.CFUNCTYPE(c_double, c_void_p, _dp, _dp, c_size_t)


class CpuShooting:
    """The same calls on either library: prefix 'orc' (C restatement) or 'ref' (reference build)."""

    def __init__(self, lib, prefix):
        self.lib = lib
        self.prefix = prefix
        red = [c_int, c_size_t, c_uint]
        sig = {
            "last_diverged_step": ([], c_int),
            "gaussian_kernel": ([c_int, c_double, c_double], c_double),
            "kernel_scale": ([c_int, c_double], c_double),
            "tree_sum": ([c_int, _dp, c_size_t], c_double),
            "rng_uniforms": ([c_ulonglong, c_size_t, _dp], None),
            "rng_normals": ([c_ulonglong, c_size_t, _dp], None),
            "rng_stream": ([c_ulonglong, c_size_t, POINTER(c_ubyte), _dp], None),
            "hamiltonian": ([c_int, c_int, c_size_t, c_double, _dp, _dp, c_uint, _dp], c_int),
            "derivatives": ([c_int, c_int, c_size_t, c_double, _dp, _dp, _dp, _dp] + red, c_int),
            "integrate_forward": ([c_int, c_int, c_size_t, c_double, c_int, _dp, _dp, _dp, _dp] + red, c_int),
            "adjoint_step": ([c_int, c_int, c_size_t, c_double, _dp, _dp, _dp, _dp, _dp, _dp] + red, c_int),
            "mismatch_sq": ([c_int, c_int, c_size_t, _dp, _dp, _dp], c_int),
            "landmark_distances": ([c_int, c_size_t, _dp, _dp, _dp], c_int),
            "compute_gradient": (
                [c_int, c_int, c_size_t, c_double, c_double, c_int, _dp, _dp, _dp, _dp, _dp] + red,
                c_int,
            ),
            "velocities": ([c_int, c_int, c_size_t, c_size_t, c_double, _dp, _dp, _dp, _dp] + red, c_int),
            "warp_points": (
                [c_int, c_int, c_size_t, c_size_t, c_double, c_int, _dp, _dp, _dp, _dp] + red,
                c_int,
            ),
        }
        for name, (argtypes, restype) in sig.items():
            if name == "landmark_distances" and prefix == "ref":
                continue  # landmarks.cpp needs Eigen (unbuildable here): restated in the C oracle only
            fn = getattr(lib, f"{prefix}_{name}")
            fn.argtypes = argtypes
            fn.restype = restype
            setattr(self, "_" + name, fn)
        if prefix == "ref":
            lib.ref_minimize.argtypes = [
                OBJECTIVE_FN, c_void_p, c_size_t, _dp, c_int, c_double, c_int, c_double, c_double, c_int,
                _dp, _dp, POINTER(RefMinimizeOut), _dp, _dp, _dp, POINTER(c_int),
            ]
            lib.ref_minimize.restype = c_int
            lib.ref_register.argtypes = [
                c_int, c_int, c_size_t, c_double, c_double, c_int, c_int, c_double, _dp, _dp, _dp, _dp,
                POINTER(RefMinimizeOut), _dp, c_int, c_size_t, c_uint,
            ]
            lib.ref_register.restype = c_int
            lib.ref_hardware_threads.restype = c_uint

    # -- helpers ---------------------------------------------------------------------------------
    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._last_diverged_step())

    @staticmethod
    def _red(strategy, block, threads):
        return STRATEGY[strategy] if isinstance(strategy, str) else int(strategy), int(block), int(threads)

    # -- scalars / rng -----------------------------------------------------------------------------
    def gaussian_kernel(self, prec, r_sq, sigma):
        return self._gaussian_kernel(PREC[prec], float(r_sq), float(sigma))

    def kernel_scale(self, prec, sigma):
        return self._kernel_scale(PREC[prec], float(sigma))

    def tree_sum(self, prec, values):
        v = _arr(values)
        return self._tree_sum(PREC[prec], _p(v), v.size)

    def rng_uniforms(self, seed, count):
        out = np.empty(count)
        self._rng_uniforms(seed, count, _p(out))
        return out

    def rng_normals(self, seed, count):
        out = np.empty(count)
        self._rng_normals(seed, count, _p(out))
        return out

    def rng_stream(self, seed, kinds):
        kinds = np.ascontiguousarray(kinds, dtype=np.uint8)
        out = np.empty(kinds.size)
        self._rng_stream(seed, kinds.size, kinds.ctypes.data_as(POINTER(c_ubyte)), _p(out))
        return out

    # -- hot path ----------------------------------------------------------------------------------
    def hamiltonian(self, prec, q, p, sigma, threads=0):
        q, p = _arr(q), _arr(p)
        n, d = q.shape
        out = c_double()
        self._check(self._hamiltonian(PREC[prec], d, n, sigma, _p(q), _p(p), threads, ctypes.byref(out)))
        return out.value

    def derivatives(self, prec, q, p, sigma, strategy="blocked_tree", block=256, threads=0):
        q, p = _arr(q), _arr(p)
        n, d = q.shape
        hq, hp = np.empty_like(q), np.empty_like(q)
        self._check(self._derivatives(PREC[prec], d, n, sigma, _p(q), _p(p), _p(hq), _p(hp),
                                      *self._red(strategy, block, threads)))
        return hq, hp

    def integrate_forward(self, prec, q0, p0, sigma, timesteps, strategy="blocked_tree", block=256, threads=0):
        q0, p0 = _arr(q0), _arr(p0)
        n, d = q0.shape
        tq = np.empty((timesteps + 1, n, d))
        tp = np.empty((timesteps + 1, n, d))
        self._check(self._integrate_forward(PREC[prec], d, n, sigma, timesteps, _p(q0), _p(p0), _p(tq), _p(tp),
                                            *self._red(strategy, block, threads)))
        return tq, tp

    def adjoint_step(self, prec, q, p, alpha, beta, sigma, strategy="blocked_tree", block=256, threads=0):
        q, p, alpha, beta = _arr(q), _arr(p), _arr(alpha), _arr(beta)
        n, d = q.shape
        da, db = np.empty_like(q), np.empty_like(q)
        self._check(self._adjoint_step(PREC[prec], d, n, sigma, _p(q), _p(p), _p(alpha), _p(beta), _p(da), _p(db),
                                       *self._red(strategy, block, threads)))
        return da, db

    def mismatch_sq(self, prec, a, b):
        a, b = _arr(a), _arr(b)
        n, d = a.shape
        out = c_double()
        self._check(self._mismatch_sq(PREC[prec], d, n, _p(a), _p(b), ctypes.byref(out)))
        return out.value

    def landmark_distances(self, a, b):
        """(average_dist, max_dist) of two paired landmark sets (landmarks.cpp:164-179)."""
        a, b = _arr(a), _arr(b)
        n, d = a.shape
        out = np.zeros(2)
        self._check(self._landmark_distances(d, n, _p(a), _p(b), _p(out)))
        return float(out[0]), float(out[1])

    def compute_gradient(self, prec, q0, p0, target, sigma, lam, timesteps, strategy="blocked_tree", block=256,
                         threads=0):
        """Returns (loss, kinetic, mismatch, grad)."""
        q0, p0, target = _arr(q0), _arr(p0), _arr(target)
        n, d = q0.shape
        sc = np.empty(3)
        g = np.empty_like(q0)
        self._check(self._compute_gradient(PREC[prec], d, n, sigma, lam, timesteps, _p(q0), _p(p0), _p(target),
                                           _p(sc), _p(g), *self._red(strategy, block, threads)))
        return sc[0], sc[1], sc[2], g

    def pair_rows(self, prec, q, p, rows, sigma, alpha=None, beta=None, strategy="blocked_tree", block=256,
                  threads=0):
        """(hq, hp) -- or (d_alpha, d_beta) when alpha/beta are given -- for the listed rows only."""
        assert self.prefix == "orc"
        q, p = _arr(q), _arr(p)
        n, d = q.shape
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        fn = self.lib.orc_pair_rows
        fn.argtypes = [c_int, c_int, c_size_t, c_double, _dp, _dp, _dp, _dp, c_size_t, POINTER(c_size_t), _dp,
                       c_int, c_size_t, c_uint]
        fn.restype = c_int
        sums = np.empty((rows.size, 2 * d))
        a = _arr(alpha) if alpha is not None else None
        b = _arr(beta) if beta is not None else None
        self._check(fn(PREC[prec], d, n, sigma, _p(q), _p(p), _p(a) if a is not None else None,
                       _p(b) if b is not None else None, rows.size, rows.ctypes.data_as(POINTER(c_size_t)), _p(sums),
                       *self._red(strategy, block, threads)))
        return sums[:, :d].copy(), sums[:, d:].copy()

    def velocities(self, prec, q, p, points, sigma, strategy="blocked_tree", block=256, threads=0):
        q, p, points = _arr(q), _arr(p), _arr(points)
        n, d = q.shape
        out = np.empty_like(points)
        self._check(self._velocities(PREC[prec], d, n, points.shape[0], sigma, _p(q), _p(p), _p(points), _p(out),
                                     *self._red(strategy, block, threads)))
        return out

    def warp_points(self, prec, traj_q, traj_p, points, sigma, strategy="blocked_tree", block=256, threads=0):
        traj_q, traj_p, points = _arr(traj_q), _arr(traj_p), _arr(points)
        t1, n, d = traj_q.shape
        out = np.empty_like(points)
        self._check(self._warp_points(PREC[prec], d, n, points.shape[0], sigma, t1 - 1, _p(traj_q), _p(traj_p),
                                      _p(points), _p(out), *self._red(strategy, block, threads)))
        return out

    # -- reference-only: the unmodified optimiser ------------------------------------------------------
    def minimize(self, objective, x0, max_iter=100, grad_tol=1e-6, memory=10, c1=1e-4, c2=0.9, max_line_search=20):
        """Drive the reference's own minimize (lbfgs.cpp:186-282) with a Python objective
        ``objective(x: ndarray) -> (loss, grad ndarray)``."""
        assert self.prefix == "ref"
        x0 = _arr(x0).ravel()
        n = x0.size
        err = []

        def trampoline(_user, xp, gp, nn):
            try:
                x = np.ctypeslib.as_array(xp, shape=(nn,))
                loss, g = objective(x.copy())
                np.ctypeslib.as_array(gp, shape=(nn,))[:] = np.asarray(g, dtype=np.float64).ravel()
                return float(loss)
            except Exception as e:  # surface to the caller after minimize unwinds
                err.append(e)
                return float("nan")

        cb = OBJECTIVE_FN(trampoline)
        x_out, g_out = np.empty(n), np.empty(n)
        out = RefMinimizeOut()
        hl, hg, hs = np.zeros(max_iter), np.zeros(max_iter), np.zeros(max_iter)
        he = np.zeros(max_iter, dtype=np.int32)
        rc = self.lib.ref_minimize(cb, None, n, _p(x0), max_iter, grad_tol, memory, c1, c2, max_line_search,
                                   _p(x_out), _p(g_out), ctypes.byref(out), _p(hl), _p(hg), _p(hs),
                                   he.ctypes.data_as(POINTER(c_int)))
        if err:
            raise err[0]
        self._check(rc)
        k = out.iterations
        return {
            "x": x_out, "grad": g_out, "loss": out.loss, "evaluations": out.evaluations, "iterations": k,
            "reason": out.reason, "initial_loss": out.initial_loss,
            "initial_grad_inf_norm": out.initial_grad_inf_norm,
            "hist_loss": hl[:k], "hist_gnorm": hg[:k], "hist_step": hs[:k], "hist_evals": he[:k],
        }

    def register(self, prec, q0, target, sigma, lam, timesteps, max_iter, grad_tol=1e-6, strategy="blocked_tree",
                 block=256, threads=0):
        assert self.prefix == "ref"
        q0, target = _arr(q0), _arr(target)
        n, d = q0.shape
        mom, warped = np.empty_like(q0), np.empty_like(q0)
        out = RefMinimizeOut()
        hl = np.zeros(max_iter)
        self._check(self.lib.ref_register(PREC[prec], d, n, sigma, lam, timesteps, max_iter, grad_tol, _p(q0),
                                          _p(target), _p(mom), _p(warped), ctypes.byref(out), _p(hl),
                                          *self._red(strategy, block, threads)))
        return {"momenta": mom, "warped": warped, "loss": out.loss, "evaluations": out.evaluations,
                "iterations": out.iterations, "reason": out.reason, "initial_loss": out.initial_loss,
                "hist_loss": hl[: out.iterations]}

    def hardware_threads(self):
        if self.prefix == "ref":
            return int(self.lib.ref_hardware_threads())
        self.lib.orc_hardware_threads_public.restype = c_uint
        return int(self.lib.orc_hardware_threads_public())


def load_oracle():
    if not os.path.exists(_ORACLE_SO):
        raise FileNotFoundError(f"{_ORACLE_SO} missing: run `make -C oracle` (or __graft_entry__.build())")
    return CpuShooting(ctypes.CDLL(_ORACLE_SO), "orc")


def reference_available():
    return os.path.exists(_REF_SO)


def load_reference():
    if not os.path.exists(_REF_SO):
        raise FileNotFoundError(f"{_REF_SO} missing: it is built by `make -C oracle` where /root/reference exists")
    return CpuShooting(ctypes.CDLL(_REF_SO), "ref")
