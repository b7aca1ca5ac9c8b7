"""ctypes loader for liblmshoot_b200.so (the C ABI in include/lmshoot_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).  If it is
missing, importing the compute entry points fails loudly: there is no Python or CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_longlong, c_size_t, c_ubyte, c_uint64, c_void_p

from .errors import CommError, CudaError, DivergedError, NumericalError, ShapeError, StateError

_HERE = os.path.dirname(os.path.abspath(__file__))
# LMS_LIB_PATH: a side-by-side measurement build of the same library (see __graft_entry__.py, LMS_BUILD_TAG)
LIB_PATH = os.environ.get("LMS_LIB_PATH") or os.path.join(_HERE, "liblmshoot_b200.so")

LMS_OK, LMS_ERR_SHAPE, LMS_ERR_DIVERGED, LMS_ERR_INVALID = 0, 1, 2, 3
LMS_ERR_NUMERICAL, LMS_ERR_CUDA, LMS_ERR_STATE, LMS_ERR_COMM = 4, 5, 6, 7

_dp = POINTER(c_double)


class LmsConfig(ctypes.Structure):
    _fields_ = [
        ("precision", c_int),
        ("dim", c_int),
        ("n", c_size_t),
        ("sigma", c_double),
        ("max_timesteps", c_int),
        ("device", c_int),
        ("variant", c_int),
        ("flags", c_int),
    ]


class LmsLbfgsParams(ctypes.Structure):
    _fields_ = [
        ("memory", c_int),
        ("max_iter", c_int),
        ("grad_tol", c_double),
        ("c1", c_double),
        ("c2", c_double),
        ("max_line_search", c_int),
    ]


class LmsMinimizeResult(ctypes.Structure):
    _fields_ = [
        ("loss", c_double),
        ("initial_loss", c_double),
        ("initial_grad_inf_norm", c_double),
        ("evaluations", c_int),
        ("iterations", c_int),
        ("reason", c_int),
    ]


OBJECTIVE_FN = ctypes.CFUNCTYPE(c_double, c_void_p, _dp, _dp, c_size_t)

# name -> (argtypes, restype); every symbol include/lmshoot_b200.h declares.
SIGNATURES = {
    "lms_system_create": ([POINTER(LmsConfig), POINTER(c_void_p)], c_int),
    "lms_system_destroy": ([c_void_p], None),
    "lms_last_diverged_step": ([c_void_p], c_int),
    "lms_last_diverged_point": ([c_void_p], c_longlong),
    "lms_last_error_message": ([c_void_p], c_char_p),
    "lms_status_string": ([c_int], c_char_p),
    "lms_variant_name": ([c_int, c_int], c_char_p),
    "lms_system_kernel_names": ([c_void_p], c_char_p),
    "lms_hamiltonian": ([c_void_p, _dp, _dp, _dp], c_int),
    "lms_derivatives": ([c_void_p, _dp, _dp, _dp, _dp], c_int),
    "lms_integrate_forward": ([c_void_p, _dp, _dp, c_int, _dp, _dp], c_int),
    "lms_adjoint_step": ([c_void_p, _dp, _dp, _dp, _dp, _dp, _dp], c_int),
    "lms_mismatch_sq": ([c_void_p, _dp, _dp, _dp], c_int),
    "lms_compute_gradient": ([c_void_p, _dp, _dp, _dp, c_double, c_int, _dp, _dp], c_int),
    "lms_bind_registration": ([c_void_p, _dp, _dp, c_double, c_int], c_int),
    "lms_objective_eval": ([c_void_p, _dp, _dp, _dp, _dp, _dp], c_int),
    "lms_objective_eval_device": ([c_void_p, c_void_p, c_void_p, _dp], c_int),
    "lms_objective_final_q": ([c_void_p, _dp], c_int),
    "lms_registration_metrics": ([c_void_p, _dp], c_int),
    "lms_last_eval_device_ms": ([c_void_p], c_double),
    "lms_last_eval_kernel_launches": ([c_void_p], c_int),
    "lms_set_kernel_timing": ([c_void_p, c_int], c_int),
    "lms_last_kernel_ms": ([c_void_p, c_int], c_double),
    "lms_velocities": ([c_void_p, _dp, _dp, c_size_t, _dp, _dp], c_int),
    "lms_warp_points_stored": ([c_void_p, c_size_t, _dp, _dp], c_int),
    "lms_lbfgs_default_params": ([POINTER(LmsLbfgsParams)], None),
    "lms_minimize": (
        [OBJECTIVE_FN, c_void_p, c_size_t, _dp, POINTER(LmsLbfgsParams), _dp, _dp, POINTER(LmsMinimizeResult),
         _dp, _dp, _dp, POINTER(c_int)],
        c_int,
    ),
    "lms_register": ([c_void_p, POINTER(LmsLbfgsParams), _dp, _dp, POINTER(LmsMinimizeResult), _dp], c_int),
    "lms_batch_create": ([POINTER(LmsConfig), c_size_t, POINTER(c_void_p)], c_int),
    "lms_batch_size": ([c_void_p], c_size_t),
    "lms_batch_eval": ([c_void_p, c_size_t, POINTER(c_int), _dp, _dp, _dp, POINTER(c_int)], c_int),
    "lms_batch_final_q": ([c_void_p, _dp], c_int),
    "lms_batch_register": ([c_void_p, POINTER(LmsLbfgsParams), _dp, _dp, POINTER(LmsMinimizeResult), POINTER(c_int),
                            POINTER(c_int)], c_int),
    "lms_register_device": ([c_void_p, POINTER(LmsLbfgsParams), _dp, _dp, POINTER(LmsMinimizeResult), _dp], c_int),
    "lms_comm_unique_id": ([POINTER(c_ubyte)], c_int),
    "lms_row_partition": ([c_size_t, c_int, c_int, POINTER(c_longlong), POINTER(c_longlong), POINTER(c_longlong),
                           POINTER(c_longlong)], c_int),
    "lms_system_comm_init": ([c_void_p, POINTER(c_ubyte), c_int, c_int], c_int),
    "lms_local_group_create": ([c_int, POINTER(c_void_p)], c_int),
    "lms_local_group_destroy": ([c_void_p], None),
    "lms_system_join_local_group": ([c_void_p, c_void_p, c_int], c_int),
    "lms_p2p_export": ([c_void_p, c_int, c_int, POINTER(c_ubyte)], c_int),
    "lms_p2p_connect": ([c_void_p, POINTER(c_ubyte)], c_int),
    "lms_rng_normals": ([c_uint64, c_size_t, _dp], None),
    "lms_rng_uniforms": ([c_uint64, c_size_t, _dp], None),
    "lms_synth_sphere": ([c_size_t, c_double, _dp], None),
}

_lib = None


def load():
    """Load the C-ABI library and type every declared entry point.  Raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`. "
            "lmshoot_b200 has no CPU fallback."
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (argtypes, restype) in SIGNATURES.items():
        fn = getattr(lib, name)  # AttributeError here means header and library disagree
        fn.argtypes = argtypes
        fn.restype = restype
    _lib = lib
    return lib


def check(status, handle=None):
    """Map a C-ABI status to the reference's exception types (errors.hpp)."""
    if status == LMS_OK:
        return
    lib = load()
    detail = ""
    if handle is not None:
        msg = lib.lms_last_error_message(handle)
        detail = msg.decode() if msg else ""
    text = lib.lms_status_string(status).decode() + (f": {detail}" if detail else "")
    if status == LMS_ERR_SHAPE:
        raise ShapeError(text)
    if status == LMS_ERR_DIVERGED:
        step = lib.lms_last_diverged_step(handle) if handle is not None else -1
        point = lib.lms_last_diverged_point(handle) if handle is not None else -1
        raise DivergedError(step, point)
    if status == LMS_ERR_INVALID:
        raise ValueError(text)  # std::invalid_argument
    if status == LMS_ERR_NUMERICAL:
        raise NumericalError(text)
    if status == LMS_ERR_STATE:
        raise StateError(text)
    if status == LMS_ERR_COMM:
        raise CommError(text)
    raise CudaError(text)
