"""lmshoot_b200: B200-native (sm_100a) objective-and-gradient hot path of landmark geodesic shooting
(arXiv 1907.04839) behind the reference's own interface.  See DESIGN.md and include/lmshoot_b200.h.

Importing this package does not touch the GPU; the C-ABI library is loaded on first use and its
absence is an error (no CPU fallback)."""
from .batch import BatchedRegistrations, BatchRegistrationResult  # noqa: F401
from .errors import (CommError, CudaError, DivergedError, IoError, NumericalError, ParseError, ShapeError,  # noqa: F401
                     StateError)
from .formats import (ResultDocument, load_landmarks, load_result, result_document_from, save_landmarks,  # noqa: F401
                      save_result)
from .lbfgs import LbfgsParams, MinimizeResult, minimize  # noqa: F401
from .registration import RegistrationResult, register_landmarks  # noqa: F401
from .shooting import (GradientResult, HamiltonianSystem, ShootingConfig, comm_unique_id, gaussian_kernel,  # noqa: F401
                       kernel_scale, row_partition, LocalGroup)
from .synth import make_synthetic_pair, make_template_points, rng_normals, rng_uniforms  # noqa: F401

__all__ = [
    "HamiltonianSystem", "BatchedRegistrations", "BatchRegistrationResult", "ShootingConfig", "GradientResult", "LbfgsParams", "MinimizeResult", "minimize",
    "register_landmarks", "RegistrationResult", "make_synthetic_pair", "make_template_points", "rng_normals",
    "rng_uniforms", "gaussian_kernel", "kernel_scale", "comm_unique_id", "row_partition", "LocalGroup", "ShapeError", "DivergedError",
    "NumericalError", "CudaError", "StateError", "CommError", "IoError", "ParseError", "ResultDocument", "load_landmarks",
    "save_landmarks", "load_result", "save_result", "result_document_from",
]
