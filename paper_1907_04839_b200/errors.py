"""Error taxonomy of the reference (errors.hpp:10-77), raised from C-ABI status codes."""


class ShapeError(RuntimeError):
    """Mismatched landmark counts/dimensions (errors.hpp:31-34)."""


class NumericalError(RuntimeError):
    """Non-finite state during integration or optimisation (errors.hpp:55-58)."""


class DivergedError(NumericalError):
    """Integration produced NaN/Inf; records where (errors.hpp:61-75)."""

    def __init__(self, timestep, point=-1):
        msg = f"non-finite state at timestep {timestep}"
        if point >= 0:
            msg += f" (point {point})"
        super().__init__(msg)
        self.timestep = timestep
        self.point = point


class CudaError(RuntimeError):
    """CUDA runtime failure or no usable sm_100 device.  There is no CPU fallback."""


class StateError(RuntimeError):
    """Call-order violation (e.g. evaluating before binding a registration)."""


class CommError(RuntimeError):
    """NCCL failure in the row-partitioned path."""
