"""Error taxonomy of the reference (errors.hpp:10-77), raised from C-ABI status codes."""


class IoError(RuntimeError):
    """File/stream level failure: missing file, unwritable destination (errors.hpp:10-13)."""


class ParseError(RuntimeError):
    """Malformed input data; carries a 1-based line number when known (errors.hpp:16-28)."""

    def __init__(self, msg, line=0):
        super().__init__(f"{msg} at line {line}" if line else msg)
        self.line = line


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
