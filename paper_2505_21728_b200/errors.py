"""Exception classes mirroring the reference (include/hygt/errors.hpp:23-45) and the mapping
from C-ABI status codes (include/hygt_gpu.h) onto them."""


class ArgumentError(ValueError):
    """Invalid argument or violated invariant (errors.hpp:24-27). CLI exit code 1."""


class IoError(RuntimeError):
    """File read/write failure (errors.hpp:30-33). CLI exit code 2."""


class NumericalError(RuntimeError):
    """Numerical failure (errors.hpp:36-39). CLI exit code 3."""


class OverflowError_(NumericalError):
    """Fixed-point integer range exceeded (errors.hpp:42-45), a NumericalError."""


# The reference spells it OverflowError; keep that public name without shadowing the builtin in
# this module's own code.
OverflowError = OverflowError_  # noqa: A001


class CudaError(RuntimeError):
    """CUDA runtime failure inside the GPU library (status 5, no reference counterpart)."""


_BY_STATUS = {1: ArgumentError, 2: IoError, 3: NumericalError, 4: OverflowError_, 5: CudaError}


def raise_for(status: int, message: str) -> None:
    if status:
        raise _BY_STATUS.get(status, RuntimeError)(message or f"hygt status {status}")
