"""Exception taxonomy of the reference (proj/include/tloom/errors.hpp:9-31), raised from C-ABI codes."""
from __future__ import annotations


class Error(RuntimeError):
    """tloom::Error -- base class for all library errors."""


class ShapeError(Error):
    """tloom::ShapeError -- shape/rank contract violations."""


class BoundsError(ShapeError):
    """tloom::BoundsError -- out-of-range index."""


class FormatError(Error):
    """tloom::FormatError -- malformed input bytes."""


class ValueError_(FormatError):
    """tloom::ValueError -- well-formed container holding an out-of-domain value."""


class CudaError(Error):
    """CUDA runtime failure inside the library (no CPU fallback exists)."""


class ArgumentError(Error):
    """Invalid C-ABI argument (null pointer, bad mode...)."""


_BY_CODE = {1: Error, 2: ShapeError, 3: BoundsError, 4: FormatError, 5: ValueError_, 10: CudaError,
            11: CudaError, 12: ArgumentError}


def raise_for(code: int, message: str) -> None:
    if code != 0:
        raise _BY_CODE.get(code, Error)(message)
