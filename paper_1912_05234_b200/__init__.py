"""tensorloom-B200: the reference's Zhang-CNN training path (tloom::net / tloom::nn) on sm_100a.

The product is the CUDA library ``lib/libtloom_b200.so`` (C ABI: ``include/tloom_b200.h``; C++ API
mirroring the reference headers: ``include/tloom/*.hpp``).  This Python package is the host-side
mirror used by the tests and the benchmark; names follow the reference
(``net.train``, ``net.forward``, ``nn.mconv`` ...).
"""
from .errors import BoundsError, Error, FormatError, ShapeError, ValueError_  # noqa: F401
from .runtime import Context  # noqa: F401
