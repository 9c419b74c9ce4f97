"""B200-native out-of-core Adam step of Fuyou (arXiv 2403.06504).

The product is the native library ``lib/liboffsim.so.0`` (C++ host code +
sm_100a CUDA kernels) behind the reference's ``offsim`` C/C++ API
(``include/offsim``) and the executor ABI ``include/fuyou/fy_adam.h``.
This Python package only loads it (``_lib``) and offers thin plumbing
helpers (``optim``) for tests and the bench.
"""
from . import _lib  # noqa: F401  (raises ImportError if the library is not built)

__all__ = ["_lib"]
