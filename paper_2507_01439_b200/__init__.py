"""paper_2507_01439_b200 — B200-native (sm_100a) TurboReg hot path behind a C ABI.

The compute lives in ``lib/libturboreg.so`` (hand-written CUDA kernels, see ``csrc/``); this package is
only the thin Python binding (argument marshalling).  There is no CPU fallback: importing the binding
fails loudly when the shared library is missing.
"""
from ._binding import (  # noqa: F401
    HYPOTHESIS_DTYPE,
    RESULT_DTYPE,
    Params,
    Result,
    Status,
    TurboReg,
    TurboRegError,
    library,
    library_path,
)

__all__ = ["TurboReg", "HYPOTHESIS_DTYPE", "Params", "Result", "Status", "TurboRegError", "RESULT_DTYPE", "library", "library_path"]
