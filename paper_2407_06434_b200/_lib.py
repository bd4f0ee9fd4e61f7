"""ctypes binding of libomp_b200.so (include/omp_b200.h).  Argument marshalling only.

The functions below carry the C ABI's names and argument order; pointers are plain
integers (device addresses) and `stream` is a cudaStream_t as an integer.  If the
shared library is missing or cannot be loaded this module raises: there is no
fallback implementation anywhere in the product.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_float, c_int, c_int32, c_int64, c_void_p, c_char_p

HERE = os.path.dirname(os.path.abspath(__file__))
# OMP_B200_LIB: load another build of the same library (A/B measurements of kernel variants)
LIB_PATH = os.environ.get("OMP_B200_LIB") or os.path.join(HERE, "libomp_b200.so")

OMP_OK = 0
OMP_ERR_INVALID_ARG = 1
OMP_ERR_ZERO_COLUMN = 2
OMP_ERR_NONFINITE = 3
OMP_ERR_NOMEM = 4
OMP_ERR_CUDA = 5
OMP_ERR_UNSUPPORTED = 6

OMP_SIG_MAXITER = 0
OMP_SIG_EPS = 1
OMP_SIG_DEGENERATE = 2
OMP_SIG_NAN = 3

OMP_CORR_BF16 = 0
OMP_CORR_FP32_SIMT = 1
OMP_CORR_3XTF32 = 2
OMP_ALGO_AUTO = 0
OMP_ALGO_RESIDUAL = 1
OMP_ALGO_PROJECTION = 2
PATH_NAMES = ("residual", "small", "projection")
OMP_NUM_KERNEL_SLOTS = 5
KERNEL_SLOTS = ("init", "correlation", "select", "update", "small")

# name -> (restype, argtypes); the list is also the ABI inventory tests check against the header
SIGNATURES = {
    "ompCreate": (c_int, [POINTER(c_void_p), c_int, c_void_p, c_int64, c_int64, c_int64, c_int, c_void_p]),
    "ompBatch": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int32, c_float, c_void_p, c_int64,
                         c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ompBatchHost": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int32, c_float, c_void_p, c_int64,
                             c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ompDensify": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int32,
                           c_void_p, c_int64, c_void_p]),
    "ompCorrelate": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p]),
    "ompScreeningWindow": (c_float, [c_int, c_int64]),
    "ompGetGram": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "ompGetFactor": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p]),
    "ompSetGraphs": (c_int, [c_void_p, c_int]),
    "ompProfileEnable": (c_int, [c_void_p, c_int]),
    "ompProfileRead": (c_int, [c_void_p, POINTER(c_double), POINTER(c_int64), c_int]),
    "ompGetLaunchCount": (c_int64, [c_void_p]),
    "ompSetSmallBatchLimit": (c_int, [c_void_p, c_int64]),
    "ompSetAlgorithm": (c_int, [c_void_p, c_int]),
    "ompGetLastPath": (c_int, [c_void_p]),
    "ompDestroy": (c_int, [c_void_p]),
    "ompGetErrorString": (c_char_p, [c_int]),
    "ompGetErrorDetail": (c_int64, [c_void_p]),
    "omp_batch": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_int32, c_float, c_void_p,
                          c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
}

_LIB = None


def load(path: str = LIB_PATH):
    """Load the shared library (raises OSError/FileNotFoundError loudly if absent)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise FileNotFoundError(
            f"{path} is missing: build it with `python -m paper_2407_06434_b200.build` "
            "(there is no CPU or eager fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        if os.environ.get("OMP_B200_LIB") and not hasattr(lib, name):
            continue                    # an older build under A/B test: only its own entry points
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


class OmpError(RuntimeError):
    def __init__(self, status: int, where: str, detail: int):
        msg = load().ompGetErrorString(status).decode()
        super().__init__(f"{where}: {msg} (detail {detail})")
        self.status = status
        self.detail = detail


def check(status: int, where: str, handle=None):
    if status != OMP_OK:
        raise OmpError(status, where, int(load().ompGetErrorDetail(handle)))
