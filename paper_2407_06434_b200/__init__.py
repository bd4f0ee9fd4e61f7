"""B200-native batched Orthogonal Matching Pursuit (arXiv 2407.06434), behind a C ABI.

    from paper_2407_06434_b200 import OMP, omp_batch
    res = omp_batch(A, Y, S, eps)          # A (M,N), Y (B,M) float32 CUDA tensors

The hot path (correlation GEMM, normalised argmax, inverse-Cholesky factor append,
residual gather) is libomp_b200.so (sm_100a); see include/omp_b200.h and DESIGN.md.
"""

from ._lib import (  # noqa: F401
    OMP_SIG_DEGENERATE,
    OMP_SIG_EPS,
    OMP_SIG_MAXITER,
    OMP_SIG_NAN,
    OmpError,
)
from .omp import OMP, OMPResult, omp_batch  # noqa: F401

__all__ = ["OMP", "OMPResult", "omp_batch", "OmpError"]
