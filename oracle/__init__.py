"""FP64 CPU oracle — TEST INFRASTRUCTURE, NOT PRODUCT.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg and
``--impl reference``) may import anything under ``oracle/``.  It is independent
of the CUDA path: it shares no code with ``paper_2407_06434_b200`` and neither
imports the other.  See omp_oracle.py for the algorithm and its citations.
"""

from .omp_oracle import (  # noqa: F401
    DEGENERATE,
    EPS,
    MAXITER,
    NAN,
    OracleResult,
    StepRecord,
    atom_norms,
    host_cores,
    least_squares_residual,
    omp,
    omp_batch,
)
