"""Python binding over the C ABI — argument marshalling only.

Every step of the OMP path runs in libomp_b200.so's sm_100a kernels; torch is used
for device memory, streams and dtype/layout plumbing (BASELINE.json north_star:
"PyTorch is used only for device memory, streams and process groups").

Shapes follow the paper's Python interface ("the same functionality as
that from Scikit-Learn, except that the y is batched in the first dimension"):
    A: (M, N) dictionary,  Y: (B, M) signals,  S sparsity,  eps optional tolerance.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

from . import _lib
from ._lib import check

MODES = {"bf16": _lib.OMP_CORR_BF16, "simt": _lib.OMP_CORR_FP32_SIMT, "3xtf32": _lib.OMP_CORR_3XTF32}


def _torch():
    import torch
    return torch


def _stream_ptr(stream, device) -> int:
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


@dataclass
class OMPResult:
    X: "object"          # (B, S) float32, coefficient of support[b, j]
    support: "object"    # (B, S) int32, atom ids in selection order, -1 padded
    resid_norm: "object"  # (B,) float32, ||y_b - A_S x_b||
    n_iter: "object"     # (B,) int32
    status: "object"     # (B,) int32, ompSigStatus_t


class OMP:
    """A dictionary bound to one GPU (ompCreate): setup, Gram matrix and workspaces are cached."""

    def __init__(self, A, mode: str = "bf16", stream=None):
        torch = _torch()
        if not (isinstance(A, torch.Tensor) and A.is_cuda and A.dtype == torch.float32 and A.dim() == 2):
            raise TypeError("A must be a 2-D float32 CUDA tensor of shape (M, N)")
        self.lib = _lib.load()
        self.M, self.N = A.shape
        self.device = A.device
        self.mode = mode
        At = A.t()
        if At.stride(1) != 1 or (self.N > 1 and At.stride(0) < self.M):
            At = At.contiguous()      # column-major (atom-contiguous) layout the ABI takes; lda = At.stride(0)
        h = ctypes.c_void_p()
        st = _stream_ptr(stream, self.device)
        lda = At.stride(0) if self.N > 1 else self.M
        rc = self.lib.ompCreate(ctypes.byref(h), self.device.index, At.data_ptr(), self.M, self.N,
                                lda, MODES[mode], st)
        check(rc, "ompCreate", None)
        self.handle = h

    # -- life cycle ---------------------------------------------------------------------
    def close(self):
        if getattr(self, "handle", None):
            self.lib.ompDestroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- the batch call ---------------------------------------------------------------
    def batch(self, Y, S: int, eps: Optional[float] = None, stream=None, out: Optional[OMPResult] = None) -> OMPResult:
        torch = _torch()
        if not (isinstance(Y, torch.Tensor) and Y.is_cuda and Y.dtype == torch.float32 and Y.dim() == 2):
            raise TypeError("Y must be a 2-D float32 CUDA tensor of shape (B, M)")
        if Y.shape[1] != self.M:
            raise ValueError(f"Y has {Y.shape[1]} measurements, dictionary has M={self.M}")
        B = Y.shape[0]
        # rows must not overlap (an expanded Y has stride(0) = 0): the library reads B x ldy floats
        if Y.stride(1) != 1 or (B > 1 and Y.stride(0) < self.M):
            Y = Y.contiguous()
        ldy = Y.stride(0) if B > 1 else self.M
        dev = self.device
        if out is None:
            out = OMPResult(torch.empty((B, S), dtype=torch.float32, device=dev),
                            torch.empty((B, S), dtype=torch.int32, device=dev),
                            torch.empty((B,), dtype=torch.float32, device=dev),
                            torch.empty((B,), dtype=torch.int32, device=dev),
                            torch.empty((B,), dtype=torch.int32, device=dev))
        e = float("nan") if eps is None else float(eps)
        rc = self.lib.ompBatch(self.handle, Y.data_ptr(), B, ldy, S, e,
                               out.X.data_ptr(), out.X.stride(0), out.support.data_ptr(),
                               out.support.stride(0), out.resid_norm.data_ptr(), out.n_iter.data_ptr(),
                               out.status.data_ptr(), _stream_ptr(stream, dev))
        check(rc, "ompBatch", self.handle)
        return out

    def batch_host(self, Y, S: int, eps: Optional[float] = None, stream=None, out=None):
        """Host (numpy) in, host out: H2D and D2H happen inside the library call (ompBatchHost)."""
        import numpy as np
        Y = np.ascontiguousarray(Y, dtype=np.float32)
        B = Y.shape[0]
        if out is None:
            out = (np.empty((B, S), np.float32), np.empty((B, S), np.int32), np.empty(B, np.float32),
                   np.empty(B, np.int32), np.empty(B, np.int32))
        X, sup, res, nit, st = out
        e = float("nan") if eps is None else float(eps)
        rc = self.lib.ompBatchHost(self.handle, Y.ctypes.data, B, self.M, S, e, X.ctypes.data, S,
                                   sup.ctypes.data, S, res.ctypes.data, nit.ctypes.data, st.ctypes.data,
                                   _stream_ptr(stream, self.device))
        check(rc, "ompBatchHost", self.handle)
        return OMPResult(X, sup, res, nit, st)

    # -- diagnostics / test entry points ---------------------------------------------
    def correlate(self, R, stream=None):
        torch = _torch()
        R = R.contiguous()
        C = torch.empty((R.shape[0], self.N), dtype=torch.float32, device=self.device)
        rc = self.lib.ompCorrelate(self.handle, R.data_ptr(), R.shape[0], R.stride(0), C.data_ptr(),
                                   C.stride(0), _stream_ptr(stream, self.device))
        check(rc, "ompCorrelate", self.handle)
        return C

    def gram(self, stream=None):
        torch = _torch()
        G = torch.empty((self.N, self.N), dtype=torch.float32, device=self.device)
        check(self.lib.ompGetGram(self.handle, G.data_ptr(), self.N, _stream_ptr(stream, self.device)),
              "ompGetGram", self.handle)
        return G

    def factor(self, b0: int, count: int, S: int, stream=None):
        torch = _torch()
        F = torch.empty((count, S * (S + 1) // 2), dtype=torch.float32, device=self.device)
        u = torch.empty((count, S), dtype=torch.float32, device=self.device)
        check(self.lib.ompGetFactor(self.handle, b0, count, F.data_ptr(), u.data_ptr(),
                                    _stream_ptr(stream, self.device)), "ompGetFactor", self.handle)
        return F, u

    def densify(self, res: OMPResult, stream=None):
        torch = _torch()
        B, S = res.X.shape
        Xd = torch.empty((B, self.N), dtype=torch.float32, device=self.device)
        check(self.lib.ompDensify(self.handle, res.X.data_ptr(), res.X.stride(0), res.support.data_ptr(),
                                  res.support.stride(0), res.n_iter.data_ptr(), B, S, Xd.data_ptr(),
                                  Xd.stride(0), _stream_ptr(stream, self.device)), "ompDensify", self.handle)
        return Xd

    def set_graphs(self, enable: bool = True):
        """Capture batches into CUDA graphs and replay them (default) or launch kernel by kernel."""
        check(self.lib.ompSetGraphs(self.handle, int(enable)), "ompSetGraphs", self.handle)

    def profile(self, enable: bool = True):
        check(self.lib.ompProfileEnable(self.handle, int(enable)), "ompProfileEnable", self.handle)

    def profile_read(self, reset: bool = True):
        ms = (ctypes.c_double * _lib.OMP_NUM_KERNEL_SLOTS)()
        n = (ctypes.c_int64 * _lib.OMP_NUM_KERNEL_SLOTS)()
        check(self.lib.ompProfileRead(self.handle, ms, n, int(reset)), "ompProfileRead", self.handle)
        return {name: (ms[i], n[i]) for i, name in enumerate(_lib.KERNEL_SLOTS)}

    ALGOS = {"auto": 0, "residual": 1, "projection": 2}

    def set_algorithm(self, algo: str):
        """'auto' (default), 'residual' or 'projection' (the paper's algorithm v0), see ompSetAlgorithm."""
        check(self.lib.ompSetAlgorithm(self.handle, self.ALGOS[algo]), "ompSetAlgorithm", self.handle)

    def set_small_batch_limit(self, max_batch: int):
        """-1 automatic (default), 0 never, else the largest batch run by the persistent kernel."""
        check(self.lib.ompSetSmallBatchLimit(self.handle, int(max_batch)), "ompSetSmallBatchLimit", self.handle)

    def last_path(self) -> str:
        """'residual', 'small' or 'projection': the path the last batch ran."""
        return _lib.PATH_NAMES[int(self.lib.ompGetLastPath(self.handle))]

    def launch_count(self) -> int:
        return int(self.lib.ompGetLaunchCount(self.handle))


def screening_window(mode: str, M: int) -> float:
    """W / ||r||: the tensor-core screen's candidate window for a dictionary of M rows
    (ompScreeningWindow; host arithmetic only, no GPU needed).  -1 for the SIMT mode."""
    return float(_lib.load().ompScreeningWindow(MODES[mode], int(M)))


def omp_batch(A, Y, S: int, eps: Optional[float] = None, mode: str = "bf16") -> OMPResult:
    """One-shot omp_batch(A, Y, S, eps) -> (X, support, resid_norm, n_iter, status)  (north star)."""
    with OMP(A, mode=mode) as h:
        return h.batch(Y, S, eps)
