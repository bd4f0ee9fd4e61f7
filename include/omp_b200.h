/*
 * omp_b200.h — C ABI of the B200-native batched Orthogonal Matching Pursuit library.
 *
 * The operation (Algorithm 1 "Orthogonal Matching Pursuit"):
 *   input  A in R^{M x N} dictionary, y in R^M measurement, S sparsity level,
 *          eps target error (optional)
 *   output x_hat, the S-sparse reconstruction
 *   for k = 1..S:  n* = argmax_n |<r_{k-1}, a_n>| / ||a_n||
 *                  S_k = S_{k-1} u {n*}
 *                  x_k = (A_Sk^T A_Sk)^{-1} A_Sk^T y
 *                  r_k = y - A_Sk x_k
 *   or stop when ||y - A_Sk x_k|| <= eps
 * batched over B signals that share one dictionary ("y is batched", PAPER.md:290;
 * "the whole reason for batching").  The least-squares step uses the
 * inverse-Cholesky update of Section 2.2 with Gram entries
 * [A^T A]_{n*}.
 *
 * Conventions (all functions):
 *  - Array arguments are DEVICE pointers on the handle's device unless the name ends
 *    in _host.  Layouts are column-major (BLAS / scikit-learn):
 *      A  M x N, lda >= M : atom n occupies A[n*lda .. n*lda+M-1]
 *      Y  M x B, ldy >= M : signal b occupies Y[b*ldy .. b*ldy+M-1]
 *      X, support : B rows of S entries, row stride ldx / lds >= S
 *    Indices are zero-based.
 *  - Ownership: the caller owns every buffer passed in.  The handle owns its copies of
 *    the dictionary (FP32 + TF32 hi/lo planes), 1/||a_n||, the Gram matrix, and a
 *    workspace grown lazily for the largest B seen.  A handle is bound to one device
 *    and is not thread-safe across concurrent calls.
 *  - Streams: `stream` is a cudaStream_t (CUstream) passed as void*; NULL = legacy
 *    default stream.  Work is stream-ordered; outputs are valid once the stream has
 *    synchronised.  Functions restore the caller's current device before returning.
 *  - Errors: argument errors are detected before any launch and leave outputs
 *    untouched.  Per-signal trouble (NaN in y_b, rank deficiency) never fails a call;
 *    it is reported in status[b].
 *  - There is no CPU fallback: every step runs in this library's sm_100a kernels.
 */
#ifndef OMP_B200_H
#define OMP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OMP_B200_VERSION 100  /* 1.0.0 */

typedef struct ompHandle_st* ompHandle_t;

typedef enum {
  OMP_OK = 0,
  OMP_ERR_INVALID_ARG = 1,   /* bad size / stride / pointer / option                     */
  OMP_ERR_ZERO_COLUMN = 2,   /* ||a_n|| = 0: selection divides by it; detail = n */
  OMP_ERR_NONFINITE = 3,     /* NaN/Inf in A; detail = column index                        */
  OMP_ERR_NOMEM = 4,         /* device allocation failed                                   */
  OMP_ERR_CUDA = 5,          /* a CUDA runtime/driver call failed; detail = cudaError_t     */
  OMP_ERR_UNSUPPORTED = 6    /* shape outside what the kernels support (e.g. S > 512)      */
} ompStatus_t;

/* per-signal outcome, status[b] */
typedef enum {
  OMP_SIG_MAXITER = 0,     /* k reached S                                     */
  OMP_SIG_EPS = 1,         /* ||r_k|| <= eps, tested from k = 0 (r_0 = y)    */
  OMP_SIG_DEGENERATE = 2,  /* n* re-selected, max correlation 0, or the factor pivot
                              ||a||^2 - ||z||^2 <= 1e-5 ||a||^2; the previous
                              x, support and ||r|| are kept                                  */
  OMP_SIG_NAN = 3          /* y_b (hence a correlation) is not finite                        */
} ompSigStatus_t;

/* how the correlation C = A^T R is evaluated.  In both tensor-core modes the
 * tcgen05 GEMM is a screen with a rigorous error bound; every atom inside the bound window is then
 * re-evaluated as an exact FP32 dot, so the selected atom is the FP32 argmax. */
typedef enum {
  OMP_CORR_BF16 = 0,        /* default: bf16 tcgen05 screen (kind::f16) + FP32 re-evaluation          */
  OMP_CORR_FP32_SIMT = 1,   /* FP32 FFMA GEMM writes C; standalone argmax kernel (fallback)           */
  OMP_CORR_3XTF32 = 2       /* 3xTF32 tcgen05 screen (kind::tf32, tighter window) + FP32 re-evaluation */
} ompCorrMode_t;

/* ompCreate — bind a dictionary to `device` and run the one-time setup (K0):
 *   validate A (finite, every ||a_n|| > 0), ||a_n|| in FP64 and 1/||a_n||,
 *   the screening planes of A^T, and the Gram matrix G = A^T A in FP32.
 *   Setup cost is amortised across batches.
 *   A: device, M x N column-major, lda >= M.  Synchronises `stream` before returning.
 *   Errors: OMP_ERR_INVALID_ARG (M,N < 1, lda < M, A == NULL, bad mode),
 *           OMP_ERR_ZERO_COLUMN / OMP_ERR_NONFINITE (no handle is returned),
 *           OMP_ERR_NOMEM, OMP_ERR_CUDA.                                                  */
ompStatus_t ompCreate(ompHandle_t* handle, int device, const float* A, int64_t M, int64_t N,
                      int64_t lda, int corr_mode, void* stream);

/* ompBatch — run OMP on B signals (all device pointers).
 *   Y: M x B column-major (ldy >= M).  S: 1 <= S <= min(M, N, 512).
 *   eps: residual-norm tolerance; eps < 0 or NaN means "no tolerance" (PAPER.md:35 optional).
 *   Outputs (written for every b):
 *     X[b*ldx + j]       coefficient of atom support[b*lds + j], j < n_iter[b]; 0 after
 *     support[b*lds + j] atom index in selection order, -1 for j >= n_iter[b]
 *     resid_norm[b]      ||y_b - A_S x_b|| of the returned x (NaN for OMP_SIG_NAN)
 *     n_iter[b]          number of selected atoms
 *     status[b]          ompSigStatus_t
 *   Coefficients are in the units of the given A (no 1/||a|| rescale is needed).
 *   Asynchronous on `stream`.                                                             */
ompStatus_t ompBatch(ompHandle_t handle, const float* Y, int64_t B, int64_t ldy, int32_t S, float eps,
                     float* X, int64_t ldx, int32_t* support, int64_t lds, float* resid_norm,
                     int32_t* n_iter, int32_t* status, void* stream);

/* ompBatchHost — ompBatch with HOST buffers (pageable or pinned): copies Y host->device,
 *   runs the batch and copies the five outputs device->host through handle-owned staging
 *   buffers; returns after `stream` has synchronised.  Same layouts and errors as ompBatch. */
ompStatus_t ompBatchHost(ompHandle_t handle, const float* Y_host, int64_t B, int64_t ldy, int32_t S,
                         float eps, float* X_host, int64_t ldx, int32_t* support_host, int64_t lds,
                         float* resid_norm_host, int32_t* n_iter_host, int32_t* status_host,
                         void* stream);

/* ompDensify — scatter compact results into a dense B x N row-major matrix
 *   (Xdense[b*ldxd + support[b,j]] = X[b,j], zero elsewhere; "x_hat").          */
ompStatus_t ompDensify(ompHandle_t handle, const float* X, int64_t ldx, const int32_t* support,
                       int64_t lds, const int32_t* n_iter, int64_t B, int32_t S, float* Xdense,
                       int64_t ldxd, void* stream);

/* ompCorrelate — the correlation GEMM alone: C[b*ldc + n] = sum_m R[b*ldr + m] A[m, n]
 *   ("a single call to gemm"), through the handle's correlation kernel
 *   (tensor-core modes return the SCREEN values, accurate to the mode's bound c0 ||a|| ||r||).
 *   R: B x M row-major (= M x B column-major), ldr >= M.  C: B x N row-major, ldc >= N.
 *   Diagnostic / test entry point.                                                         */
ompStatus_t ompCorrelate(ompHandle_t handle, const float* R, int64_t B, int64_t ldr, float* C,
                         int64_t ldc, void* stream);

/* ompScreeningWindow — the screen's candidate window W / ||r|| for a correlation mode and a
 *   dictionary of M rows (host-only arithmetic, no device work; callable without a GPU).
 *   In a tensor-core mode the exact selection n* = argmax |<r, a_n>| / ||a_n||
 *   re-evaluates in FP32 every atom whose screened value is within W ||r|| of the screen's
 *   maximum; W = 2.5 (c0 + c0'), c0 the rigorous per-element bound of the screen
 *   (bf16: 2^-7 + 2^-16 + 2^-22 + Mp 2^-23; 3xTF32: 2^-20 + 2^-22 + 3 Mp 2^-23) and c0' that of
 *   the FP32 re-evaluation, (Mp/32 + 8) 2^-23; Mp = M rounded up to 64.
 *   Returns -1 for M < 1 or a mode without a screen (OMP_CORR_FP32_SIMT) or an unknown mode.  */
float ompScreeningWindow(int corr_mode, int64_t M);

/* ompGetGram — copy G = A^T A (N x N row-major, ldg >= N) from the handle.                */
ompStatus_t ompGetGram(ompHandle_t handle, float* G, int64_t ldg, void* stream);

/* ompGetFactor — copy the inverse-Cholesky state of the last ompBatch for signals
 *   [b0, b0+count): F packed by columns (column j holds F[0..j, j] at offset j(j+1)/2,
 *   S(S+1)/2 floats per signal) and u = F^T A_k^T y (S floats per signal).  F_k = V_k^{-T}
 *   (PAPER.md:149-161).  Entries past n_iter[b] are unspecified.                          */
ompStatus_t ompGetFactor(ompHandle_t handle, int64_t b0, int64_t count, float* F, float* u,
                         void* stream);

/* ompSetGraphs — a batch's launch sequence (1 + 2S kernels; 1 + 3S in SIMT mode) is captured into a
 *   CUDA graph on first use and replayed on later calls with the same shape, eps and buffers
 *   (enable = 1, default; one graph launch per batch, PAPER.md:243 on per-call
 *   overhead), or launched kernel by kernel (enable = 0; debugging, sanitizers).  Same results.   */
ompStatus_t ompSetGraphs(ompHandle_t handle, int enable);

/* Profiling: when enabled, ompBatch brackets every kernel with CUDA events on `stream` (in the
 * captured graph: an external event-record node on either side of every kernel node, so a replayed
 * batch times its own kernels; a replay collects an earlier unread replay's times first);
 * ompProfileRead returns, per kernel slot (0 init, 1 correlation, 2 standalone argmax [SIMT
 * mode], 3 update = exact selection + factor append + residual, 4 small-batch persistent
 * kernel = all S iterations of a small batch in one launch), the summed
 * milliseconds and the number of launches since the last reset.  Reading synchronises the
 * events.                                                                                  */
#define OMP_NUM_KERNEL_SLOTS 5
ompStatus_t ompProfileEnable(ompHandle_t handle, int enable);
ompStatus_t ompProfileRead(ompHandle_t handle, double* ms, int64_t* launches, int reset);

/* ompSetAlgorithm — which formulation of the iteration a batch runs:
 *   OMP_ALGO_RESIDUAL: the residual path (a2-a5 above; the small-batch kernel for small B);
 *   OMP_ALGO_PROJECTION: the paper's algorithm v0 -- projections p = A^T r_k instead of the
 *     M-length residual.  Once per batch P0 = A^T Y (FP32 GEMM); per iteration, one kernel
 *     selects n* = argmax |p_n| / ||a_n||, appends the factor and recomputes
 *     p = P0 - sum_j x_j G[s_j, :] (O(N k) per signal).  The eps test uses
 *     ||r||^2 = ||y||^2 - ||u||^2 (q_j orthonormal); the returned resid_norm is the exact
 *     ||y - A_S x|| computed after the last iteration.  Cheaper when M is large against N
 *     (the paper's Yale shape, M = 8064, N = 1207).
 *   OMP_ALGO_AUTO (default): a per-signal-iteration cost model picks one.
 *   OMP_ERR_INVALID_ARG for any other value.                                               */
typedef enum { OMP_ALGO_AUTO = 0, OMP_ALGO_RESIDUAL = 1, OMP_ALGO_PROJECTION = 2 } ompAlgorithm_t;
ompStatus_t ompSetAlgorithm(ompHandle_t handle, int algorithm);

/* ompSetSmallBatchLimit — batches of at most `max_batch` signals run on the small-batch path:
 *   one persistent cooperative kernel for all S iterations (exact FP32 correlation over all N
 *   atoms, then factor append + residual per signal, PAPER.md:243 on
 *   per-call overhead at small batch sizes) instead of 1 + 2S launches.  Results are bitwise
 *   identical to the screened path's.  max_batch = -1 (default): automatic (B <= 8 and
 *   B * N * Mp <= 2^26, the measured crossover); 0: never; else B <= max_batch (<= 64).  Tensor-core correlation modes only (SIMT mode keeps its own argmax);
 *   the path also needs Mp <= 2048 and B x Mp x 4 bytes of shared memory (<= 150 KB), else the
 *   screened path runs.  OMP_ERR_INVALID_ARG for max_batch < -1.                           */
ompStatus_t ompSetSmallBatchLimit(ompHandle_t handle, int64_t max_batch);

/* Which path the last ompBatch ran: OMP_PATH_RESIDUAL (screen + update per iteration),
 * OMP_PATH_SMALL (the small-batch persistent kernel), OMP_PATH_PROJECTION (algorithm v0);
 * -1 for a NULL handle.                                                                   */
typedef enum { OMP_PATH_RESIDUAL = 0, OMP_PATH_SMALL = 1, OMP_PATH_PROJECTION = 2 } ompPath_t;
int ompGetLastPath(ompHandle_t handle);

/* Kernel launches issued by the last ompBatch (launch accounting; the per-iteration kernel
 * sequence of SURVEY §8(a) a1-a5: 1 + 2S, 1 + 3S in SIMT mode, 2 on the small-batch path).  */
int64_t ompGetLaunchCount(ompHandle_t handle);

/* ompDestroy — release everything the handle owns (synchronises its device): the dictionary
 *   copies and Gram matrix of ompCreate, the batch workspaces, cached graphs; restores the device's
 *   persisting-L2 limit when the last handle on the device goes (ownership: SURVEY §8(b)).     */
ompStatus_t ompDestroy(ompHandle_t handle);

/* ompGetErrorString — static text of a call-level status (SURVEY §8(b) "Errors").          */
const char* ompGetErrorString(ompStatus_t status);

/* ompGetErrorDetail — detail of the last error on this handle (the offending column of a zero or
 * non-finite atom, S:117-120 / S:132; a cudaError_t, ...); with handle == NULL, the detail of the
 * last failed ompCreate on this thread.                                                   */
int64_t ompGetErrorDetail(ompHandle_t handle);

/* omp_batch — one-shot convenience in the north-star's phrasing
 *   omp_batch(A, Y[M x B], S, eps) -> X, support sets, residual norms:
 *   ompCreate + ompBatch + ompDestroy on the current device, lda = ldy = M, ldx = lds = S.
 *   Synchronises `stream`.                                                                 */
ompStatus_t omp_batch(const float* A, int64_t M, int64_t N, const float* Y, int64_t B, int32_t S,
                      float eps, float* X, int32_t* support, float* resid_norm, int32_t* n_iter,
                      int32_t* status, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* OMP_B200_H */
