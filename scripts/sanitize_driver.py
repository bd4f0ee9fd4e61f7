"""One small run of every library path, for compute-sanitizer (scripts/sanitize.sh):

    compute-sanitizer --tool memcheck python scripts/sanitize_driver.py [paths...]

Paths: bf16, 3xtf32, simt (screened residual path in each correlation mode, direct launches and the
CUDA-graph replay), small (the persistent small-batch kernel), proj (the projection path, 3xTF32 P0),
proj_simt (the projection path with the SIMT P0 GEMM), host (ompBatchHost, chunked), densify, correlate,
variants (the update's one-warp and 512-thread launch shapes).
Shapes: tiny and c2-like with a ragged B, eps stops on half the signals.  Each result is checked
for sanity (statuses, supports in range) so a silent corruption also fails the run.
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2407_06434_b200 import OMP  # noqa: E402
from synth import make_dictionary, make_signals  # noqa: E402


def check(r, N, S):
    sup = r.support.cpu().numpy()
    nit = r.n_iter.cpu().numpy()
    st = r.status.cpu().numpy()
    assert np.all((st >= 0) & (st <= 3)), st
    assert np.all((nit >= 0) & (nit <= S))
    for b in range(sup.shape[0]):
        k = nit[b]
        assert np.all((sup[b, :k] >= 0) & (sup[b, :k] < N)) and np.all(sup[b, k:] == -1), (b, sup[b])
    assert np.all(np.isfinite(r.X.cpu().numpy()))


def run(path, M, N, B, S, seed):
    A = make_dictionary(M, N, seed)
    Y = make_signals(A, range(B), seed, max(2, S // 2), sigma=0.01)
    Ad, Yd = torch.from_numpy(A).cuda(), torch.from_numpy(Y).cuda()
    mode = {"3xtf32": "3xtf32", "simt": "simt"}.get(path, "bf16")
    if path == "proj_simt":
        os.environ["OMP_B200_P0"] = "simt"
    with OMP(Ad, mode=mode) as h:
        h.set_small_batch_limit(64 if path == "small" else 0)
        h.set_algorithm("projection" if path.startswith("proj") else "residual")
        eps = 0.05
        if path == "host":
            r = h.batch_host(Y, S, eps)
            assert np.all(r.n_iter <= S)
            return
        if path == "densify":
            r = h.batch(Yd, S, eps)
            Xd = h.densify(r)
            torch.cuda.synchronize()
            assert Xd.shape == (B, N)
            return
        if path == "correlate":
            C = h.correlate(Yd)
            torch.cuda.synchronize()
            assert torch.isfinite(C).all()
            return
        h.profile(True)                    # direct launches
        r1 = h.batch(Yd, S, eps)
        torch.cuda.synchronize()
        check(r1, N, S)
        h.profile(False)                   # captured into a CUDA graph, then replayed
        for _ in range(2):
            r2 = h.batch(Yd, S, eps)
            torch.cuda.synchronize()
        check(r2, N, S)
        assert torch.equal(r1.support, r2.support) and torch.equal(r1.X, r2.X)
    if path == "proj_simt":
        os.environ.pop("OMP_B200_P0")


def main(paths):
    paths = paths or ["bf16", "3xtf32", "simt", "small", "proj", "host", "densify", "correlate"]
    for path in paths:
        if path == "variants":
            # the update's launch-shape variants the shapes above do not reach: one warp per signal
            # (B >= 8192 at M <= 512: no staged residual row, ||r||^2 in registers), and one CTA of 512
            # threads per SM (B <= 2 x SMs at M = 2048, F_k in L2 from k = 64)
            for (M, N, B, S) in ((512, 1024, 8200, 3), (2048, 4096, 12, 68)):
                run("bf16", M, N, B, S, 7)
            print("sanitize_driver: variants ok", flush=True)
            continue
        for (M, N, B, S) in ((32, 64, 16, 4), (256, 1024, 300 if path != "small" else 12, 32)):
            run(path, M, N, B, S, 7)
        print(f"sanitize_driver: {path} ok", flush=True)
    # every library handle is destroyed by now; hand torch's cached device / pinned blocks back too, so
    # memcheck --leak-check full reports only what the library itself might have leaked
    import gc
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    if hasattr(torch._C, "_host_emptyCache"):
        torch._C._host_emptyCache()


if __name__ == "__main__":
    main(sys.argv[1:])
