"""Quick numerics check of the correlation kernel (K1) against FP64 (dev tool)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_06434_b200 import OMP  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "3xtf32"
for (M, N, B) in [(32, 256, 128), (64, 512, 300), (256, 1024, 1000), (1024, 4096, 520), (2048, 8192, 4096)]:
    rng = np.random.default_rng(M + N + B)
    A = rng.standard_normal((M, N)).astype(np.float32)
    R = rng.standard_normal((B, M)).astype(np.float32)
    t = time.time()
    with OMP(torch.from_numpy(A).cuda(), mode=mode) as h:
        C = h.correlate(torch.from_numpy(R).cuda()).cpu().numpy()
    ref = R.astype(np.float64) @ A.astype(np.float64)
    scale = np.linalg.norm(R, axis=1)[:, None] * np.linalg.norm(A, axis=0)[None, :]
    err = np.abs(C - ref) / scale
    bad = np.argwhere(err > 1e-5)
    print(f"{mode} cg={os.environ.get('OMP_B200_CTA_GROUP', '2')} M={M} N={N} B={B}: max err {err.max():.3e} "
          f"bad={len(bad)} first={bad[:3].tolist()} ({time.time() - t:.2f}s)", flush=True)
