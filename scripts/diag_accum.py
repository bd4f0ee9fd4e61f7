"""Accumulation-error diagnostics for the correlation kernel (dev tool)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_06434_b200 import OMP  # noqa: E402
from synth import make_problem  # noqa: E402


def run(mode, A, R):
    with OMP(torch.from_numpy(A).cuda(), mode=mode) as h:
        return h.correlate(torch.from_numpy(R).cuda()).cpu().numpy().astype(np.float64)


# 1) positive data: truncation shows up as a negative mean error
for K in (256, 1024, 2048):
    rng = np.random.default_rng(K)
    A = rng.uniform(0.5, 1.0, (K, 512)).astype(np.float32)
    R = rng.uniform(0.5, 1.0, (256, K)).astype(np.float32)
    ref = R.astype(np.float64) @ A.astype(np.float64)
    for mode in ("3xtf32", "simt"):
        C = run(mode, A, R)
        rel = (C - ref) / ref
        print(f"positive K={K} {mode:7s}: mean rel err {rel.mean():+.3e}  max |rel| {np.abs(rel).max():.3e}")

# 2) OMP-like data: error relative to the row's top normalised correlation t1
prob = make_problem("c4", B=512, device="cuda")
A, Y = prob.A, prob.Y
ref = Y.astype(np.float64) @ A.astype(np.float64)
t1 = np.abs(ref).max(axis=1, keepdims=True)
for mode in ("3xtf32", "simt"):
    C = run(mode, A, Y)
    e = np.abs(C - ref) / t1
    top = np.argmax(np.abs(ref), axis=1)
    etop = np.abs(C[np.arange(len(top)), top] - ref[np.arange(len(top)), top]) / t1[:, 0]
    print(f"c4 y: {mode:7s}: max err/t1 {e.max():.3e}  p99 {np.quantile(e, 0.99):.3e}  top-atom err/t1 max {etop.max():.3e}")
# a late-iteration-like residual: y minus its projection on the true support plus noise
rng = np.random.default_rng(0)
Rr = (rng.standard_normal(Y.shape) * 0.01).astype(np.float32)
ref = Rr.astype(np.float64) @ A.astype(np.float64)
t1 = np.abs(ref).max(axis=1, keepdims=True)
for mode in ("3xtf32", "simt"):
    C = run(mode, A, Rr)
    e = np.abs(C - ref) / t1
    print(f"noise r: {mode:7s}: max err/t1 {e.max():.3e}  p99 {np.quantile(e, 0.99):.3e}")
