"""Phase breakdown of the per-iteration update kernel (diagnostic; not part of the product).

    python scripts/trace_update.py [config] [B] [k ...]

Builds paper_2407_06434_b200/libomp_b200_trace.so with -DOMP_UPDATE_TRACE if it is missing (do it on
the CPU side: `python scripts/trace_update.py --build`), loads it through OMP_B200_LIB, and for each
traced iteration k prints thread 0's clock64 time per phase, averaged over the launch's CTAs.
"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "paper_2407_06434_b200", "libomp_b200_trace.so")

PHASES = {0: "partials+cand list", 1: "wait rows", 2: "refine dots", 4: "w (Gram row)", 5: "z = F^T w",
          6: "|z|^2", 7: "F z, F u", 8: "gather", 9: "y, |r|^2", 11: "eps + planes"}


def build():
    from paper_2407_06434_b200 import build as b
    b.build(defines=["-DOMP_UPDATE_TRACE"], out=LIB)


def main():
    if "--build" in sys.argv:
        build()
        return
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
    ks = [int(x) for x in sys.argv[3:]] or [16, 64, 120]
    if not os.path.exists(LIB):
        build()
    os.environ["OMP_B200_LIB"] = LIB
    os.environ["OMP_B200_GRAPH"] = "0"
    import numpy as np
    import torch
    from synth import make_problem
    from paper_2407_06434_b200 import OMP
    prob = make_problem(cfg, B=B, device="cuda")
    h = OMP(torch.as_tensor(prob.A).cuda())
    Y = torch.as_tensor(prob.Y).cuda()
    lib = ctypes.CDLL(LIB)
    lib.omp_debug_update_trace.argtypes = [ctypes.c_int, ctypes.c_void_p]
    h.batch(Y, prob.S, prob.eps)
    torch.cuda.synchronize()
    for k in ks:
        lib.omp_debug_update_trace(k, None)
        h.batch(Y, prob.S, prob.eps)
        torch.cuda.synchronize()
        buf = (ctypes.c_ulonglong * 16)()
        lib.omp_debug_update_trace(k, buf)
        v = np.array(buf, dtype=np.float64)
        n = max(1.0, v[15])
        tot = sum(v[p] for p in PHASES) / n
        print(f"{cfg} B={B} k={k}: {int(n)} CTAs, {tot:.0f} cycles per CTA")
        for p, name in PHASES.items():
            print(f"   {name:20s} {v[p] / n:9.0f}  {100 * v[p] / n / tot:5.1f} %")
        print(f"   candidates: mean {v[12] / n:.2f}, > 16: {int(v[13])}, with an overflowing group: {int(v[14])}, "
              f"all-N fallback: {int(v[3])} of {int(n)} signals")
        fq = (ctypes.c_ulonglong * 8)()
        lib.omp_debug_update_freq.argtypes = [ctypes.c_void_p]
        lib.omp_debug_update_freq(fq)
        f = np.array(fq, dtype=np.float64)
        mhz = [1e3 * (f[2 * e] - f[2 * s]) / max(1.0, f[2 * e + 1] - f[2 * s + 1]) for s, e in ((0, 1), (2, 3))]
        print(f"   SM clock inside the launch: first CTA {mhz[0]:.0f} MHz, last CTA {mhz[1]:.0f} MHz")


if __name__ == "__main__":
    main()
