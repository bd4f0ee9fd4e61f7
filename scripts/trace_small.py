"""Timeline of the small-batch persistent kernel (diagnostic; OMP_B200_SMALL_TRACE=1)."""
import ctypes, os, sys
import numpy as np
os.environ["OMP_B200_SMALL_TRACE"] = "1"
os.environ["OMP_B200_GRAPH"] = "0"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import make_problem
from paper_2407_06434_b200 import OMP, _lib
cfg, B = sys.argv[1], int(sys.argv[2])
prob = make_problem(cfg, B=B)
h = OMP(torch.from_numpy(prob.A).cuda())
Y = torch.from_numpy(prob.Y).cuda()
for _ in range(3):
    h.batch(Y, prob.S)
torch.cuda.synchronize()
lib = ctypes.CDLL(_lib.LIB_PATH)
buf = (ctypes.c_ulonglong * (8 * prob.S))()
lib.omp_debug_small_trace(buf, prob.S)
t = np.array(buf, dtype=np.float64).reshape(prob.S, 8)[:, :7]
d = np.diff(t, axis=1)
names = ["live+stage", "phaseA", "barrier1", "select", "tail", "barrier2"]
print(f"{cfg} B={B}: per-iteration ns (mean over k, then k=0, k=S/2, k=S-1)")
for i, nm in enumerate(names):
    print(f"  {nm:12s} {d[:, i].mean():8.0f} {d[0, i]:8.0f} {d[prob.S // 2, i]:8.0f} {d[-1, i]:8.0f}")
it = t[1:, 0] - t[:-1, 0]
print(f"  iteration    {it.mean():8.0f}")
c = (ctypes.c_ulonglong * (8 * prob.S))()
lib.omp_debug_small_clk(c, prob.S)
cc = np.array(c, dtype=np.float64).reshape(prob.S, 8)[:, :7]
dc = np.diff(cc, axis=1)
print("  cycles:", " ".join(f"{nm}={dc[:, i].mean():.0f}" for i, nm in enumerate(names)))
print(f"  SM clock from clock64/globaltimer: {(cc[-1, 6] - cc[0, 0]) / (t[-1, 6] - t[0, 0]) * 1e3:.0f} MHz")
x = np.array(buf, dtype=np.float64).reshape(prob.S, 8)
print(f"  select: pbest loads {np.mean(x[:, 7] - x[:, 3]):.0f} ns, then {np.mean(x[:, 4] - x[:, 7]):.0f} ns")
xc = np.array(c, dtype=np.float64).reshape(prob.S, 8)
print(f"  select cycles: pbest loads {np.mean(xc[:, 7] - xc[:, 3]):.0f}, then {np.mean(xc[:, 4] - xc[:, 7]):.0f}")
tc = (ctypes.c_ulonglong * (8 * prob.S))()
lib.omp_debug_tail_clk(tc, prob.S)
tcc = np.array(tc, dtype=np.float64).reshape(prob.S, 8)[:, :6]
tcc = np.concatenate([xc[:, 4:5], tcc], axis=1)
dd = np.diff(tcc, axis=1)
tn = ["w/dup", "z", "zz", "v/t+wait", "gather", "y+norm"]
print("  tail cycles:", " ".join(f"{nm}={dd[1:, i].mean():.0f}" for i, nm in enumerate(tn)))
print("  tail cycles k=S-1:", " ".join(f"{nm}={dd[-1, i]:.0f}" for i, nm in enumerate(tn)))
