"""Write tests/golden/oracle_cache/{c3,c4,c5}.npz: FP64 oracle results for the survey-sized parity
samples (tests/oracle_cache.py SAMPLES).  Calls only synth (inputs) and oracle (Algorithm 1).

    python scripts/build_oracle_cache.py [c4 c3 c5] [--workers N]
"""

import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

from oracle import host_cores, omp_batch  # noqa: E402
from oracle_cache import SAMPLES, save  # noqa: E402
from synth import make_problem  # noqa: E402
from synth.generator import config  # noqa: E402


def main(argv):
    names = [a for a in argv if not a.startswith("--")] or ["c5", "c3", "c4"]
    workers = host_cores()
    if "--workers" in argv:
        workers = int(argv[argv.index("--workers") + 1])
    for name in names:
        rows = SAMPLES[name]
        t0 = time.time()
        prob = make_problem(name, indices=rows)          # numpy generator (the reference inputs)
        cfg = config(name)
        eps = None if cfg["eps"] is None else float(__import__("numpy").float32(cfg["eps"]))
        res = omp_batch(prob.A, prob.Y, prob.S, eps, workers=workers)
        path = save(name, cfg["seed"], prob.S, eps, rows, prob.Y, res)
        print(f"{name}: {len(rows)} signals in {time.time() - t0:.1f} s on {workers} workers -> {path}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
