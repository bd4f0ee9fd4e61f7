"""Survey-sized parity of the CUDA path against the FP64 oracle, per config and path, as one JSON
report (SURVEY §8(c) "Report", §8(d) "Oracle / parity subsample"; run on the GPU box):

    python scripts/parity_report.py [--out profiles/parity_r02.json] [--only c4,c3]

Every config runs at its full BASELINE.json batch in the library's own launch configuration
(the default path is what bench.py times); the sampled rows are compared signal by signal with the
protocol of tests/parity.py.  Oracle results come from tests/golden/oracle_cache (written by
scripts/build_oracle_cache.py from synth + oracle only) when the signal's FP32 bytes match, else
the oracle runs on the spot.  Outcome counts, the oracle's flag counts on the sample, the largest
coefficient / residual errors and any bug are written per (config, path).
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

from gpu_helpers import eps32, run_gpu  # noqa: E402
from oracle_cache import SAMPLES, oracle_for_rows  # noqa: E402
from parity import compare_batch  # noqa: E402
from synth import make_problem  # noqa: E402

FLAG_KINDS = ("primary", "extended", "stop", "near_degenerate")


def flags_of(o):
    if hasattr(o, "flags"):
        return o.flags
    return dict(primary=any(s.primary_tie for s in o.steps), extended=any(s.extended_tie for s in o.steps),
                stop=bool(o.init_stop_flag) or any(s.stop_flag for s in o.steps),
                near_degenerate=any(s.near_degenerate for s in o.steps))


def one(report, label, name, prob, mode, rows, cache_name=None):
    t0 = time.time()
    out = run_gpu(prob.A, prob.Y, prob.S, prob.eps, mode)
    t_gpu = time.time() - t0
    rows = [int(r) for r in rows]
    if cache_name:
        ora, hits = oracle_for_rows(cache_name, prob.A, prob.Y, rows, prob.indices, prob.S, eps32(prob.eps))
    else:
        from oracle import omp_batch
        ora, hits = omp_batch(prob.A, prob.Y[rows], prob.S, eps32(prob.eps)), 0
    rep = compare_batch(out["support"], out["X"], out["resid"], out["n_iter"], out["status"], ora, prob.N, rows=rows)
    d = rep.as_dict()
    flags = {k: int(sum(bool(flags_of(o)[k]) for o in ora)) for k in FLAG_KINDS}
    entry = dict(config=name, path=out["path"], mode=mode, batch=int(prob.B), signals_compared=len(rows),
                 oracle_from_cache=int(hits), outcomes=d["counts"], bugs=d["bugs"],
                 oracle_flagged_signals=flags, max_coef_rel_err=d["max_coef_err"],
                 max_resid_err_over_ynorm=d["max_res_err_over_ynorm"],
                 statuses={int(k): int(v) for k, v in zip(*np.unique(out["status"], return_counts=True))},
                 gpu_s=round(t_gpu, 2), total_s=round(time.time() - t0, 2))
    report[label] = entry
    print(json.dumps({label: entry}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "parity_r02.json"))
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    only = set(filter(None, args.only.split(",")))
    report = {}

    def want(n):
        return not only or n in only

    if want("tiny"):
        p = make_problem("tiny")
        for mode in ("bf16", "3xtf32", "simt", "small", "proj"):
            one(report, f"tiny/{mode}", "tiny", p, mode, range(p.B))
    if want("c2"):
        p = make_problem("c2")
        for mode in ("auto", "3xtf32", "simt", "proj"):
            one(report, f"c2/{mode}", "c2", p, mode, range(p.B))
    if want("c3"):
        p = make_problem("c3", device="cuda")
        for mode in ("auto", "3xtf32", "simt"):
            one(report, f"c3/{mode}", "c3", p, mode, SAMPLES["c3"], "c3")
    if want("c4"):
        p = make_problem("c4", device="cuda")
        for mode in ("auto", "3xtf32"):
            one(report, f"c4/{mode}", "c4", p, mode, SAMPLES["c4"], "c4")
    if want("c5"):
        p = make_problem("c5", device="cuda")                        # B = 10^6
        one(report, "c5_B1e6/auto", "c5", p, "auto", SAMPLES["c5"], "c5")
        for B in (1, 10, 100, 1000, 10000, 100000):
            q = make_problem("c5", B=B, device="cuda" if B > 1000 else None)
            rows = np.unique(np.linspace(0, B - 1, min(B, 200)).astype(int))
            one(report, f"c5_B{B}/auto", "c5", q, "auto", rows, "c5")
    if want("yale"):
        p = make_problem("yale")
        one(report, "yale/auto", "yale", p, "auto", range(0, p.B, 6))
    total = {k: sum(e["outcomes"].get(k, 0) for e in report.values())
             for k in ("exact", "flagged_ok", "tie_divergent", "explained", "bug")}
    doc = dict(what=__doc__.strip().splitlines()[0], protocol="tests/parity.py (SURVEY §8(c)); tolerances: supports "
               "exact outside oracle-flagged steps, coefficients <= 1e-4 relative L2, |r| within 1e-4 |r| + 1e-5 |y|",
               totals=total, signals=sum(e["signals_compared"] for e in report.values()), runs=report)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(dict(totals=total, signals=doc["signals"])))
    return 1 if total["bug"] else 0


if __name__ == "__main__":
    sys.exit(main())
