"""Summarise an ncu --set full report and a launch-list CSV into profiles/ (dev tool, runs on CPU).

    python scripts/summarize_ncu.py TAG CONFIG   # reads gpurun_out/prof_TAG.ncu-rep, launches_TAG.csv
"""

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"k1_corr_tc": "correlation", "k1_corr_simt": "correlation", "k2_refine": "select", "k2_select": "select",
        "k3_factor": "factor_append", "k4_residual": "residual", "k_batch_init": "init", "k_update": "update",
        "k_small": "small", "k_sum_slabs": "slab_sum", "k_final_resid": "final_resid", "k_make_planes": "planes"}
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Tbyte": 1e12, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
         "s": 1.0, "Ghz": 1e9, "Mhz": 1e6}


def key_of(name):
    for k, v in KEYS.items():
        if k in name:
            return v
    return None


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = {}
    for d in data:
        k = key_of(d[hdr.index("Kernel Name")])
        if not k:
            continue
        ent = {"kernel_name": d[hdr.index("Kernel Name")].split("(")[0]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(d[i].replace(",", ""))
                except ValueError:
                    continue
                ent[m] = v * SCALE.get(units[i], 1.0) if units[i] in SCALE else v
        ent["dram_bytes_per_launch"] = ent.get("dram__bytes_read.sum", 0) + ent.get("dram__bytes_write.sum", 0)
        ent["l2_bytes_per_launch"] = 32.0 * ent.get("lts__t_sectors.sum", 0)
        res[k] = ent
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = key_of(d["Kernel Name"]) or d["Kernel Name"].split("(")[0][:40]
        v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
        tot[k] += v
        cnt[k] += 1
    allt = sum(tot.values())
    return {k: {"launches": cnt[k], "total_ms": tot[k] * 1e3, "share": tot[k] / allt} for k in tot}


def main():
    tag, cfg = sys.argv[1], sys.argv[2]
    rep = os.path.join(ROOT, "gpurun_out", f"prof_{tag}.ncu-rep")
    lst = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    summ_path = os.path.join(prof, "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {"configs": {}}
    full = raw(rep) if os.path.exists(rep) else {}
    share = launches(lst) if os.path.exists(lst) else {}
    summ["configs"][cfg] = {**full, "_launch_shares": share, "_tag": tag}
    json.dump(summ, open(summ_path, "w"), indent=1, sort_keys=True)
    lines = [f"# ncu summary {tag} ({cfg})", "",
             "Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, one bench step, "
             "cold-cache and serialised: compare shares, not absolutes):", "",
             "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(share.items(), key=lambda kv: -kv[1]["total_ms"]):
        lines.append(f"| {k} | {v['launches']} | {v['total_ms']:.2f} | {100 * v['share']:.1f}% |")
    lines += ["", "Full capture (`ncu --set full`; which launches: see `scripts/profile_round.sh` / the round notes):", "",
              "| kernel | time ms | DRAM read GB | DRAM write GB | L2 bytes GB | DRAM % | L2 % | SM % | tensor % | regs |",
              "|---|---|---|---|---|---|---|---|---|---|"]
    for k, e in full.items():
        lines.append("| {} | {:.3f} | {:.3f} | {:.3f} | {:.2f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.0f} |".format(
            e["kernel_name"], e.get("gpu__time_duration.sum", 0) * 1e3, e.get("dram__bytes_read.sum", 0) / 1e9,
            e.get("dram__bytes_write.sum", 0) / 1e9, e.get("l2_bytes_per_launch", 0) / 1e9,
            e.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 0),
            e.get("lts__throughput.avg.pct_of_peak_sustained_elapsed", 0),
            e.get("sm__throughput.avg.pct_of_peak_sustained_elapsed", 0),
            e.get("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                  e.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0)),
            e.get("launch__registers_per_thread", 0)))
    open(os.path.join(prof, f"ncu_{tag}_{cfg}.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
