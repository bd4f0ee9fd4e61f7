"""Warp-stall samples per CUDA source line from an ncu report (dev tool; runs without a GPU):

    python scripts/ncu_hot_lines.py gpurun_out/prof_TAG.ncu-rep [top]

Uses `ncu -i REP --page source --csv --print-source cuda,sass`; the source-line rows carry the sums of
their SASS rows.  Prints the top lines by samples with their executed instructions.
"""
import csv
import io
import subprocess
import sys


def main(rep, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = []
    fname = "?"
    total = 0
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] and r[0].isdigit() and len(r) > 7 and r[4].isdigit():
            s = int(r[4])
            total += s
            rows.append((s, int(r[5]), fname, int(r[0]), r[1].strip()[:90], r[7]))
    rows.sort(reverse=True)
    print(f"total samples {total}")
    for s, ni, f, ln, src, inst in rows[:top]:
        print(f"{100.0 * s / max(1, total):5.1f}%  {s:7d} (not-issued {ni:6d}) inst {inst:>12s}  {f}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
