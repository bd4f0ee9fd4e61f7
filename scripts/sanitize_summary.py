"""Summarise compute-sanitizer logs of scripts/sanitize.sh (profiles/r02/sanitize/):
errors per tool and, for memcheck's leak report, which allocations came from libomp_b200.so versus
from torch's caching allocators (blocks the test driver's tensors still hold at exit)."""
import re
import sys


def leaks(text):
    out = {"library": 0, "torch": 0, "other": 0}
    for block in re.split(r"========= Leaked ", text)[1:]:
        frames = block.split("=========     Saved host backtrace")[1] if "Saved host backtrace" in block else block
        frames = frames.split("=========\n")[0]
        if "libomp_b200" in frames:
            out["library"] += 1
        elif "c10::" in frames or "at::" in frames:
            out["torch"] += 1
        else:
            out["other"] += 1
    return out


def main(paths):
    for p in paths:
        t = open(p).read()
        errs = [int(x) for x in re.findall(r"ERROR SUMMARY: (\d+) error", t)]
        race = re.findall(r"RACECHECK SUMMARY: .*", t)
        print(p, "error summaries:", errs, race or "", "leaks:", leaks(t))
        if "racecheck" in p:
            pcs = sorted(set(re.findall(r"(Read|Write) access at [^+]*\+(0x[0-9a-f]+)", t)))
            print("   racecheck access sites:", pcs)


if __name__ == "__main__":
    main(sys.argv[1:])
