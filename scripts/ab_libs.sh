#!/bin/bash
# A/B/... of library builds (OMP_B200_LIB) on a set of bench configs (graph path), interleaved on one box:
#   bash scripts/ab_libs.sh TAG "libA.so libB.so ..." "bench args 1" "bench args 2" ...
# (library names relative to paper_2407_06434_b200/)
set -u
TAG=$1; LIBS=$2; shift 2
OUT=gpurun_out/ab_${TAG}.txt
mkdir -p gpurun_out
for args in "$@"; do
  for rep in 1 2; do
    for lib in $LIBS; do
      line=$(env OMP_B200_LIB=$PWD/paper_2407_06434_b200/$lib timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-kernel-profile $args 2>/dev/null | tail -1)
      python - "$lib" "$args" "$line" >> $OUT <<'PY'
import json, sys
v, args, line = sys.argv[1:4]
try:
    d = json.loads(line)
    k = d.get("kernels", {})
    upd = k.get("update", {})
    cor = k.get("correlation", {})
    print(f"{args:45s} {v:>24s}  {d['value']:14,.0f} signals/s  {d['ms_per_step']:9.3f} ms/step  update {upd.get('ms_total', 0) / max(1, upd.get('launches', 1)):.4f} ms  corr {cor.get('ms_total', 0) / max(1, cor.get('launches', 1)):.4f} ms  clk {d['clocks'].get('sm_mhz')}")
except Exception as e:
    print(f"{args:45s} {v:>24s}  FAILED {e}")
PY
    done
  done
done
cat $OUT
