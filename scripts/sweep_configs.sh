#!/bin/bash
# One bench line per BASELINE config (and the paper's own shapes), current build; run under gpurun.
#   scripts/sweep_configs.sh TAG   -> gpurun_out/sweep_TAG.jsonl
set -u
TAG=${1:-r01h}
OUT=gpurun_out/sweep_${TAG}.jsonl
mkdir -p gpurun_out
: > $OUT
run() {   # label, bench args...
  local label=$1; shift
  local line
  line=$(timeout 600 python bench.py --no-cpu-baseline "$@" 2> gpurun_out/sweep_${TAG}_${label}.err | tail -1)
  echo "{\"label\": \"$label\", \"args\": \"$*\", \"line\": ${line:-null}}" >> $OUT
}
run tiny --config tiny --no-kernel-profile --steps 20
run c2 --config c2 --no-kernel-profile --steps 20
run c2_simt --config c2 --mode simt --no-kernel-profile --steps 20
run c2_3xtf32 --config c2 --mode 3xtf32 --no-kernel-profile --steps 20
run c3 --config c3 --no-kernel-profile --steps 10
run c3_3xtf32 --config c3 --mode 3xtf32 --no-kernel-profile --steps 10
for B in 1 10 100 1000 10000 100000 1000000; do
  st=10; [ $B -ge 100000 ] && st=3
  run c5_B$B --config c5 --batch $B --no-kernel-profile --steps $st
done
run c4_3xtf32 --config c4 --mode 3xtf32 --steps 2 --warmup 3
run yale --config yale --no-kernel-profile --steps 10
run t2m1024 --config t2m1024 --no-kernel-profile --steps 5
run t2m2048 --config t2m2048 --no-kernel-profile --steps 3
python - "$OUT" <<'EOF'
import json, sys
for l in open(sys.argv[1]):
    d = json.loads(l)
    x = d["line"] or {}
    e = (x.get("e2e") or {}).get("value")
    print(f'{d["label"]:12s} {x.get("value", 0):>14,.0f} signals/s  ms/step {x.get("ms_per_step", 0):9.3f}  e2e {e or 0:>14,.0f}  path {x.get("config", {}).get("path")}')
EOF
