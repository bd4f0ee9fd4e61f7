#!/bin/bash
# ncu evidence for the bench workload (run under gpurun; single GPU).  Usage: scripts/profile_round.sh TAG [extra bench args]
set -u
TAG=${1:-r01}; shift || true
OUT=gpurun_out
mkdir -p $OUT
# 1) every launch of one bench step with its device time (cold-cache, serialised: compare SHARES)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_${TAG}.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline "$@" > $OUT/launches_${TAG}.bench.json 2> $OUT/launches_${TAG}.err
echo "launch list rc=$?"
# 2) one full capture of each hot kernel at iteration 64 (k = 64 = mean support size at c4)
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k1_corr_tc|k_update" -s 128 -c 2 -o $OUT/prof_${TAG} -f \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline "$@" > $OUT/prof_${TAG}.bench.json 2> $OUT/prof_${TAG}.err
echo "full capture rc=$?"
ls -la $OUT
