#!/bin/bash
# ncu --set full of one update-kernel launch (iteration K) of a bench step (run under gpurun; 1 GPU):
#   bash scripts/profile_update.sh TAG CONFIG BATCH K [extra bench args]  -> gpurun_out/prof_TAG.ncu-rep
set -u
TAG=$1; CFG=$2; B=$3; K=$4; shift 4
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_update" -s $K -c 1 -o $OUT/prof_$TAG -f \
  python bench.py --config $CFG --batch $B --steps 1 --warmup 0 --no-e2e --no-cpu-baseline "$@" \
  > $OUT/prof_$TAG.bench.json 2> $OUT/prof_$TAG.err
echo "full capture $TAG rc=$?"
ncu -i $OUT/prof_$TAG.ncu-rep --page details --csv > $OUT/prof_$TAG.details.csv 2>/dev/null
ncu -i $OUT/prof_$TAG.ncu-rep --page raw --csv > $OUT/prof_$TAG.raw.csv 2>/dev/null
ncu -i $OUT/prof_$TAG.ncu-rep --page source --csv > $OUT/prof_$TAG.source.csv 2>/dev/null
ls -la $OUT/prof_$TAG*
