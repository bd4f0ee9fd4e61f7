#!/bin/bash
# ncu evidence for the small-batch kernel and the projection path (run under gpurun; single GPU).
#   scripts/profile_paths.sh TAG
set -u
TAG=${1:-r01f}
OUT=gpurun_out
mkdir -p $OUT
# projection path, Yale shape: launch list of one step, then full captures of P0 (split-K GEMM + slab sum)
# and of the update at iteration 15 (k = 15, the mean support size)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_${TAG}_yale.csv \
  python bench.py --config yale --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/launches_${TAG}_yale.log 2>&1
echo "yale launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_corr_simt|k_sum_slabs" -c 2 \
  -o $OUT/prof_${TAG}_yalegemm -f python bench.py --config yale --steps 1 --warmup 0 --no-e2e --no-cpu-baseline \
  > $OUT/prof_${TAG}_yalegemm.log 2>&1
echo "yale gemm capture rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_update" -s 15 -c 1 \
  -o $OUT/prof_${TAG}_yaleupd -f python bench.py --config yale --steps 1 --warmup 0 --no-e2e --no-cpu-baseline \
  > $OUT/prof_${TAG}_yaleupd.log 2>&1
echo "yale update capture rc=$?"
# small-batch kernel, c5 B = 1 (the whole 50-iteration solve is one launch)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_small" -c 1 \
  -o $OUT/prof_${TAG}_c5b1 -f python bench.py --config c5 --batch 1 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline \
  > $OUT/prof_${TAG}_c5b1.log 2>&1
echo "c5 B=1 capture rc=$?"
ls -la $OUT | grep $TAG
