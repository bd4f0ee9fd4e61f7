#!/bin/bash
# compute-sanitizer over every library path (scripts/sanitize_driver.py), one log per tool, plus the
# GPU parity tests of the small configs with every workspace NaN-filled at allocation
# (OMP_B200_DEBUG_FILL=1).  Run under gpurun:  bash scripts/sanitize.sh TAG  -> gpurun_out/sanitize_TAG_*.txt
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check full"
  for paths in "bf16 3xtf32 simt small proj host densify correlate" "proj_simt" "variants"; do
    echo "=== $tool: $paths" >> $OUT/sanitize_${TAG}_${tool}.txt
    if [ "$paths" = proj_simt ]; then envp="OMP_B200_P0=simt"; else envp=""; fi
    env $envp timeout 1500 $CS --tool $tool $extra --error-exitcode 17 --target-processes all \
      python scripts/sanitize_driver.py $paths >> $OUT/sanitize_${TAG}_${tool}.txt 2>&1
    echo "=== rc=$?" >> $OUT/sanitize_${TAG}_${tool}.txt
  done
  grep -E "ERROR SUMMARY|LEAK SUMMARY|RACECHECK SUMMARY|=== rc|sanitize_driver" $OUT/sanitize_${TAG}_${tool}.txt
done
# the screen with single-SM UMMA (no cluster mbarrier traffic between CTA pairs): racecheck's hazards on
# the 2-CTA kernel are between mbarrier instructions (SYNCS try_wait / remote arrive) only
echo "=== racecheck cta_group::1: bf16 3xtf32" >> $OUT/sanitize_${TAG}_racecheck_cg1.txt
OMP_B200_CTA_GROUP=1 timeout 1500 $CS --tool racecheck --error-exitcode 17 python scripts/sanitize_driver.py bf16 3xtf32 \
  >> $OUT/sanitize_${TAG}_racecheck_cg1.txt 2>&1
echo "=== rc=$?" >> $OUT/sanitize_${TAG}_racecheck_cg1.txt
grep -E "RACECHECK SUMMARY|=== rc" $OUT/sanitize_${TAG}_racecheck_cg1.txt
python scripts/sanitize_summary.py $OUT/sanitize_${TAG}_*.txt
OMP_B200_DEBUG_FILL=1 timeout 1200 python -m pytest tests -m gpu -q -x \
  -k "tiny or c2_all or ragged or edge or worked or graph or host_path or strided or adversarial or overflowing" \
  > $OUT/sanitize_${TAG}_debugfill_pytest.txt 2>&1
echo "debug-fill pytest rc=$?"; tail -2 $OUT/sanitize_${TAG}_debugfill_pytest.txt
