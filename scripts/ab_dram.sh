#!/bin/bash
# DRAM / L2 traffic and time of the c4 update kernel (iteration 64) for library variants, plus the
# bench's own per-launch update time for each (run under gpurun):
#   bash scripts/ab_dram.sh TAG lib1 lib2 ...   (paths relative to paper_2407_06434_b200/)
set -u
TAG=$1; shift
OUT=gpurun_out
mkdir -p $OUT
for lib in "$@"; do
  L=$PWD/paper_2407_06434_b200/$lib
  OMP_B200_LIB=$L timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:k_update -s 64 -c 1 --csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ab_${TAG}_${lib}.ncu.csv 2> $OUT/ab_${TAG}_${lib}.ncu.err
  OMP_B200_LIB=$L timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ab_${TAG}_${lib}.json 2> $OUT/ab_${TAG}_${lib}.err
  python - "$OUT/ab_${TAG}_${lib}.ncu.csv" "$OUT/ab_${TAG}_${lib}.json" "$lib" <<'EOF'
import csv, json, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
m = {}
for r in rows[1:]:
    m[r[-3]] = r[-1]
try:
    b = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    upd = b["kernels"]["update"]["ms_total"] / b["kernels"]["update"]["launches"]
    val = b["value"]
except Exception as e:
    upd, val = None, None
print(sys.argv[3], {k: m.get(k) for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum")},
      "bench update ms/launch", upd, "signals/s", val)
EOF
done
