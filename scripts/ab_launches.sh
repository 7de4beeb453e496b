#!/bin/bash
# Per-launch kernel durations (ncu launch list) of two builds:  scripts/ab_launches.sh <alt .so> <config>
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
ALT=$1; C=${2:-c2}
mkdir -p gpurun_out
for v in cur alt; do
  if [ $v = alt ]; then export RASP_LIBRARY=$ALT; else unset RASP_LIBRARY; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/abl_${v}_${C}.csv \
      python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  python - "$v" "gpurun_out/abl_${v}_${C}.csv" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[2])) if len(r) > 10]
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
ks = [(r[ki][:40], float(r[vi].replace(",", ""))) for r in rows[1:]]
ep = [v for k, v in ks if "epoch_kernel" in k]
n = len(ep) // 2   # warmup + 1 timed step: take the last step's launches
print(sys.argv[1], " ".join(f"{x/1000:.1f}" for x in ep[n:]), "us")
PY
done
