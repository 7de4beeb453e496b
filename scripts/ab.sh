#!/bin/bash
# A/B timing of two builds of the library on the same box:
#   scripts/ab.sh <alt .so> "<configs>" [rounds]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
ALT=$1; CFGS=${2:-c2}; R=${3:-2}
mkdir -p gpurun_out
for r in $(seq $R); do for c in $CFGS; do
  for v in cur alt; do
    if [ $v = alt ]; then export RASP_LIBRARY=$ALT; else unset RASP_LIBRARY; fi
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${v}_${c}.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/ab_${v}_${c}.log').read().strip().splitlines()[-1]); print('$r $c $v', round(d['roofline']['kernel_ms'],4), 'ms')" 2>&1 | tail -1
  done
done; done
