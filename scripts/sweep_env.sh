#!/bin/bash
# Sweep one RASP_* environment knob over configs:  VAR=RASP_PREFETCH VALS="0 1 2" CFGS="c2 c5" scripts/sweep_env.sh
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for c in ${CFGS:-c2}; do for v in ${VALS}; do
  env $VAR=$v timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sw_${c}_${v}.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/sw_${c}_${v}.log').read().strip().splitlines()[-1]); print('$c $VAR=$v', round(d['roofline']['kernel_ms'],4), 'ms')" 2>&1 | tail -1
done; done
