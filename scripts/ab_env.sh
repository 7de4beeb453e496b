#!/bin/bash
# A/B of one RASP_* knob in the same build, interleaved:  VAR=RASP_PDL VALS="1 0" CFGS="c2 c5" R=2 scripts/ab_env.sh
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for r in $(seq ${R:-2}); do for c in ${CFGS:-c2}; do for v in ${VALS}; do
  env $VAR=$v timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/abe_${c}_${v}.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/abe_${c}_${v}.log').read().strip().splitlines()[-1]); print('$r $c $VAR=$v step', round(d['ms_per_step'],4), 'kernel', round(d['roofline']['kernel_ms'],4), 'e2e', round(d['e2e']['ms_per_step'],3), 'ms')" 2>&1 | tail -1
done; done; done
