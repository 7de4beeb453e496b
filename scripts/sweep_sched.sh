#!/bin/bash
# Schedule sweep: stability threshold (RASP_STABLE_Q8) x first epoch, per config.
#   CFGS="paper6 c2" QS="128 230" KS="32 64" scripts/sweep_sched.sh
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for c in ${CFGS:-c2}; do for q in ${QS:-128}; do for k in ${KS:-64}; do
  RASP_STABLE_Q8=$q timeout 600 python bench.py --config $c --steps ${STEPS:-3} --warmup 3 --epoch $k --no-cpu-baseline > gpurun_out/ss.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ss.log').read().strip().splitlines()[-1]); print('$c q8=$q K0=$k', round(d['ms_per_step'],4), 'ms')" 2>&1 | tail -1
done; done; done
