#!/bin/bash
# First-epoch length sweep, refill kernel on and off:  scripts/sweep_k0.sh <config> "<epochs>" [reps]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
C=$1; EPS=$2; R=${3:-1}
for r in $(seq $R); do for k in $EPS; do for v in 1 0; do
  RASP_REFILL=$v timeout 600 python bench.py --config $C --epoch $k --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$r $C epoch $k refill $v', round(d['ms_per_step'], 4))"
done; done; done
