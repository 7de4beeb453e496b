#!/bin/bash
# Refill threshold sweep on one box, optionally against an alternate build:
#   scripts/sweep_refill.sh "<mins>" "<configs>" [alt .so] [reps]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
MINS=${1:-"8 12 16"}; CFGS=${2:-c5}; ALT=$3; R=${4:-2}
for r in $(seq $R); do for c in $CFGS; do for m in $MINS; do
  for v in cur ${ALT:+alt}; do
    if [ $v = alt ]; then export RASP_LIBRARY=$ALT; else unset RASP_LIBRARY; fi
    RASP_REFILL_MIN=$m timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$r $c min $m $v', round(d['ms_per_step'], 4))"
  done
done; done; done
