#!/bin/bash
# Time several library builds on the same box:  scripts/ab_multi.sh "<configs>" lib1.so lib2.so ...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
CFGS=$1; shift
mkdir -p gpurun_out
for c in $CFGS; do for lib in "$@"; do
  RASP_LIBRARY=$lib timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/abm.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/abm.log').read().strip().splitlines()[-1]); print('$c', '$lib'.split('/')[-2], round(d['ms_per_step'],4), 'ms')" 2>&1 | tail -1
done; done
