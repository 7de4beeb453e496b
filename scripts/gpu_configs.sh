#!/bin/bash
# Tests + bench over every config on one GPU.  scripts/gpu_configs.sh <tag>
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-cfg}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest=$?"; tail -3 gpurun_out/${TAG}_pytest.log
for c in ${CFGS:-c2 c1 c5 paper c4 c3}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 > gpurun_out/${TAG}_bench_$c.log 2>&1; echo "bench $c=$?"
done
