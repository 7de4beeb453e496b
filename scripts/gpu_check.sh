#!/bin/bash
# One GPU session: GPU tests, then quick bench lines for a list of configs.
#   scripts/gpu_check.sh <tag> "<pytest args>" "<configs>"
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-run}; PYARGS=${2:-"tests -m gpu -x -q"}; CFGS=${3:-"c2 c5"}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
if [ "$PYARGS" != "none" ]; then
  timeout 1500 python -m pytest $PYARGS > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest=$?"; tail -5 gpurun_out/${TAG}_pytest.log
fi
for c in $CFGS; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.log 2>&1
  echo "bench $c=$?"; python scripts/benchsum.py gpurun_out/${TAG}_bench_$c.log 2>/dev/null || tail -3 gpurun_out/${TAG}_bench_$c.log
done
