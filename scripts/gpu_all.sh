#!/bin/bash
# Full GPU session: smoke, every GPU test, every bench config (with CPU
# baselines), and the reference arm of the default config.
#   scripts/gpu_all.sh <tag>
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-all}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/${TAG}_pytest.log
for c in c2 c1 c3 c4 c5 paper paper6; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_$c.log 2>&1
  echo "bench $c=$?"; python scripts/benchsum.py gpurun_out/${TAG}_bench_$c.log
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_ref_c2.log 2>&1; echo "ref=$?"
