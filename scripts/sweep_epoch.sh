#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
[ -n "$NOTEST" ] || { timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/sweep_pytest.log 2>&1; echo "pytest=$?"; tail -1 gpurun_out/sweep_pytest.log; }
for q in ${QS:-128 192 230}; do for k in ${KS:-16 32 48 64}; do
  RASP_STABLE_Q8=$q timeout 300 python bench.py --config ${CFG:-c2} --steps 10 --warmup 3 --epoch $k --no-cpu-baseline > gpurun_out/sweep_${q}_${k}.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/sweep_${q}_${k}.log').read().strip().splitlines()[-1]); print('q8=$q K0=$k', round(d['roofline']['kernel_ms'],4), 'ms', round(d['value']/1e9,1), 'Gsteps/s', 'e2e', round(d['e2e']['ms_per_step'],3))"
done; done
