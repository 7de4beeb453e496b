#!/bin/bash
# Plain run, launch list and one full ncu capture of kernels matching a regex.
#   scripts/ncu_kernel.sh <tag> <config> <kernel-regex> [count] [extra bench args]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=$1; CFG=$2; KRE=$3; CNT=${4:-1}; shift 4; EXTRA="$@"
mkdir -p gpurun_out
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-graph $EXTRA"
RASP_DEBUG=1 timeout 600 $CMD > gpurun_out/${TAG}_plain.log 2>&1; echo "plain=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu1.log 2>&1
echo "ncu-launches=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 0 -c $CNT \
    -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu2.log 2>&1
echo "ncu-full=$?"
