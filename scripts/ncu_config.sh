#!/bin/bash
# ncu launch list + full profile of the epoch kernels for one config.  scripts/ncu_config.sh <tag> <config> [count]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=$1; CFG=$2; CNT=${3:-6}
mkdir -p gpurun_out
timeout 600 python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu1.log 2>&1
echo "ncu-launches=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'epoch_kernel|enum_kernel' -s 0 -c $CNT \
    -o gpurun_out/${TAG}_prof python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu2.log 2>&1
echo "ncu-full=$?"
