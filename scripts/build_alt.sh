#!/bin/bash
# /tmp/buildalt.sh <name> <extra nvcc flags...>
cd "$(dirname "$0")/.."
NAME=$1; shift
mkdir -p build/$NAME
pids=()
for f in paper_2604_12902_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude "$@" -c -o build/$NAME/$b.o $f &
  pids+=($!)
done
for p in ${pids[@]}; do wait $p || exit 1; done
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o build/$NAME/libraspvisor_b200.so build/$NAME/*.o -ldl
