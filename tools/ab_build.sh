#!/bin/bash
# Build the C ABI library from git revision REV's sources (or WORK = the
# working tree), for A/B timing on one GPU box:
#   KAPSM_LIB_PATH=gpurun_exp/libab_<NAME>.so
# Usage: tools/ab_build.sh REV NAME
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
OUT=$R/gpurun_exp; mkdir -p $OUT
T=$(mktemp -d)
if [ "$1" = "WORK" ]; then
  mkdir -p $T/paper_2201_05024_b200 && cp -r $R/paper_2201_05024_b200/csrc $T/paper_2201_05024_b200/ && cp -r $R/include $T/
else
  git -C $R archive $1 paper_2201_05024_b200/csrc include | tar -x -C $T
fi
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -I $T/include"
objs=""
for f in $T/paper_2201_05024_b200/csrc/*.cu; do
  nvcc $F -c $f -o ${f%.cu}.o & objs="$objs ${f%.cu}.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libab_$2.so $objs -lcudart
rm -rf $T
echo $OUT/libab_$2.so
