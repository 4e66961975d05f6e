#!/bin/bash
# Build the C ABI library with train.cu taken from git revision REV, for A/B
# timing on the same GPU box (KAPSM_LIB_PATH=gpurun_exp/libab_<NAME>.so).
# Usage: tools/ab_build.sh REV NAME
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
OUT=$R/gpurun_exp; mkdir -p $OUT/obj
C=$R/paper_2201_05024_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -I $R/include -I $C"
for s in gram detect screen pipeline; do
  [ -f $OUT/obj/$s.o ] || nvcc $F -c $C/$s.cu -o $OUT/obj/$s.o &
done
wait
if [ "$1" = "WORK" ]; then cp $C/train.cu $OUT/obj/train_ab_$2.cu; else git -C $R show $1:paper_2201_05024_b200/csrc/train.cu > $OUT/obj/train_ab_$2.cu; fi
nvcc $F -c $OUT/obj/train_ab_$2.cu -o $OUT/obj/train_ab_$2.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libab_$2.so $OUT/obj/train_ab_$2.o $OUT/obj/gram.o $OUT/obj/detect.o $OUT/obj/screen.o $OUT/obj/pipeline.o -lcudart
echo $OUT/libab_$2.so
