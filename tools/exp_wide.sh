#!/bin/bash
# Build timing-experiment variants of the general trainer (KAPSM_WIDE_EXP bits)
# -> gpurun_exp/libwide_<EXP>.so ; use with KAPSM_LIB_PATH.
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
OUT=$R/gpurun_exp; mkdir -p $OUT/obj
C=$R/paper_2201_05024_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -I $R/include -I $C"
for s in gram train detect screen pipeline; do
  [ -f $OUT/obj/w_$s.o ] || nvcc $F -c $C/$s.cu -o $OUT/obj/w_$s.o &
done
for e in "$@"; do nvcc $F -DKAPSM_WIDE_EXP=$e -c $C/train_wide.cu -o $OUT/obj/wide_$e.o & done
wait
for e in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libwide_$e.so $OUT/obj/wide_$e.o $OUT/obj/w_gram.o $OUT/obj/w_train.o $OUT/obj/w_detect.o $OUT/obj/w_screen.o $OUT/obj/w_pipeline.o -lcudart
done
ls $OUT/libwide_*
