#!/bin/bash
# Build experiment variants of the C ABI library with parts of the trainer's
# critical warp compiled out (KAPSM_FEAT bits, instrumentation kernel only).
# Usage: tools/exp_build.sh FEAT [FEAT ...]  -> /root/repo/gpurun_exp/libexp_<FEAT>.so
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
OUT=$R/gpurun_exp; mkdir -p $OUT/obj
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -I $R/include"
for s in gram detect screen pipeline; do
  [ -f $OUT/obj/$s.o ] || nvcc $F -c $R/paper_2201_05024_b200/csrc/$s.cu -o $OUT/obj/$s.o &
done
wait
for feat in "$@"; do
  nvcc $F -DKAPSM_EXP_ONLY -DKAPSM_FEAT=$feat -c $R/paper_2201_05024_b200/csrc/train.cu -o $OUT/obj/train_$feat.o &
done
wait
for feat in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libexp_$feat.so $OUT/obj/train_$feat.o $OUT/obj/gram.o $OUT/obj/detect.o $OUT/obj/screen.o $OUT/obj/pipeline.o -lcudart
done
ls $OUT
