#!/bin/bash
# ring depth per pass kind (contiguous C, strided S) at 2^23 / 2^25 / 2^26
OUT=gpurun_out/$1; mkdir -p $OUT
for D in 23 25 26; do
  for C in 1 2 3; do
    for S in 1 2 3; do
      echo -n "C$C S$S " >> $OUT/stages.log
      OPTR_TMA_STAGES_C=$C OPTR_TMA_STAGES_S=$S timeout 120 python tools/pass_bench.py --logd $D >> $OUT/stages.log 2>&1
    done
  done
done
