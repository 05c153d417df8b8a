#!/bin/bash
# pass kernels alone: timings at 2^23 / 2^25 / 2^27, then one ncu --set full of the 2^25 passes
OUT=gpurun_out/$1; mkdir -p $OUT
for D in 23 25 27; do timeout 120 python tools/pass_bench.py --logd $D >> $OUT/pass.log 2>&1; done
for S in 1; do OPTR_TMA_STAGES=$S timeout 120 python tools/pass_bench.py --logd 25 >> $OUT/pass_s$S.log 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tma_pass -s 4 -c 2 -o $OUT/pass25 python tools/pass_bench.py --logd 25 --iters 2 > $OUT/ncu.log 2>&1
echo "ncu rc $?" >> $OUT/ncu.log
