#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
run() { tag=$1; shift; env "$@" timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_$tag.log 2>&1; }
run default OPTR_X=0
run wide OPTR_WIDE=1
run s3 OPTR_TMA_STAGES_S=3
run wide_s2 OPTR_WIDE=1 OPTR_TMA_STAGES_S=2
run c3 OPTR_TMA_STAGES_C=3
