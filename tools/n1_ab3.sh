#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
run() { tag=$1; shift; env "$@" timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_$tag.log 2>&1; }
run default OPTR_X=0
run contig OPTR_DEC_ORDER=contig
OPTR_X=0 timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --drop 0 > $OUT/bench_nodrop.log 2>&1
