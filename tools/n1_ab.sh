#!/bin/bash
# N=1 scheduling A/B (20 steps): default / batch all workers per launch / one chain / sync buckets
OUT=gpurun_out/$1; mkdir -p $OUT
run() { tag=$1; shift; env "$@" timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_$tag.log 2>&1; }
run default OPTR_X=0
run batch OPTR_BATCH_WORKERS=1
run chains1 OPTR_CHAINS=1
run sync OPTR_BENCH_SYNC=1
run default2 OPTR_X=0
run batch_s3 OPTR_BATCH_WORKERS=1 OPTR_TMA_STAGES_S=3
