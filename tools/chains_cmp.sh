#!/bin/bash
# A/B: concurrent helper chains x async buckets at N=1 (default workload + headline)
OUT=gpurun_out/$1; mkdir -p $OUT
for W in resnet50 headline; do
  for C in 1 2; do
    for S in 0 1; do
      OPTR_CHAINS=$C OPTR_BENCH_SYNC=$S timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --workload $W > $OUT/bench_${W}_c${C}_s$S.log 2>&1
    done
  done
done
