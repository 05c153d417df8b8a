#!/bin/bash
# quick A/B timing on one GPU: the default bench line with buckets overlapped
# and serialised (OPTR_BENCH_SYNC=1: per-kernel CUDA-event times are then
# isolated), summarised.  Usage: tools/quick.sh TAG [bench args...]
TAG=${1:-q}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 20 --no-cpu-baseline "$@" > $OUT/ovl.log 2>&1
CUDA_VISIBLE_DEVICES=0 OPTR_BENCH_SYNC=1 timeout 600 python bench.py --steps 20 --no-cpu-baseline "$@" > $OUT/sync.log 2>&1
python tools/show.py $OUT/ovl.log $OUT/sync.log > $OUT/summary.txt 2>&1
cat $OUT/summary.txt
