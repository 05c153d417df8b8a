#!/bin/bash
# quick timing on one GPU: the default bench line (pipelined and serialised
# passes), summarised.  Usage: tools/quick.sh TAG [bench args...]
TAG=${1:-q}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 20 --no-cpu-baseline "$@" > $OUT/bench.log 2>&1
python tools/show.py $OUT/bench.log > $OUT/summary.txt 2>&1
cat $OUT/summary.txt
