#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > $OUT/pytest.log 2>&1; echo "rc $?" >> $OUT/pytest.log
run() { tag=$1; shift; env "$@" timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_$tag.log 2>&1; }
run cf OPTR_X=0
run sf OPTR_DEC_ORDER=strided
run cf2 OPTR_X=0
env OPTR_X=0 timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --workload headline > $OUT/bench_headline_cf.log 2>&1
env OPTR_DEC_ORDER=strided timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --workload headline > $OUT/bench_headline_sf.log 2>&1
