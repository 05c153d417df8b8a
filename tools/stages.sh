#!/bin/bash
# compare TMA ring depths on the default bench
OUT=gpurun_out/$1; mkdir -p $OUT
for S in 2 3; do
  OPTR_TMA_STAGES=$S timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_s$S.log 2>&1
done
timeout 300 python -m pytest tests -q -m gpu -p no:cacheprovider -x > $OUT/pytest.log 2>&1; echo "rc $?" >> $OUT/pytest.log
