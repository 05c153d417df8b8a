#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 600 python -m pytest tests -q -m gpu -p no:cacheprovider -x > $OUT/pytest.log 2>&1; echo "rc $?" >> $OUT/pytest.log
for B in 0 1; do
  for S in 2 3; do
    OPTR_BATCH_WORKERS=$B OPTR_TMA_STAGES=$S timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_b${B}_s$S.log 2>&1
  done
done
OPTR_BATCH_WORKERS=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x > $OUT/pytest_batch.log 2>&1; echo "rc $?" >> $OUT/pytest_batch.log
