#!/bin/bash
# GPU tests, then the default bench with / without the persistent chain kernel
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x -k "chain" > $OUT/pytest_chain.log 2>&1; echo "rc $?" >> $OUT/pytest_chain.log
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > $OUT/pytest.log 2>&1; echo "rc $?" >> $OUT/pytest.log
for W in resnet50 headline; do
  for C in 1 0; do
    OPTR_CHAIN=$C timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --workload $W > $OUT/bench_${W}_chain$C.log 2>&1
  done
done
