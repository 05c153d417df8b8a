#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x -k "tar or fp64 or lossless or datagram or sim" > $OUT/pytest.log 2>&1; echo "rc $?" >> $OUT/pytest.log
OPTR_AGG_STAGES=4 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x -k "tar or fp64 or lossless or datagram or sim" > $OUT/pytest4.log 2>&1; echo "rc $?" >> $OUT/pytest4.log
for A in 4 2 4 2; do OPTR_AGG_STAGES=$A timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_a$A.log 2>&1; done
