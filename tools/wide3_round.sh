#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x -k "three_pass or involution or fwht_matches" > $OUT/pytest.log 2>&1; echo "rc $?" >> $OUT/pytest.log
for W in 1 0; do for D in 26 27 28; do OPTR_WIDE3=$W timeout 120 python tools/pass_bench.py --logd $D >> $OUT/pass_w$W.log 2>&1; done; done
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/sweep.py --workers 4 > $OUT/sweep_1gpu.jsonl 2> $OUT/sweep_1gpu.err
