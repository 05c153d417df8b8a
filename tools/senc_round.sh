#!/bin/bash
# strided-first encode (fused path order) on one GPU: parity, timings, ncu of the strided pass
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x -k "strided_first" > $OUT/pytest.log 2>&1; echo "rc $?" >> $OUT/pytest.log
for O in contig strided; do OPTR_ENC_ORDER=$O timeout 120 python tools/pass_bench.py --logd 25 >> $OUT/pass.log 2>&1; done
OPTR_ENC_ORDER=strided timeout 120 python tools/pass_bench.py --logd 25 --iters 2 > $OUT/plain.log 2>&1 && \
OPTR_ENC_ORDER=strided timeout 600 ncu --set full --import-source on --clock-control none -k regex:tma_pass -s 2 -c 2 -o $OUT/senc python tools/pass_bench.py --logd 25 --iters 2 > $OUT/ncu.log 2>&1
echo "ncu rc $?" >> $OUT/ncu.log
