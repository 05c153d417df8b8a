#!/bin/bash
OUT=gpurun_out/$1; shift; mkdir -p $OUT
N=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 600 python -m pytest tests/test_multigpu.py -q -m gpu -p no:cacheprovider > $OUT/pytest_multi.log 2>&1; echo "rc $?" >> $OUT/pytest_multi.log
for S2 in push pull; do
 for O in contig strided; do
  for W in "$@"; do
   OPTR_STAGE2=$S2 OPTR_DEC_ORDER=$O timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus $N --steps 10 --warmup 3 --workload $W > $OUT/bench_${W}_${S2}_${O}.log 2>&1
  done
 done
done
