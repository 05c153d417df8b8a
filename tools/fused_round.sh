#!/bin/bash
# multi-GPU tests (fused kernel) then N=all benches with fused on / off
OUT=gpurun_out/$1; mkdir -p $OUT
N=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 420 python -m pytest tests/test_multigpu.py -q -m gpu -p no:cacheprovider -x > $OUT/pytest_multi.log 2>&1; echo "rc $?" >> $OUT/pytest_multi.log
for W in headline resnet50; do
  for F in 1 0; do
    OPTR_FUSED=$F timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
      bench.py --gpus $N --steps 10 --warmup 3 --workload $W --no-cpu-baseline > $OUT/bench_${W}_f$F.log 2>&1
  done
done
