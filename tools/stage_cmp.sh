#!/bin/bash
OUT=gpurun_out/$1; shift; mkdir -p $OUT
N=$(python -c "import torch;print(torch.cuda.device_count())")
for S in 1 2; do
  OPTR_TMA_STAGES=$S CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench1_s$S.log 2>&1
  OPTR_TMA_STAGES=$S CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --workers 2 --workload headline > $OUT/bench1h_s$S.log 2>&1
  for W in "$@"; do
   OPTR_TMA_STAGES=$S timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus $N --steps 10 --warmup 3 --workload $W > $OUT/bench_${W}_s$S.log 2>&1
  done
done
OPTR_TMA_STAGES=1 timeout 600 python -m pytest tests -q -m gpu -p no:cacheprovider -x > $OUT/pytest_s1.log 2>&1; echo "rc $?" >> $OUT/pytest_s1.log
