#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
N=$(python -c "import torch;print(torch.cuda.device_count())")
for S in 2 3 2 3; do
  OPTR_TMA_STAGES_S=$S timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 20 --warmup 5 --workload resnet50 --no-cpu-baseline >> $OUT/bench_s$S.log 2>&1
done
