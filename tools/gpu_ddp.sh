#!/bin/bash
# DDP training-step benchmark at N GPUs (run under gpurun --gpus N).
TAG=${1:-d}; OUT=gpurun_out/$TAG; mkdir -p $OUT
N=$(python -c "import torch;print(torch.cuda.device_count())")
for M in resnet50 gpt2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29561 \
    tools/ddp_bench.py --model $M --steps 20 > $OUT/ddp_${M}_n$N.log 2>&1; echo "rc $?" >> $OUT/ddp_${M}_n$N.log
done
