#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
N=$(python -c "import torch;print(torch.cuda.device_count())")
for W in headline resnet50; do for P in 1 0 1 0; do
  OPTR_PREP_AFTER_ENC=$P timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 20 --warmup 5 --workload $W --no-cpu-baseline >> $OUT/bench_${W}_p$P.log 2>&1
done; done
