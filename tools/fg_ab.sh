#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
N=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 500 python -m pytest tests/test_multigpu.py -q -m gpu -p no:cacheprovider -x > $OUT/pytest_multi.log 2>&1; echo "rc $?" >> $OUT/pytest_multi.log
for G in 2 1 2 1; do
  OPTR_FUSED_GROUPS=$G timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 20 --warmup 5 --workload resnet50 --no-cpu-baseline >> $OUT/bench_g$G.log 2>&1
done
