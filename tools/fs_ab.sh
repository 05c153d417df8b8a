#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
N=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 420 python -m pytest tests/test_multigpu.py -q -m gpu -p no:cacheprovider -x -k "multi_gpu or fused" > $OUT/pytest_multi.log 2>&1; echo "rc $?" >> $OUT/pytest_multi.log
for S in 3 2 3 2; do
  OPTR_FUSED_STAGES=$S timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 20 --warmup 5 --workload resnet50 --no-cpu-baseline >> $OUT/bench_s$S.log 2>&1
done
