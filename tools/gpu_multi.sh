#!/bin/bash
# multi-GPU round: parity test, then bench at N = all visible GPUs
TAG=${1:-m}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
N=$(python -c "import torch;print(torch.cuda.device_count())")
nvidia-smi topo -m > $OUT/topo.txt 2>&1
timeout 600 python -m pytest tests/test_multigpu.py -q -m gpu -p no:cacheprovider > $OUT/pytest_multi.log 2>&1; echo "rc $?" >> $OUT/pytest_multi.log
for W in "$@"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus $N --steps 10 --warmup 3 --workload $W > $OUT/bench_${W}_n$N.log 2>&1
  echo "rc $?" >> $OUT/bench_${W}_n$N.log
done
echo done
