#!/bin/bash
# run-to-run variance: the same N=all bench three times per workload
OUT=gpurun_out/$1; mkdir -p $OUT; shift
N=$(python -c "import torch;print(torch.cuda.device_count())")
for W in "$@"; do for i in 1 2 3; do
  timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus $N --steps 20 --warmup 5 --workload $W --no-cpu-baseline > $OUT/bench_${W}_$i.log 2>&1
done; done
