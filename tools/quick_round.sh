#!/bin/bash
# GPU tests + default bench + headline at N=1 (and N=all when >1 GPU)
OUT=gpurun_out/$1; mkdir -p $OUT
N=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > $OUT/pytest.log 2>&1; echo "rc $?" >> $OUT/pytest.log
for W in resnet50 headline; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --workload $W > $OUT/bench_${W}_n1.log 2>&1
  if [ "$N" -gt 1 ]; then
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
      bench.py --gpus $N --steps 10 --warmup 3 --workload $W > $OUT/bench_${W}_n$N.log 2>&1
  fi
done
