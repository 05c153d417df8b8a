#!/bin/bash
OUT=gpurun_out/$1; shift; mkdir -p $OUT
N=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > $OUT/pytest_gpu.log 2>&1; echo "rc $?" >> $OUT/pytest_gpu.log
for P in 1 0; do
  OPTR_PDL=$P CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench1_pdl$P.log 2>&1
  for W in "$@"; do
    OPTR_PDL=$P timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
      bench.py --gpus $N --steps 10 --warmup 3 --workload $W > $OUT/bench_${W}_pdl$P.log 2>&1
  done
done
