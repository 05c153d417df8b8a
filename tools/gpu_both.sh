#!/bin/bash
# all GPU tests, single-GPU bench (both decode orders), multi-GPU benches
TAG=${1:-b}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
N=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "rc $?" >> $OUT/pytest_gpu.log
for O in contig strided; do
  CUDA_VISIBLE_DEVICES=0 OPTR_DEC_ORDER=$O timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench1_$O.log 2>&1
done
for W in "$@"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus $N --steps 10 --warmup 3 --workload $W > $OUT/bench_${W}_n$N.log 2>&1
  echo "rc $?" >> $OUT/bench_${W}_n$N.log
done
echo done
