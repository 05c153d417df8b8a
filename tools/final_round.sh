#!/bin/bash
# round-end check: smoke, every GPU test, the default bench (with the CPU baseline), the reference arm, N=all bench
OUT=gpurun_out/$1; mkdir -p $OUT
N=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "rc $?" >> $OUT/smoke.log
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "rc $?" >> $OUT/pytest_gpu.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > $OUT/bench_default.log 2>&1; echo "rc $?" >> $OUT/bench_default.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.log 2>&1; echo "rc $?" >> $OUT/bench_reference.log
if [ "$N" -gt 1 ]; then
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N > $OUT/bench_n$N.log 2>&1; echo "rc $?" >> $OUT/bench_n$N.log
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --impl reference --steps 3 --warmup 3 > $OUT/bench_ref_n$N.log 2>&1; echo "rc $?" >> $OUT/bench_ref_n$N.log
fi
