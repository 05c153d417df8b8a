#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
N=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 420 python -m pytest tests/test_multigpu.py -q -m gpu -p no:cacheprovider -x > $OUT/pytest_multi.log 2>&1; echo "rc $?" >> $OUT/pytest_multi.log
run() { tag=$1; w=$2; shift; shift; env "$@" timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 20 --warmup 5 --workload $w --no-cpu-baseline > $OUT/bench_${w}_$tag.log 2>&1; }
run ovl resnet50 OPTR_X=0
run serial resnet50 OPTR_FUSED_SERIAL=1
run ovl_s2 resnet50 OPTR_TMA_STAGES_S=2
run ovl headline OPTR_X=0
run serial headline OPTR_FUSED_SERIAL=1
