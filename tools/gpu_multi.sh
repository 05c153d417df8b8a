#!/bin/bash
# Multi-GPU session (run under gpurun --gpus N): interconnect probe, the
# multi-rank tests at one rank per GPU, the fused-protocol stress test at
# OPTR_TEST_STRESS reps, and the bench at N (default + headline + reference
# arm).  Usage: tools/gpu_multi.sh TAG [stress reps]
TAG=${1:-m}; REPS=${2:-2000}
OUT=gpurun_out/$TAG; mkdir -p $OUT
N=$(python -c "import torch;print(torch.cuda.device_count())")
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python tools/nvlink_probe.py > $OUT/nvlink_probe.jsonl 2>&1
timeout 1800 python -m pytest tests/test_multigpu.py -q -m gpu -p no:cacheprovider > $OUT/pytest_multi.log 2>&1; echo "rc $?" >> $OUT/pytest_multi.log
OPTR_TEST_STRESS=$REPS timeout 1800 python -m pytest tests/test_multigpu.py -q -m gpu -p no:cacheprovider -k stress > $OUT/stress.log 2>&1; echo "rc $?" >> $OUT/stress.log
for W in resnet50 headline; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus $N --steps 20 --workload $W > $OUT/bench_${W}_n$N.log 2>&1; echo "rc $?" >> $OUT/bench_${W}_n$N.log
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --gpus $N --impl reference --steps 3 --warmup 3 > $OUT/bench_ref_n$N.log 2>&1; echo "rc $?" >> $OUT/bench_ref_n$N.log
echo done
