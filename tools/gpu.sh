#!/bin/bash
# One parametrised GPU session (run under gpurun).  Usage:
#   tools/gpu.sh TAG STEP[,STEP...] [bench args...]
# steps: build, test (pytest -m gpu), smoke, bench (default line, with the CPU
# baseline), ref (reference arm), launches (ncu launch list of one step),
# full (ncu --set full of the dominant kernels), multi (bench at N = all GPUs
# + reference arm), sanitize (compute-sanitizer memcheck/racecheck/synccheck
# of one small bucket).  Outputs land in gpurun_out/TAG/.
TAG=${1:-r}; STEPS=${2:-build,test,smoke,bench}; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
N=$(python -c "import torch;print(torch.cuda.device_count())" 2>/dev/null || echo 1)
has() { [[ ",$STEPS," == *",$1,"* ]]; }
CMD1="python bench.py --steps 1 --warmup 3 --no-cpu-baseline $*"
has build && { python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1; echo "rc $?" >> $OUT/build.log; }
has test && { timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > $OUT/pytest_gpu.log 2>&1; echo "rc $?" >> $OUT/pytest_gpu.log; }
has smoke && { timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc $?" >> $OUT/smoke.log; }
has bench && { CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py "$@" > $OUT/bench.log 2>&1; echo "rc $?" >> $OUT/bench.log; }
has ref && { CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --impl reference --steps 3 --warmup 3 "$@" > $OUT/bench_ref.log 2>&1; echo "rc $?" >> $OUT/bench_ref.log; }
has launches && { CUDA_VISIBLE_DEVICES=0 timeout 600 $CMD1 > $OUT/plain.log 2>&1 && \
  CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $OUT/launches.csv $CMD1 > $OUT/ncu_launch.log 2>&1; echo "rc $?" >> $OUT/ncu_launch.log; }
has full && { CUDA_VISIBLE_DEVICES=0 timeout 1200 ncu --set full --import-source on --clock-control none \
    -k regex:"tma|prep|aggregate" -s 20 -c 10 -o $OUT/prof $CMD1 > $OUT/ncu_full.log 2>&1; echo "rc $?" >> $OUT/ncu_full.log; }
has sanitize && for tool in memcheck racecheck synccheck; do
  CUDA_VISIBLE_DEVICES=0 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 \
    python tools/sanitize_case.py > $OUT/sanitize_$tool.log 2>&1; echo "rc $?" >> $OUT/sanitize_$tool.log; done
if has multi && [ "$N" -gt 1 ]; then
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus $N "$@" > $OUT/bench_n$N.log 2>&1; echo "rc $?" >> $OUT/bench_n$N.log
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29534 bench.py --gpus $N --impl reference --steps 3 --warmup 3 "$@" > $OUT/bench_ref_n$N.log 2>&1
  echo "rc $?" >> $OUT/bench_ref_n$N.log
fi
echo done
