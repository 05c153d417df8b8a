#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, then ncu (launch list + full set on
# the FWHT/aggregate kernels).  Usage: tools/gpu_round.sh TAG [bench args...]
TAG=${1:-r}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc $?" >> $OUT/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 "$@" > $OUT/bench.log 2>&1; echo "bench rc $?" >> $OUT/bench.log
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline $*"
timeout 600 $CMD > $OUT/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"tma|rtile|aggregate|prep" -s 24 -c 8 -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1
echo done
