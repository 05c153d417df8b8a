#!/bin/bash
# launch list + full ncu capture of one bench step (single GPU), after a plain run
TAG=${1:-p}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline $*"
timeout 300 $CMD > $OUT/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"tma|prep|aggregate" -s 24 -c 12 -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1
echo done
