#!/bin/bash
# usage: scripts/ncu_one.sh <kernel-regex> <skip> <count> <outname>   (run on the GPU box)
set -u
OUT=gpurun_out
mkdir -p $OUT
CMD="python bench.py --config ${CFG:-c2} --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > $OUT/plain_$4.log 2>&1 || { echo "plain run failed"; tail -20 $OUT/plain_$4.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$1" -s $2 -c $3 -o $OUT/$4 $CMD > $OUT/ncu_$4.log 2>&1
echo "ncu_exit=$?"
tail -3 $OUT/ncu_$4.log
