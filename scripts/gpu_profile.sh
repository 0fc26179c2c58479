#!/bin/bash
# Run on the GPU box (via gpurun): plain bench, then the ncu launch list and one full capture of one dense
# stage's kernels + an embedding launch.  Outputs land in gpurun_out/ (scratch); scripts/ncu_summarize.py
# writes the summaries under profiles/.
set -u
OUT=gpurun_out
mkdir -p $OUT
CFG=${CFG:-c2}
CMD="python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-serving"
timeout 300 $CMD > $OUT/plain_$CFG.log 2>&1
rc=$?
echo "plain_exit=$rc"
if [ $rc -ne 0 ]; then tail -20 $OUT/plain_$CFG.log; exit 1; fi
KRE='regex:embed_bag|gemm_bf16|dense_f32|unpack|mha64|head_finalize|set_call'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" --csv \
  --log-file $OUT/launches_$CFG.csv $CMD > $OUT/ncu_launches_$CFG.log 2>&1
echo "ncu_launches_exit=$?"
# full capture of 12 consecutive hot-path kernels from the middle of the run (one whole step)
timeout 1200 ncu --set full --clock-control none --import-source on -k "$KRE" -s ${SKIP:-60} -c ${COUNT:-12} \
  -o $OUT/prof_full_$CFG $CMD > $OUT/ncu_full_$CFG.log 2>&1
echo "ncu_full_exit=$?"
ncu -i $OUT/prof_full_$CFG.ncu-rep --page raw --csv > $OUT/prof_full_${CFG}_raw.csv 2>/dev/null
echo "raw_exit=$?"
