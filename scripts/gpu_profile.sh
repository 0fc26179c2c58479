#!/bin/bash
# Run on the GPU box (via gpurun): plain bench, then the ncu launch list and one full capture of
# the top kernels.  Outputs land in gpurun_out/ (scratch); summaries are copied to profiles/.
set -u
OUT=gpurun_out
mkdir -p $OUT
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > $OUT/plain.log 2>&1
rc=$?
echo "plain_exit=$rc"
if [ $rc -ne 0 ]; then tail -20 $OUT/plain.log; exit 1; fi
KRE='regex:embed_bag|gemm_bf16|dense_f32|unpack'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" --csv \
  --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
echo "ncu_launches_exit=$?"
# full capture: the 2nd gemm launch of the first timed step (tU cross) and the embed kernel
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 28 -c 9 \
  -o $OUT/prof_gemm $CMD > $OUT/ncu_full_gemm.log 2>&1
echo "ncu_full_gemm_exit=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:embed_bag -s 3 -c 1 \
  -o $OUT/prof_embed $CMD > $OUT/ncu_full_embed.log 2>&1
echo "ncu_full_embed_exit=$?"
