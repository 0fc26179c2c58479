cd $GRAFT_REPO_ROOT
OUT=gpurun_out
CFG=c4 SKIP=46 COUNT=23 bash scripts/gpu_profile.sh > $OUT/prof_c4_driver.log 2>&1; tail -3 $OUT/prof_c4_driver.log
ncu -i $OUT/prof_full_c4.ncu-rep --page details --print-kernel-base function -k regex:gemm_bf16_kernel > $OUT/prof_full_c4_details.txt 2>/dev/null; echo details=$?
timeout 2400 python -u bench_saturation.py > $OUT/saturation.log 2>&1; echo "saturation rc=$?"
timeout 1500 python -u bench.py --config c3s --steps 10 --warmup 3 --ring 2 --no-serving > $OUT/bench_c3s_unsharded.log 2>&1; echo "c3s rc=$?"; tail -c 300 $OUT/bench_c3s_unsharded.log
