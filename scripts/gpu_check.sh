cd $GRAFT_REPO_ROOT
OUT=gpurun_out
timeout 300 python -u bench_serving.py --duration 3 > $OUT/serving.log 2>&1; echo "serving rc=$?"; tail -1 $OUT/serving.log | cut -c1-1200
timeout 2400 python -u bench_saturation.py > $OUT/saturation.log 2>&1; echo "saturation rc=$?"
grep p99_bound $OUT/saturation.log | cut -c1-1500
