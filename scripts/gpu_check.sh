cd $GRAFT_REPO_ROOT
for mode in warm_dev warm_host; do timeout 80 python -u scripts/hang_probe.py $mode 2>&1 | tail -3; done
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/t3_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t3_pytest.log
grep -E "c4 full batch" -r gpurun_out/t3_pytest.log
timeout 600 python -u bench.py --steps 50 --warmup 10 > gpurun_out/bench_c2.log 2>&1; echo "bench c2 rc=$?"; tail -c 400 gpurun_out/bench_c2.log
timeout 300 python -u scripts/serve_probe.py 2>&1 | tail -12
