cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/t4_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t4_pytest.log
timeout 600 python -u bench.py --steps 50 --warmup 10 > gpurun_out/bench_c2.log 2>&1; echo "bench c2 rc=$?"; tail -c 300 gpurun_out/bench_c2.log
timeout 300 python -u bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2_driverargs.log 2>&1; echo "bench c2 (driver args) rc=$?"
