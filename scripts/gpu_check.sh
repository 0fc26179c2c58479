cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_serving.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
timeout 300 python bench_serving.py --duration 3 > gpurun_out/serving_r02.log 2>&1; echo "serving rc=$?"; tail -1 gpurun_out/serving_r02.log | cut -c1-1500
timeout 1500 python bench_saturation.py --duration 1.0 > gpurun_out/saturation_r02.log 2>&1; echo "sat rc=$?"; grep p99_bound gpurun_out/saturation_r02.log | cut -c1-3000
