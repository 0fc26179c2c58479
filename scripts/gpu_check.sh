set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -q -m gpu -x -k "not full_batch" > gpurun_out/t1_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/t1_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/t1_bench.log 2>&1; echo "bench rc=$?"
tail -c 6000 gpurun_out/t1_bench.log
