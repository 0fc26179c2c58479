cd $GRAFT_REPO_ROOT
timeout 600 python -u scripts/step_ab.py '[{}]' 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_serving.py tests/test_gpu_c4.py -q -x -k "not full_batch" 2>&1 | tail -2
CFG=c6 timeout 600 python -u scripts/step_ab.py '[{}]' 2>&1 | tail -2
