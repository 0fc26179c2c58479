cd $GRAFT_REPO_ROOT
NCCL_DEBUG=WARN timeout 120 python scripts/nccl_probe.py 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_sharded.py -q -x 2>&1 | tail -5
