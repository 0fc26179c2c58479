cd $GRAFT_REPO_ROOT
timeout 600 python -u scripts/step_ab.py '[{}, {"u_bn": 64}, {"xv_bn": 128}, {"prefetch_b": 0}]' 2>&1 | tail -12
