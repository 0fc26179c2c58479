cd $GRAFT_REPO_ROOT
timeout 300 python -u scripts/serve_probe.py 2>&1 | tail -8
