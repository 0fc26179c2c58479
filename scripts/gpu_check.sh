cd $GRAFT_REPO_ROOT
timeout 300 python -u scripts/embed_wb_ab.py 2>&1 | tail -8
CFG=c4 timeout 300 python -u scripts/embed_wb_ab.py 2>&1 | tail -8
