cd $GRAFT_REPO_ROOT
timeout 120 python tools/idx_timing.py 8 4 2>&1 | tail -5
timeout 120 python tools/idx_timing.py 1 0 2>&1 | tail -3
