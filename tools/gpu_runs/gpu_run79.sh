cd $GRAFT_REPO_ROOT
timeout 900 python tools/fit_costmodel.py 2>&1 | tail -14
