cd $GRAFT_REPO_ROOT
for m in dev zc; do MODE=$m NC0=16 timeout 300 python tools/stream_probe.py 2>&1 | tail -9; done
