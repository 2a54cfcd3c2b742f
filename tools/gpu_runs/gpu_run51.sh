cd $GRAFT_REPO_ROOT
timeout 300 python tools/fused_timeline.py --ep 8 --M 8192 --nc0 64 --g0 8 --pairs 3 2>&1 | tail -40
