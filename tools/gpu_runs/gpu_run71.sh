cd $GRAFT_REPO_ROOT
timeout 120 ./tools/copy_bench
