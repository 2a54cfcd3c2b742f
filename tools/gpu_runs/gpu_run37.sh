cd $GRAFT_REPO_ROOT
for fo in 1 0; do echo "== FOLD_ORDER=$fo"; COMET_FOLD_ORDER=$fo MODE=zc NC0=16 timeout 300 python tools/stream_probe.py 2>&1 | tail -8; done
echo "== G0=4"; MODE=zc NC0=16 G0=4 timeout 300 python tools/stream_probe.py 2>&1 | tail -8
echo "== G0=16"; MODE=zc NC0=16 G0=16 timeout 300 python tools/stream_probe.py 2>&1 | tail -8
