cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_layer.py -x -q -k "streamed or forward_host" 2>&1 | tail -3
for nc in 8 16 24 32; do echo "== NC0=$nc"; NC0=$nc timeout 300 python tools/stream_probe.py 2>&1 | tail -8; done
