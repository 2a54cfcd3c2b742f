cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_layer.py -m gpu -q -x -k "zerocopy and 129" 2>&1 | grep -E "^E |Error|error" | head -20
for v in "COMET_ZC_ILV=0" "COMET_ZC_DL=0" "COMET_ZC_DEDUP=0" "COMET_ZC_ILV=0 COMET_ZC_DL=0"; do echo "== $v"; env $v timeout 300 python -m pytest tests/test_gpu_layer.py -m gpu -q -x -k "zerocopy and 129" 2>&1 | tail -1; done
