cd $GRAFT_REPO_ROOT
for i in 1 2; do for ks in 0 8; do
echo -n "KS1=$ks MX EP8: "; COMET_KSPLIT1_FORCE=$ks timeout 300 python tools/fused_timeline.py --ep 8 --M 8192 --nc0 64 --g0 8 --pairs 0 2>&1 | grep -E "measured|EPI L1 " | sed "s/.kernels_ms_hot_rank.*//" | tr '\n' ' '; echo
done; done
