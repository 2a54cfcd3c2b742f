cd $GRAFT_REPO_ROOT
for ks in 0 2 3; do
echo "== KS1=$ks MX EP8"; COMET_KSPLIT1_FORCE=$ks timeout 300 python tools/fused_timeline.py --ep 8 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|EPI|pair end" | sed "s/.kernels_ms_max.*//"
done
echo "== KS1=2 MX EP4"; COMET_KSPLIT1_FORCE=2 timeout 300 python tools/fused_timeline.py --ep 4 --M 8192 --nc0 32 --g0 4 --pairs 0 2>&1 | grep -E "measured|span" | sed "s/.kernels_ms_max.*//"
