cd $GRAFT_REPO_ROOT
for cv in 0 1; do
echo "== CARVEOUT=$cv MX EP8"; COMET_CARVEOUT=$cv timeout 300 python tools/fused_timeline.py --ep 8 --M 8192 --nc0 64 --g0 8 --pairs 0 2>&1 | grep -E "measured|span|CTA lifetime|dispatch" | sed "s/.kernels_ms_max.*//"
echo "== CARVEOUT=$cv MX EP1"; COMET_CARVEOUT=$cv timeout 300 python tools/fused_timeline.py --ep 1 --M 8192 --nc0 64 --g0 8 --pairs 0 2>&1 | grep -E "measured|span|CTA lifetime" | sed "s/.kernels_ms_max.*//"
echo "== CARVEOUT=$cv QW EP8"; COMET_CARVEOUT=$cv timeout 300 python tools/fused_timeline.py --shape QW --ep 8 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|CTA lifetime" | sed "s/.kernels_ms_max.*//"
done
