cd $GRAFT_REPO_ROOT
for ch in 8 16 32; do for nc in 32 64 96; do echo "== chunk=$ch nc0=$nc"; COMET_CHUNK=$ch timeout 300 python tools/fused_timeline.py --nc0 $nc --g0 4 --pairs 0 2>&1 | grep -E "measured|dispatch|span|pair end"; done; done
python tools/idx_timing.py 8 4 2>&1 | tail -4
python tools/idx_timing.py 1 0 2>&1 | tail -4
