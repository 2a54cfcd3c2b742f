cd $GRAFT_REPO_ROOT
for dbg in 0 24; do for ch in 4 16 32; do for nc in 16 32; do echo "== debug=$dbg chunk=$ch nc0=$nc"; COMET_DEBUG=$dbg COMET_CHUNK=$ch timeout 300 python tools/fused_timeline.py --nc0 $nc --g0 4 --pairs 0 2>&1 | grep -E "dispatch|span"; done; done; done
