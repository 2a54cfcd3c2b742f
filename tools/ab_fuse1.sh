#!/bin/bash
# A/B of the EP=1 fused combine (COMET_FUSE1) in alternating bench runs
for i in 1 2 3; do
  for f in 0 1; do
    COMET_FUSE1=$f timeout -s KILL 300 python bench.py --no-cpu-baseline --no-unfused 2>/dev/null | tail -1 > /tmp/ab.json
    python -c "import json; d=json.load(open('/tmp/ab.json')); print('FUSE1=$f', d['value'], d['kernels_ms'], d['clocks']['sm_mhz'])"
  done
done
