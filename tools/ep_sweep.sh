#!/bin/bash
# emulated EP=W layer timings over comm-CTA counts / layer0 grouping
for W in ${WS:-8}; do for nc in ${NCS:-2 4 6 8 10}; do for g in ${GS:-1 4}; do
  echo -n "nc0=$nc g0=$g: "; NC0=$nc G0=$g timeout -s KILL 120 python tools/ep_emulate.py $W 2>&1 | tail -1
done; done; done
