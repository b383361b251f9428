#!/bin/bash
for V in 4 2; do for ring in 98304 163840 196608; do for ctas in 1 2; do
  for cfg in "c4a 2 0" "c4a 2 1" "c4b 2 0"; do
    r=$(CP_MAX_V=$V CP_RING_BYTES=$ring CP_CTAS_PER_SM=$ctas python tools/prof_mttkrp.py $cfg 2>&1 | tail -1)
    echo "V=$V ring=$ring ctas=$ctas :: $r"
  done
done; done; done
