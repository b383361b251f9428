#!/bin/bash
for sb in 24576 32768 40960; do for ring in 98304 112640; do
  for cfg in "c4a 2 0" "c4a 2 1" "c4a 2 2" "c4b 2 0" "c4b 2 1" "c3 2 0"; do
    r=$(CP_STAGE_BYTES=$sb CP_RING_BYTES=$ring python tools/prof_mttkrp.py $cfg 2>&1 | tail -1)
    echo "stage=$sb ring=$ring :: $r"
  done
done; done
