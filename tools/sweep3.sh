#!/bin/bash
for V in 8 4; do for sb in 16384 32768 65536; do
  for cfg in "c4a 2 0" "c4a 2 1" "c4b 2 0"; do
    r=$(CP_MAX_V=$V CP_STAGE_BYTES=$sb python tools/prof_mttkrp.py $cfg 2>&1 | tail -1)
    echo "V=$V stage=$sb :: $r"
  done
done; done
