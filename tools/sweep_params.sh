#!/bin/bash
# parameter sweep of the stream kernel launch plan (env overrides read by capi.cu)
for cfg in "c4a 2 0" "c4a 2 2" "c4b 2 0" "c4b 2 1"; do
  for sb in 16384 32768 65536; do
    for rb in 98304 163840; do
      for ctas in 1 2; do
        r=$(CP_MTTKRP_W0=512 CP_STAGE_BYTES=$sb CP_RING_BYTES=$rb CP_CTAS_PER_SM=$ctas python tools/prof_mttkrp.py $cfg 2>&1 | tail -1)
        echo "stage=$sb ring=$rb ctas=$ctas :: $r"
      done
    done
  done
done
