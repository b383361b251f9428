for e in "CP_X=0" "CP_STAGE_BYTES=26624" "CP_STAGE_BYTES=13312" "CP_STAGE_BYTES=26624 CP_RING_BYTES=106496" "CP_MMA_MTMAX=2" "CP_L2KEEP_MB=0"; do
  echo "$e :: $(env $e python tools/c3_knobs.py 2>&1 | tail -1)"
done
