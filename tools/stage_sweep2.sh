# one CTA per SM with a deep ring vs the default two CTAs per SM (experiments build alt/exp/libcp.so)
export CP_LIB_PATH=$PWD/alt/exp/libcp.so
run() { echo -n "$* :: "; env "$@" NSW=50 python tools/time_sweep.py ${CFG:-c4a} 200 2>&1 | tail -1 | sed 's/.*: \([0-9.]* ms\/sweep; stream kernels [0-9.]* ms avg\).*/\1/'; }
run CP_STAGE_BYTES=53248
run CP_STAGE_BYTES=61440 CP_RING_BYTES=126976 CP_SMEM_CAP=131072
for sb in 53248 36864 26624; do
  for rb in 163840 212992; do
    run CP_CTAS_PER_SM=1 CP_SMEM_CAP=225280 CP_RING_BYTES=$rb CP_STAGE_BYTES=$sb
  done
done
run CP_L2KEEP_MB=0
run CP_L2KEEP_MB=24
run CP_L2KEEP_MB=64
