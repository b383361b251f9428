# Stage-size / ring-depth sweep of the streaming passes on a config (experiments build: alt/exp/libcp.so,
# tools/build_variant.py exp "-DCP_EXPERIMENTS" capi.cu).   CFG=c4a bash tools/stage_sweep.sh
export CP_LIB_PATH=$PWD/alt/exp/libcp.so
for sb in 53248 45056 36864 32768 26624 20480 16384; do
  for rb in 98304 110592; do
    echo -n "stage=$sb ring=$rb :: "
    CP_STAGE_BYTES=$sb CP_RING_BYTES=$rb NSW=50 python tools/time_sweep.py ${CFG:-c4a} 200 2>&1 | tail -1 | sed 's/.*: \([0-9.]* ms\/sweep; stream kernels [0-9.]* ms avg\).*/\1/'
  done
done
