# the TMA ring alone (CP_STREAM_DBG=1: consumers skip the DMMA loop) against stage size and ring depth
export CP_LIB_PATH=$PWD/alt/exp/libcp.so
run() { echo -n "$* :: "; env "$@" NSW=50 python tools/time_sweep.py ${CFG:-c4a} 200 2>&1 | tail -1 | sed 's/.*: \([0-9.]* ms\/sweep; stream kernels [0-9.]* ms avg\).*/\1/'; }
for dbg in 1 0; do
for sb in 53248 36864 26624 20480 16384; do
  run CP_STREAM_DBG=$dbg CP_STAGE_BYTES=$sb CP_RING_BYTES=110592
done; done
run CP_STREAM_DBG=1 CP_STAGE_BYTES=53248 CP_CTAS_PER_SM=1 CP_SMEM_CAP=225280 CP_RING_BYTES=163840
run CP_STREAM_DBG=1 CP_STAGE_BYTES=26624 CP_CTAS_PER_SM=1 CP_SMEM_CAP=225280 CP_RING_BYTES=163840
