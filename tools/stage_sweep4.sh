# TMA ring alone vs the shared-memory column stride (destination alignment of the 2 KB bulk copies)
export CP_LIB_PATH=$PWD/alt/exp/libcp.so
run() { echo -n "$* :: "; env "$@" NSW=50 python tools/time_sweep.py ${CFG:-c4a} 200 2>&1 | tail -1 | sed 's/.*: \([0-9.]* ms\/sweep; stream kernels [0-9.]* ms avg\).*/\1/'; }
for dbg in 1 0; do for pad in 4 8 16 0 12 2; do run CP_STREAM_DBG=$dbg CP_ZCS_PAD=$pad; done; done
