# c4b (96^4, R = 10) MTTKRP stream-plan knob sweep (mode 1): ms/call per setting
run() { echo "$* :: $(env "$@" python tools/prof_mttkrp.py c4b 2 1 2>&1 | tail -1)"; }
run CP_X=0
run CP_STREAM_DBG=1
for mt in 2 3 4 6 8; do run CP_MMA_MTMAX=$mt; done
for sb in 26624 40960 65536; do run CP_STAGE_BYTES=$sb; done
for rb in 65536 131072; do run CP_RING_BYTES=$rb; done
run CP_RING_BYTES=180000 CP_SMEM_CAP=200000 CP_CTAS_PER_SM=1
run CP_RING_BYTES=65536 CP_SMEM_CAP=74000 CP_CTAS_PER_SM=3
run CP_STAGE_BYTES=26624 CP_RING_BYTES=65536 CP_SMEM_CAP=74000 CP_CTAS_PER_SM=3
run CP_MMA_SROWS=0
