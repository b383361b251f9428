# ncu launch list of a c1 multigrid solve (5 setup cycles + 3 solve cycles, plain launches)
mkdir -p gpurun_out
CYC=8 CP_MG_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mg_c1_launches.csv python tools/mg_one_cycle.py c1 > gpurun_out/mg_c1_ncu.log 2>&1
tail -2 gpurun_out/mg_c1_ncu.log
