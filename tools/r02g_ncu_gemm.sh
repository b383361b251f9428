mkdir -p gpurun_out
python tools/prof_modeprod.py c3 20 > gpurun_out/modeprod_c3.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_dmma_pipe -c 2 -o gpurun_out/r02g_gemm_c3 python tools/prof_modeprod.py c3 1 > gpurun_out/ncu_gemm.log 2>&1
cat gpurun_out/modeprod_c3.txt; tail -3 gpurun_out/ncu_gemm.log
