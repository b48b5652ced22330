ncu --set full --clock-control none --import-source on -k regex:gemm_tma_kernel -s 4 -c 4 -o gpurun_out/prof_tma ./tools/gemm_bench > gpurun_out/ncu_tma.log 2>&1
tail -1 gpurun_out/ncu_tma.log
