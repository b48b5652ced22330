ncu --set full --clock-control none --import-source on -k regex:gemm_ws_kernel -s 17 -c 2 -o gpurun_out/prof_ws ./tools/gemm_bench > gpurun_out/ncu_ws.log 2>&1
tail -3 gpurun_out/ncu_ws.log
