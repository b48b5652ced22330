./tools/gemm_bench
ncu --set full --clock-control none --import-source on -k regex:gemm_ws_kernel -s 4 -c 2 -o gpurun_out/prof_ws2 ./tools/gemm_bench > gpurun_out/ncu_ws2.log 2>&1
tail -1 gpurun_out/ncu_ws2.log
