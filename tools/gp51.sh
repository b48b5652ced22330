mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:"potrf" -c 4 -o gpurun_out/potrf_variants ./tools/potrf_bench > gpurun_out/potrf_ncu.log 2>&1
tail -3 gpurun_out/potrf_ncu.log
