mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01_launches_v3.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_v3.log 2>&1
tail -1 gpurun_out/ncu_launch_v3.log | cut -c1-200
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"gemm_tma_kernel.*Lb1ELb1ELi1E" -s 20 -c 1 -o gpurun_out/r01_full_syrk_v3 python tools/quick_time.py 16384 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"gemm_tma_kernel.*Lb1ELb0ELi0E" -s 60 -c 1 -o gpurun_out/r01_full_adjgemm_v3 python tools/quick_time.py 16384 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"gemm_tma_kernel.*Lb0ELb0ELi2E" -s 30 -c 1 -o gpurun_out/r01_full_splitk_v3 python tools/quick_time.py 16384 > /dev/null 2>&1
python tools/cusolver_context.py 4096 16384 > gpurun_out/r01_cusolver_context.jsonl 2>&1
cat gpurun_out/r01_cusolver_context.jsonl
python tools/run_big.py 32768 > gpurun_out/r01_large_n_v2.jsonl 2>&1
python tools/run_big.py 65536 >> gpurun_out/r01_large_n_v2.jsonl 2>&1
cat gpurun_out/r01_large_n_v2.jsonl
ls -la gpurun_out
