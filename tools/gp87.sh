# Profiles v5 (code after fused diagonal step, symmetric SE builder, pipelined POTRF, PDL)
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/r01_bench_v8.json
python -c "import json; d=json.load(open('gpurun_out/r01_bench_v8.json')); print(d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['gpu_launches'], d['clocks'])"
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01_launches_v5.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_v5.log 2>&1
tail -1 gpurun_out/ncu_launch_v5.log | cut -c1-100
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"gemm_tma_kernel.*Lb1ELb0ELi0E" -s 60 -c 1 -o gpurun_out/r01_full_adjgemm_v5 python tools/quick_time.py 16384 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"potrf_tile_kernel" -s 40 -c 1 -o gpurun_out/r01_full_potrf_v5 python tools/quick_time.py 16384 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"adj_diag_kernel" -s 30 -c 1 -o gpurun_out/r01_full_adjdiag_v5 python tools/quick_time.py 16384 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"se_cov_kernel" -s 2 -c 1 -o gpurun_out/r01_full_secov_v5 python tools/quick_time.py 16384 > /dev/null 2>&1
python tools/run_big.py 32768 > gpurun_out/r01_large_n_v4.jsonl 2>&1
python tools/run_big.py 65536 >> gpurun_out/r01_large_n_v4.jsonl 2>&1
cat gpurun_out/r01_large_n_v4.jsonl
ls gpurun_out
