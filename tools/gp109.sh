# Final round-1 evidence (v6): full GPU suite, smoke, bench, launch list, full captures, large n
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/r01_gpu_tests_v9.txt; cat gpurun_out/r01_gpu_tests_v9.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/r01_bench_v9.json
python -c "import json; d=json.load(open('gpurun_out/r01_bench_v9.json')); print(d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['gpu_launches'], d['clocks'])"
python tools/quick_time.py 1024 4096 8192 16384 > gpurun_out/r01_quick_time_v9.jsonl 2>&1; cat gpurun_out/r01_quick_time_v9.jsonl
python tools/dist11_probe.py 8192 16384 > gpurun_out/r01_dist11_v9.jsonl 2>&1; cat gpurun_out/r01_dist11_v9.jsonl
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01_launches_v6.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_v6.log 2>&1
tail -1 gpurun_out/ncu_launch_v6.log | cut -c1-100
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"gemm_tma_kernel.*Lb1ELb0ELi0E" -s 60 -c 1 -o gpurun_out/r01_full_adjgemm_v6 python tools/quick_time.py 16384 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"potrf_tile_kernel" -s 40 -c 1 -o gpurun_out/r01_full_potrf_v6 python tools/quick_time.py 16384 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"trsm_panel_kernel" -s 40 -c 1 -o gpurun_out/r01_full_trsm_v6 python tools/quick_time.py 16384 > /dev/null 2>&1
python tools/run_big.py 32768 > gpurun_out/r01_large_n_v5.jsonl 2>&1
python tools/run_big.py 65536 >> gpurun_out/r01_large_n_v5.jsonl 2>&1
cat gpurun_out/r01_large_n_v5.jsonl
python tools/bench_batched.py > gpurun_out/r01_batched_bench_v4.jsonl 2>&1
python tools/bench_gp.py 4096 16384 > gpurun_out/r01_gp_bench_v3.txt 2>&1; tail -3 gpurun_out/r01_gp_bench_v3.txt
ls gpurun_out
