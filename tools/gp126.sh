# Round-1 final evidence on the final code
python -m pytest tests -m gpu -q 2>&1 | tail -1 > gpurun_out/r01_gpu_tests_v13.txt; cat gpurun_out/r01_gpu_tests_v13.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py 2>&1 | tail -1 > gpurun_out/r01_bench_v13.json
python -c "import json; d=json.load(open('gpurun_out/r01_bench_v13.json')); print(d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['checked_vs_device'], d['roofline']['frac'], d['cpu_baseline']['value'], d['gpu_launches'], d['clocks'])"
python tools/quick_time.py 1024 2048 4096 8192 16384 > gpurun_out/r01_quick_time_v13.jsonl 2>&1; cat gpurun_out/r01_quick_time_v13.jsonl
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01_launches_v8.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_v8.log 2>&1
tail -1 gpurun_out/ncu_launch_v8.log | cut -c1-80
