# Round-1 final: the committed code (tests, smoke, bench, launch list)
python -m pytest tests -m gpu -q 2>&1 | tail -1 > gpurun_out/r01_gpu_tests_v10.txt; cat gpurun_out/r01_gpu_tests_v10.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py 2>&1 | tail -1 > gpurun_out/r01_bench_v10.json
python -c "import json; d=json.load(open('gpurun_out/r01_bench_v10.json')); print(d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline'], d['cpu_baseline']['value'], d['gpu_launches'], d['clocks'])"
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01_launches_v7.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_v7.log 2>&1
tail -1 gpurun_out/ncu_launch_v7.log | cut -c1-80
python bench.py --impl reference --steps 1 --warmup 3 2>&1 | tail -1 | cut -c1-200
