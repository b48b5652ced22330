mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/r01_bench_v4.json
python -c "import json; d=json.load(open('gpurun_out/r01_bench_v4.json')); print(d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['gpu_launches'], d['clocks'])"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01_launches_v2.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_v2.log 2>&1
tail -2 gpurun_out/ncu_launch_v2.log
ncu --set full --clock-control none --import-source on -k regex:gemm_dmma_kernel -s 40 -c 1 -o gpurun_out/r01_full_syrk_v2 python tools/quick_time.py 16384 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tma_kernel -s 300 -c 2 -o gpurun_out/r01_full_tma_v2 python tools/quick_time.py 16384 > /dev/null 2>&1
ls -la gpurun_out
