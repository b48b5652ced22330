set -x
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01_launches_traffic.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_dmma_kernel -s 40 -c 1 -o gpurun_out/r01_full_syrk python tools/quick_time.py 16384 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tma_kernel -s 300 -c 2 -o gpurun_out/r01_full_tma python tools/quick_time.py 16384 > /dev/null 2>&1
python bench.py --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/r01_bench_v1.json
cat gpurun_out/r01_bench_v1.json | cut -c1-600
ls -la gpurun_out
