# Re-entry check: full GPU suite, smoke, bench, launch list (fresh container)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/r01_gpu_tests_v8.txt
cat gpurun_out/r01_gpu_tests_v8.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/bench_v8.json 2> gpurun_out/bench_v8.err; tail -1 gpurun_out/bench_v8.json
