# Round-1 final (after the host-adjoint race fix): tests, smoke, bench line
python -m pytest tests -m gpu -q 2>&1 | tail -1 > gpurun_out/r01_gpu_tests_v11.txt; cat gpurun_out/r01_gpu_tests_v11.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py 2>&1 | tail -1 > gpurun_out/r01_bench_v11.json
python -c "import json; d=json.load(open('gpurun_out/r01_bench_v11.json')); print(d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['cpu_baseline']['value'], d['gpu_launches'], d['clocks'])"
python tools/quick_time.py 1024 2048 4096 8192 16384 > gpurun_out/r01_quick_time_v11.jsonl 2>&1; cat gpurun_out/r01_quick_time_v11.jsonl
