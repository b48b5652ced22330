python -m pytest tests -m gpu -q 2>&1 | tail -1 > gpurun_out/r01_gpu_tests_v14.txt; cat gpurun_out/r01_gpu_tests_v14.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py 2>&1 | tail -1 > gpurun_out/r01_bench_v14.json
python -c "import json; d=json.load(open('gpurun_out/r01_bench_v14.json')); print(d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['checked_vs_device'], d['roofline']['frac'], d['clocks'])"
