python -m pytest tests -q -m gpu 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/r01_bench_v6.json
python -c "import json; d=json.load(open('gpurun_out/r01_bench_v6.json')); print(d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['gpu_launches'], d['clocks'])"
python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1
