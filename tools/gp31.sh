python -m pytest tests -q -m gpu 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/r01_bench_v2.json
cut -c1-3500 gpurun_out/r01_bench_v2.json
python bench.py --impl reference --steps 2 --warmup 3 2>&1 | tail -1 | cut -c1-400
