python -m pytest tests/test_gpu_batched.py -q -x 2>&1 | tail -3
python tools/bench_batched.py 2>&1 | tee gpurun_out/r01_batched_bench_v2.jsonl
