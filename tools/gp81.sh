# fused R4 with self-resetting barrier: parity + timing
python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_gp.py -q -x 2>&1 | tail -2
python tools/quick_time.py 1024 4096 8192 16384
