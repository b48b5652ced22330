# fused lookahead forward (trigger after the counter wait): parity, timing
timeout 120 python tools/quick_time.py 1024 4096 8192 16384
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_gp.py -q -x 2>&1 | tail -2
