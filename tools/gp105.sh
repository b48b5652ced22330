timeout 600 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -1
timeout 300 python tools/dist11_probe.py 8192 16384
