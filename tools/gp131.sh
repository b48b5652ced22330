timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -q -x 2>&1 | tail -1
timeout 300 python tools/dist11_probe.py 8192 16384
timeout 120 python tools/dist11_classes.py 16384
