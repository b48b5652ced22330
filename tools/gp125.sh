timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
timeout 300 python tools/quick_time.py 1024 2048 4096 8192 16384
