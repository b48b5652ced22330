set -x
python -m pytest tests -x -q -m gpu 2>&1 | tail -30
python tools/quick_time.py 1024 4096 8192 16384 2>&1 | tail -8
