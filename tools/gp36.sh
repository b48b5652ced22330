python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
python tools/profile_classes.py 16384 g128fix
python tools/quick_time.py 1024 2>&1 | tail -1
