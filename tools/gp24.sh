python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
python tools/profile_classes.py 16384 t32
