./tools/potrf_lab | grep -v validate | tail -2
python -m pytest tests/test_gpu_parity.py -q -x -k "cholesky" 2>&1 | tail -1
python tools/quick_time.py 1024 4096 16384
python tools/profile_classes.py 4096 n4096
python tools/profile_classes.py 1024 n1024
