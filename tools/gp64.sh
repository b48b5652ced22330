./tools/potrf_lab | grep -v validate
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -q -x 2>&1 | tail -2
python tools/quick_time.py 1024 4096 8192 16384
python tools/profile_classes.py 16384 potrfC
