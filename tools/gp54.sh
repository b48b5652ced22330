python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -q -x -k "adj or Adj or dist or host or determin" 2>&1 | tail -2
python tools/quick_time.py 1024 4096 16384
python tools/profile_classes.py 16384 csym
