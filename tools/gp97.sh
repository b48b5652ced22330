# fused lookahead forward: parity, timing fused vs not
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_gp.py -q -x 2>&1 | tail -2
STAN_CL_FUSE_LOOKAHEAD=0 timeout 300 python tools/quick_time.py 4096 8192 16384
timeout 300 python tools/quick_time.py 1024 4096 8192 16384
