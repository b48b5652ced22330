./tools/gemm_bench
python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python tools/quick_time.py 1024 8192 16384 2>&1 | tail -3
STAN_CL_PERSIST=0 STAN_CL_GEMM_CFG=w8,w8,w8 python tools/quick_time.py 16384 2>&1 | tail -1
