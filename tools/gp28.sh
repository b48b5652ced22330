./tools/gemm_bench 2>&1 | grep check
TAG=default python tools/dbg_nb.py 16384
