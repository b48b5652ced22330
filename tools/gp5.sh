python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for cfg in mid,mid,big w8,w8,big w16,w16,w16 w8,w8,w8 w16,w8,w16 big,big,mid; do
  echo "cfg=$cfg"; STAN_CL_GEMM_CFG=$cfg python -m pytest tests/test_gpu_parity.py -x -q -k "parity_se and (1000 or 1024 or 300)" 2>&1 | tail -1
  STAN_CL_GEMM_CFG=$cfg python tools/quick_time.py 16384 2>&1 | tail -1
done
