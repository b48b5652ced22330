python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for pp in 0 1; do for cfg in mid,mid,big w8,w8,big w8,w8,w8 mid,mid,mid; do
  echo "pingpong=$pp cfg=$cfg"; STAN_CL_PINGPONG=$pp STAN_CL_GEMM_CFG=$cfg python tools/quick_time.py 16384 2>&1 | tail -1
done; done
ncu --set full --clock-control none --import-source on -k regex:gemm_dmma.*Li2EEEv -s 6 -c 2 -o gpurun_out/prof_splitk_r01 python tools/quick_time.py 8192 > gpurun_out/ncu_full3.log 2>&1
tail -2 gpurun_out/ncu_full3.log
