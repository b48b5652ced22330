for r in 8,16,8192 8,24,8192 12,24,8192 8,16,12288 8,32,4096 8,24,6144; do echo "== $r"; STAN_CL_SYRK_RESERVE=$r python tools/quick_time.py 4096 8192 16384; done
