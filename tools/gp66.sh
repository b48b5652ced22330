for r in 8,24,8192 4,16,8192 6,16,8192 4,24,8192 8,16,8192 4,12,8192 8,32,8192; do echo "== $r"; STAN_CL_SYRK_RESERVE=$r python tools/quick_time.py 4096 8192 16384; done
