for r in 0 4 8 12 16 24; do STAN_CL_SYRK_RESERVE=$r python tools/profile_classes.py 16384 reserve$r; done
STAN_CL_TMA=0,1,1 python tools/profile_classes.py 16384 w8syrk
for r in 4 8 16; do STAN_CL_SYRK_RESERVE=$r python tools/quick_time.py 1024 4096 8192; done
