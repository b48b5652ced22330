for t in 1,1,1 0,1,1 0,0,1 1,0,1 0,0,0; do STAN_CL_TMA=$t STAN_CL_GEMM_CFG=w8,w8,w8 python tools/profile_classes.py 16384 tma=$t; done
