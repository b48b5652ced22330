TAG=default python tools/dbg_nb.py 16384
TAG=nolook STAN_CL_NO_LOOKAHEAD=1 python tools/dbg_nb.py 16384
TAG=notma STAN_CL_TMA=0 python tools/dbg_nb.py 16384
