# warm per-class event times with the chain serialized (no lookahead), n = 4096 and 8192
STAN_CL_GRAPH=0 STAN_CL_NO_LOOKAHEAD=1 python tools/profile_classes.py 4096 serial
STAN_CL_GRAPH=0 STAN_CL_NO_LOOKAHEAD=1 python tools/profile_classes.py 8192 serial
STAN_CL_GRAPH=0 python tools/profile_classes.py 4096 lookahead
