# PDL on the dependent chains: parity (graphs on and off), timing with and without PDL
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
STAN_CL_PDL=0 python tools/quick_time.py 1024 4096 8192 16384
python tools/quick_time.py 1024 4096 8192 16384
