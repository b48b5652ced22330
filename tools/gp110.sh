# A/B: adjoint narrow GEMMs (R1, R5) on the one-tile-per-CTA kernel
for m in 0 1 2 3; do echo "== NARROW_W8=$m"; STAN_CL_NARROW_W8=$m python tools/quick_time.py 4096 8192 16384 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['n'], round(d['adj_ms'], 3))"; done
