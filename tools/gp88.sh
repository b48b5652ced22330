# dist lookahead parity; e2e with PDL on/off
python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -2
for pdl in 1 0 1; do STAN_CL_PDL=$pdl python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import sys, json; d = json.loads(sys.stdin.read()); print('pdl=$pdl', round(d['ms_per_step'], 2), 'e2e', round(d['e2e']['ms_per_step'], 2))"; done
