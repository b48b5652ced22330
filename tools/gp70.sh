python -m pytest tests/test_gpu_gp.py -q -x 2>&1 | tail -2
python tools/bench_gp.py 4096 16384 2>&1 | python3 -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['n'], round(d['gp_lpdf_grad_ms'], 3), {k: round(v['ms'], 3) for k, v in d['trsv'].items()})"
