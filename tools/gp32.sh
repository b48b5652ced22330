python -m pytest tests -q -m gpu -x 2>&1 | tail -3
python bench.py --steps 3 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], json.dumps(d['e2e']))"
