python -m pytest tests -q -m gpu -x 2>&1 | tail -3
python tools/profile_classes.py 16384 adj256
python tools/time_host.py 16384 2>&1 | tail -1
