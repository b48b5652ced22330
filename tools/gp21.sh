python -m pytest tests -x -q -m gpu --durations=8 2>&1 | tail -14
python tools/profile_classes.py 16384 default
