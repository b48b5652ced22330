python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python tools/profile_classes.py 16384 ob256
