python -m pytest tests -q -m gpu 2>&1 | tail -3
python tools/profile_classes.py 16384 ob256fix
