compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "parity_se and (300 or 129)" 2>&1 | tail -12
compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "parity_se and (300 or 129)" 2>&1 | tail -6
