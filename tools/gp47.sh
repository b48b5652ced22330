compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 6 python -m pytest tests/test_gpu_parity.py -q -x -k "parity_se and 300" 2>&1 | grep -v "Host Frame" | head -60
