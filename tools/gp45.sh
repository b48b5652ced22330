compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "parity_se and (300 or 129 or 1024) or host_entry_points and 300 or blocking_invariance and 300" 2>&1 | tail -15
compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_dist.py -q -x -k "768" 2>&1 | tail -6
