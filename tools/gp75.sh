compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_gp.py tests/test_gpu_batched.py -q -x -k "not 4096 and not 2048 and not 5000 and not chunks" 2>&1 | tail -6 > gpurun_out/r01_sanitizer_next_rows.txt
compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_gpu_gp.py tests/test_gpu_batched.py -q -x -k "not 4096 and not 2048 and not 5000 and not chunks" 2>&1 | tail -4 >> gpurun_out/r01_sanitizer_next_rows.txt
compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 10 python -m pytest tests/test_gpu_batched.py -q -x -k "parity and (1-1 or 64-32 or 20-128)" 2>&1 | tail -6 >> gpurun_out/r01_sanitizer_next_rows.txt
cat gpurun_out/r01_sanitizer_next_rows.txt
