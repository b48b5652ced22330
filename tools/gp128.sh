compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 10 --kernel-name kns=adj_diag_kernel python tools/fwd_once.py 1024 adj 2>&1 | tail -2 > gpurun_out/r01_sanitizer_v8.txt
compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 10 --kernel-name kns=adj_diag_kernel python tools/fwd_once.py 300 adj 2>&1 | tail -2 >> gpurun_out/r01_sanitizer_v8.txt
compute-sanitizer --tool memcheck --print-limit 10 python tools/fwd_once.py 1024 adj 2>&1 | tail -2 >> gpurun_out/r01_sanitizer_v8.txt
compute-sanitizer --tool synccheck --print-limit 10 python tools/fwd_once.py 1024 adj 2>&1 | tail -2 >> gpurun_out/r01_sanitizer_v8.txt
cat gpurun_out/r01_sanitizer_v8.txt
