# racecheck / synccheck restricted to the kernels changed this session; batched bench refresh
compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 10 --kernel-regex kns=potrf_tile_kernel,kns=adj_diag_kernel,kns=trsm_panel_kernel,kns=se_cov_kernel python tools/fwd_once.py 1024 adj 2>&1 | tail -3 > gpurun_out/r01_sanitizer_v6.txt
compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 10 --kernel-regex kns=potrf_w32_kernel,kns=potrf_batched_kernel python -m pytest tests/test_gpu_batched.py -q -x -k "parity and (1-1 or 64-32 or 20-128)" 2>&1 | tail -3 >> gpurun_out/r01_sanitizer_v6.txt
compute-sanitizer --tool memcheck --print-limit 10 python tools/fwd_once.py 1024 adj 2>&1 | tail -2 >> gpurun_out/r01_sanitizer_v6.txt
compute-sanitizer --tool synccheck --print-limit 10 python tools/fwd_once.py 1024 adj 2>&1 | tail -2 >> gpurun_out/r01_sanitizer_v6.txt
cat gpurun_out/r01_sanitizer_v6.txt
python tools/bench_batched.py > gpurun_out/r01_batched_bench_v3.jsonl 2>&1; cat gpurun_out/r01_batched_bench_v3.jsonl
