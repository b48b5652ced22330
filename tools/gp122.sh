# memcheck/synccheck over the host-streamed and distributed paths; final bench line with the checked e2e
compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "host" 2>&1 | tail -2 > gpurun_out/r01_sanitizer_v7.txt
compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_dist.py -q -x -k "sim2 and not 2304" 2>&1 | tail -2 >> gpurun_out/r01_sanitizer_v7.txt
compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_gpu_dist.py -q -x -k "sim2 and 1280" 2>&1 | tail -2 >> gpurun_out/r01_sanitizer_v7.txt
cat gpurun_out/r01_sanitizer_v7.txt
python bench.py 2>&1 | tail -1 > gpurun_out/r01_bench_v12.json
python -c "import json; d=json.load(open('gpurun_out/r01_bench_v12.json')); print(d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['checked_vs_device'], d['roofline']['frac'], d['clocks'])"
