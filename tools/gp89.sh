# e2e with PDL off inside the host entry points; sanitizer on the fused diagonal step + PDL chains
python -m pytest tests/test_gpu_parity.py -q -x -k "host" 2>&1 | tail -2
python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import sys, json; d = json.loads(sys.stdin.read()); print(round(d['ms_per_step'], 2), 'e2e', round(d['e2e']['ms_per_step'], 2))"
compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "adjoint and not full and not 4096" 2>&1 | tail -4 > gpurun_out/r01_sanitizer_v5.txt
compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 10 python tools/fwd_once.py 1024 adj 2>&1 | tail -4 >> gpurun_out/r01_sanitizer_v5.txt
compute-sanitizer --tool synccheck --print-limit 10 python tools/fwd_once.py 1024 adj 2>&1 | tail -4 >> gpurun_out/r01_sanitizer_v5.txt
cat gpurun_out/r01_sanitizer_v5.txt
