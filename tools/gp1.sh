nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks_fp64peak.csv &
SMI=$!
./tools/fp64_peak > gpurun_out/fp64_peak.jsonl 2>&1
kill $SMI
nvidia-smi -q | grep -iE "product name|fp64|Max Clocks" -A0 | head; nproc; grep "model name" /proc/cpuinfo | head -1
