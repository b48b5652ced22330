# one-launch block-cyclic trailing update in the distributed forward
for i in 1 2; do timeout 600 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -1; done
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
timeout 300 python tools/dist11_probe.py 4096 8192 16384
