# distributed adjoint with lookahead: simulated grids + single-rank NCCL, repeated to shake out races
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -1; done
