# 2-D block-cyclic distributed layer: simulated P x Q grids vs the oracle
python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -15
