# fused R4 (adj_diag_kernel) + symmetric tiled SE builder: parity, timing, bench
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python tools/quick_time.py 1024 4096 8192 16384
python - <<'PY'
import torch, sys
sys.path.insert(0, '.')
import paper_1907_01063_b200 as sc
from paper_1907_01063_b200 import inputs
x = torch.from_numpy(inputs.gp_x(16384)).cuda()
K = sc.gp_exp_quad_cov(x, 1.0, 1.0, 1e-6)
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
for _ in range(3):
    torch.cuda.synchronize(); a.record(); sc.gp_exp_quad_cov(x, 1.0, 1.0, 1e-6, out=K); b.record(); torch.cuda.synchronize()
print("se_cov n=16384 ms", a.elapsed_time(b), "GB/s", 8 * 16384**2 / a.elapsed_time(b) / 1e6)
PY
python bench.py --no-cpu-baseline > gpurun_out/bench_v9.json 2> gpurun_out/bench_v9.err; tail -1 gpurun_out/bench_v9.json | cut -c1-400
