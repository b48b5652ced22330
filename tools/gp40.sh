python -m pytest tests -q -m gpu -x 2>&1 | tail -3
python tools/profile_classes.py 16384 graphs_off_profile
python - <<'PY'
import sys, torch, json
sys.path.insert(0,'.')
import paper_1907_01063_b200 as sc
from paper_1907_01063_b200 import inputs
for n in (1024, 4096, 16384):
    x = torch.from_numpy(inputs.gp_x(n)).cuda(); K = sc.gp_exp_quad_cov(x,1,1,1e-6); W = torch.from_numpy(inputs.lbar(n)).cuda()
    A = torch.empty_like(K); L = torch.empty_like(K); Ab = torch.empty_like(K)
    def step():
        sc.gp_exp_quad_cov(x,1,1,1e-6,out=K); sc.cholesky(K, out=K); sc.cholesky_adjoint(K, W, out=Ab)
    for _ in range(3): step()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): step()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b)/5
    print(json.dumps({"n": n, "ms_per_step": ms, "tflops": n**3/ms/1e9}), flush=True)
PY
python tools/time_host.py 16384 2>&1 | tail -1
