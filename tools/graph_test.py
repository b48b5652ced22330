"""Does CUDA-graph capture of the library's enqueue sequence cut time? (dev experiment)"""
import sys, torch, json
sys.path.insert(0, '.')
import paper_1907_01063_b200 as sc
from paper_1907_01063_b200 import inputs
for n in [int(a) for a in sys.argv[1:]] or [1024, 16384]:
    x = torch.from_numpy(inputs.gp_x(n)).cuda()
    K0 = sc.gp_exp_quad_cov(x, 1, 1, 1e-6)
    K = K0.clone(); L = torch.empty_like(K); W = torch.from_numpy(inputs.lbar(n)).cuda(); A = torch.empty_like(K)
    info = torch.zeros(2, dtype=torch.int32, device='cuda')
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        sc.cholesky_async(K, L, info[0:1]); sc.cholesky_adjoint_async(L, W, A, info[1:2])
    torch.cuda.synchronize()
    def t(fn, reps=5):
        best = 1e9
        for _ in range(reps):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); a.record(); fn(); b.record(); torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        return best
    eager_f = t(lambda: sc.cholesky_async(K, L, info[0:1]))
    eager_a = t(lambda: sc.cholesky_adjoint_async(L, W, A, info[1:2]))
    gf = torch.cuda.CUDAGraph(); ga = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gf, stream=s):
        sc.cholesky_async(K, L, info[0:1])
    with torch.cuda.graph(ga, stream=s):
        sc.cholesky_adjoint_async(L, W, A, info[1:2])
    graph_f = t(lambda: gf.replay()); graph_a = t(lambda: ga.replay())
    Lg = L.clone(); Ag = A.clone()
    sc.cholesky_async(K, L, info[0:1]); sc.cholesky_adjoint_async(L, W, A, info[1:2]); torch.cuda.synchronize()
    print(json.dumps({"n": n, "eager_fwd": eager_f, "graph_fwd": graph_f, "eager_adj": eager_a, "graph_adj": graph_a,
                      "same_L": bool(torch.equal(Lg, L)), "same_A": bool(torch.equal(Ag, A)), "info": info.tolist()}), flush=True)
