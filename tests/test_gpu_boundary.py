"""GPU checks of the C-ABI contract beyond the numerics (include/stan_cl.h):
the CUDA-graph cache across workspace growth, the caller-owned workspace
(stan_cl_set_workspace), status reporting while kernels on
other streams run, and the binding's argument checks.  Numerical results are
compared with the oracle at the parity bars of tests/test_gpu_parity.py."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest
import torch

import oracle
from paper_1907_01063_b200 import inputs

pytestmark = pytest.mark.gpu

L_TOL = 1e-11
A_TOL = 1e-9


@pytest.fixture(scope="module")
def sc():
    import paper_1907_01063_b200 as m
    m.load()
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def relf(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def se(n, seed=inputs.X_SEED):
    return oracle.se_cov(inputs.gp_x(n, seed), 1.0, 1.0, 1e-6)


def not_pd(n, row):
    """Toeplitz with one pivot pushed far negative: info = row + 1."""
    A = inputs.toeplitz(n)
    A[row, row] = -1e12
    return A


@pytest.mark.parametrize("n_small,n_big", [(1024, 8192), (1000, 4000)])
def test_graph_cache_survives_workspace_growth(sc, n_small, n_big):
    """A captured graph must not replay through workspace freed by a later, larger
    call.  n=1000 is the padded path (its
    graph writes the padded copy in a library matrix slot)."""
    lib = sc.load()
    sc.finalize()                                        # start from an empty workspace
    A = torch.empty((n_small, n_small), dtype=torch.float64, device="cuda")
    L = torch.empty_like(A)
    for it in range(2):                                  # 1st eager, 2nd captures
        K = se(n_small, seed=500 + it)
        A.copy_(torch.from_numpy(K))
        sc.cholesky(A, out=L)
    # a larger adjoint grows (frees and re-allocates) the shared workspace and slots
    Lb = dev(np.linalg.cholesky(se(n_big)))
    Wb = dev(inputs.lbar(n_big, seed=9))
    sc.cholesky_adjoint(Lb, Wb, out=Wb)
    del Lb, Wb
    torch.cuda.synchronize()
    # same buffers again: new SPD contents -> oracle parity
    K = se(n_small, seed=777)
    A.copy_(torch.from_numpy(K))
    sc.cholesky(A, out=L)
    assert relf(L.cpu().numpy(), oracle.cholesky(K)) <= L_TOL
    # ... and a non-PD matrix must report its info through the (new) status word
    A.copy_(torch.from_numpy(not_pd(n_small, n_small // 2)))
    rc = lib.stan_cl_cholesky(n_small, A.data_ptr(), L.data_ptr())
    assert rc == n_small // 2 + 1
    # and once more with good data (the graph is re-captured / replayed correctly)
    for it in range(3):
        K = se(n_small, seed=800 + it)
        A.copy_(torch.from_numpy(K))
        sc.cholesky(A, out=L)
        assert relf(L.cpu().numpy(), oracle.cholesky(K)) <= L_TOL, it


@pytest.mark.parametrize("n", [256, 1000, 1024, 2000])
def test_caller_workspace(sc, n):
    """stan_cl_set_workspace: every call carves its memory from the caller's
    buffer of stan_cl_workspace_bytes(n) bytes and gives the oracle's results;
    a buffer one allocation short returns STAN_CL_ENOMEM."""
    lib = sc.load()
    need = sc.workspace_bytes(n)
    buf = torch.empty(need // 8 + 1, dtype=torch.float64, device="cuda")
    assert buf.data_ptr() % 256 == 0
    sc.set_workspace(buf)
    try:
        K = se(n)
        Lo = oracle.cholesky(K)
        W = inputs.lbar(n)
        Ao = oracle.cholesky_adjoint(Lo, W)
        for _ in range(3):                               # eager, capture, replay
            L = sc.cholesky(dev(K))
            assert relf(L.cpu().numpy(), Lo) <= L_TOL
            Ab = sc.cholesky_adjoint(dev(Lo), dev(W))
            assert relf(Ab.cpu().numpy(), Ao) <= A_TOL
        Lh = torch.empty((n, n), dtype=torch.float64).pin_memory()
        assert sc.cholesky_host(torch.from_numpy(K).pin_memory(), Lh) == 0
        assert relf(np.tril(Lh.numpy()), Lo) <= L_TOL
        Ah = torch.empty((n, n), dtype=torch.float64).pin_memory()
        assert sc.cholesky_adjoint_host(torch.from_numpy(Lo).pin_memory(), torch.from_numpy(W).pin_memory(),
                                        Ah) == 0
        assert relf(Ah.numpy(), Ao) <= A_TOL
        x = sc.trsv(dev(Lo), dev(np.ones(n)))
        assert relf(x.cpu().numpy(), oracle.trsv(Lo, np.ones(n))) <= 1e-10
        xs = inputs.gp_x(n)
        ys = inputs.gp_y(xs)
        out, _ = sc.gp_lpdf_grad(dev(xs), dev(ys), 1.0, 1.0, 0.5)
        lp, gr, _ = oracle.gp_lpdf_grad(xs, ys, 1.0, 1.0, 0.5)
        assert abs(out[0].item() - lp) <= 1e-10 * abs(lp)
        assert relf(out[1:].cpu().numpy(), gr) <= 1e-7
        # a non-PD input still reports its pivot through the workspace's status word
        Ab_ = dev(not_pd(n, n // 3))
        assert lib.stan_cl_cholesky(n, Ab_.data_ptr(), Ab_.data_ptr()) == n // 3 + 1
    finally:
        sc.set_workspace(None)
    # too small: the largest consumer at this order fails cleanly with ENOMEM
    small = torch.empty(max(need // 2 // 8, 64), dtype=torch.float64, device="cuda")
    sc.set_workspace(small)
    try:
        Lh = torch.empty((n, n), dtype=torch.float64).pin_memory()
        Ah = torch.empty((n, n), dtype=torch.float64).pin_memory()
        rc = lib.stan_cl_cholesky_adjoint_host(n, Lh.data_ptr(), Lh.data_ptr(), Ah.data_ptr())
        assert rc == -2, rc
        assert b"caller workspace too small" in lib.stan_cl_status_string(-2)
    finally:
        sc.set_workspace(None)
    # library-owned workspace again
    L = sc.cholesky(dev(se(n)))
    assert relf(L.cpu().numpy(), oracle.cholesky(se(n))) <= L_TOL


def test_set_workspace_rejects_bad_buffers(sc):
    lib = sc.load()
    buf = torch.empty(1024, dtype=torch.float64, device="cuda")
    assert lib.stan_cl_set_workspace(ctypes.c_void_p(buf.data_ptr() + 8), 4096) == -1   # misaligned
    assert lib.stan_cl_set_workspace(ctypes.c_void_p(buf.data_ptr()), 128) == -1         # < header
    assert lib.stan_cl_set_workspace(None, 0) == 0


@pytest.mark.parametrize("n,row", [(8192, 5000), (4096, 300), (16384, 12000)])
def test_not_pd_with_lookahead_does_not_hang(sc, n, row):
    """A failing pivot found by the lookahead POTRF (side stream) while the
    persistent TMA GEMMs start on the main stream: every CTA must take the same
    exit decision, and the info must be the oracle's row."""
    lib = sc.load()
    for _ in range(3):
        A = dev(not_pd(n, row))
        assert lib.stan_cl_cholesky(n, A.data_ptr(), A.data_ptr()) == row + 1
        del A
    L = dev(se(1024))
    assert lib.stan_cl_cholesky(1024, L.data_ptr(), L.data_ptr()) == 0


def test_host_adjoint_bad_diagonal_does_not_hang(sc):
    """The streamed host adjoint checks each row block's diagonal on the copy
    stream while the sweep runs the grid-barrier diagonal kernel on the main
    stream: a bad diagonal must come back as its info."""
    for n, bad in ((4096, 3000), (4096, 100), (2000, 1999)):
        Lb = np.eye(n)
        Lb[bad, bad] = 0.0
        out = torch.empty((n, n), dtype=torch.float64).pin_memory()
        W = torch.from_numpy(inputs.lbar(n)).pin_memory()
        for _ in range(2):
            assert sc.cholesky_adjoint_host(torch.from_numpy(Lb).pin_memory(), W, out) == bad + 1


def test_binding_rejects_bad_out(sc):
    A = dev(se(64))
    with pytest.raises(ValueError):
        sc.cholesky(A, out=torch.empty((64, 64), dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        sc.cholesky(A, out=torch.empty((63, 63), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        sc.cholesky(A, out=torch.empty((64, 64), dtype=torch.float64))              # host tensor
    with pytest.raises(ValueError):
        sc.cholesky(A, out=torch.empty((64, 128), dtype=torch.float64, device="cuda")[:, :64])
    T = dev(se(64)).t()                                                             # strided view
    with pytest.raises(ValueError):
        sc.cholesky(T, out=T)
    with pytest.raises(ValueError):
        sc.cholesky_adjoint(A, A, out=torch.empty((64, 64), dtype=torch.float64, device="cuda").t())
    with pytest.raises(ValueError):
        sc.cholesky_async(A, torch.empty((64, 64), dtype=torch.float64, device="cuda").t())
    with pytest.raises(ValueError):
        sc.cholesky_adjoint_async(A, A, A, info=torch.empty(1, dtype=torch.int64, device="cuda"))
    # a non-contiguous INPUT is fine when it is not also the output (copied)
    L = sc.cholesky(T)
    assert relf(L.cpu().numpy(), oracle.cholesky(se(64))) <= L_TOL


@pytest.mark.parametrize("n", [1, 3, 31, 32, 33, 100, 257, 1000])
def test_check_matrix_vs_oracle(sc, n):
    """stan_cl_check_matrix against oracle_check_matrix on
    clean and corrupted SE matrices: every bit, every combination of checks."""
    K = se(n)
    cases = [K]
    g = np.random.default_rng(n)
    for kind in range(4):
        A = K.copy()
        i, j = int(g.integers(0, n)), int(g.integers(0, n))
        if kind == 0:
            A[i, j] = np.nan
        elif kind == 1 and n > 1:
            A[max(i, j), min(i, j)] += 1e-6 if i != j else 0.0
            A[n - 1, 0] += 3e-8
        elif kind == 2:
            A[i, i] = 0.0
        else:
            A[i, i] = -0.0
            A[j, (j + 1) % n] = np.inf
        cases.append(A)
    for A in cases:
        for checks in (1, 2, 4, 7):
            for tol in (1e-8, 1e-5):
                want = oracle.check_matrix(A, checks, tol)
                assert sc.check_matrix(dev(A), checks, tol) == want, (checks, tol)
    lib = sc.load()
    assert lib.stan_cl_check_matrix(-1, None, 1, 0.0) == -1
    assert lib.stan_cl_check_matrix(0, None, 7, 0.0) == 0
    assert lib.stan_cl_check_matrix(2, None, 8, 0.0) == -1


def test_trace_timeline(sc):
    """stan_cl_trace_*: every launch of a call is recorded with its stream and
    ordered times; the forward uses the library stream, the lookahead side
    stream and (split lookahead, the default at this size) the third stream
    for the rows below the next diagonal tile; classes match the launch kinds."""
    n = 2048
    K = dev(se(n))
    sc.cholesky(K)                                 # warm
    before = sc.kernel_launches()
    sc.trace(True)
    sc.cholesky(K)
    torch.cuda.synchronize()
    recs = sc.trace_read()
    sc.trace(False)
    assert len(recs) == sc.kernel_launches() - before
    assert all(0.0 <= a <= b for _, _, a, b in recs)
    kinds = {k for k, _, _, _ in recs}
    assert {"potrf", "trsm", "syrk", "lookahead"} <= kinds
    assert {s for _, s, _, _ in recs} == {0, 1, 2}
    sc.cholesky(K)                                 # not traced any more
    assert len(sc.trace_read()) == len(recs)


def test_c_api_demo_from_plain_c(sc, tmp_path):
    """The boundary is usable from plain C (no Python, no torch): build
    examples/c_api_demo.c with gcc against include/stan_cl.h and libstancl.so
    and run it (log-det gradient identity, status codes, caller workspace)."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "c_api_demo")
    lib_dir = os.path.join(root, "paper_1907_01063_b200")
    cmd = ["gcc", "-O2", "-std=c99", os.path.join(root, "examples", "c_api_demo.c"), "-I", os.path.join(root, "include"),
           "-I/usr/local/cuda/include", "-L" + lib_dir, "-lstancl", "-L/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath," + lib_dir, "-lm", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, timeout=120)
    r = subprocess.run([exe, "1500"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.stdout, r.stderr)
    assert "not-PD info = 1" in r.stdout
