"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star): relative Frobenius error <= 1e-11 for L and
<= 1e-9 for A_bar, with the SAME input bits on both sides (the oracle's K for
the forward, the oracle's L for the adjoint).  Integer work
(the integer-exact families, status codes) is compared bit-exactly.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_1907_01063_b200 import inputs

pytestmark = pytest.mark.gpu

L_BAR_TOL = 1e-11
A_BAR_TOL = 1e-9


@pytest.fixture(scope="module")
def sc():
    import paper_1907_01063_b200 as m
    m.load()
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.cpu().numpy()


def relf(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def se(n, seed=inputs.X_SEED, jitter=1e-6):
    return oracle.se_cov(inputs.gp_x(n, seed), 1.0, 1.0, jitter)


SIZES = [1, 2, 3, 31, 64, 100, 127, 128, 129, 255, 256, 300, 511, 512, 1000, 1024]


# ------------------------------------------------------------------ SE builder
@pytest.mark.parametrize("n", [1, 7, 64, 300, 1024])
def test_se_cov_matches_oracle(sc, n):
    x = inputs.gp_x(n)
    for alpha, rho, jit in [(1.0, 1.0, 1e-6), (2.5, 0.3, 0.0), (0.7, 5.5, 1e-3)]:
        want = oracle.se_cov(x, alpha, rho, jit)
        got = host(sc.gp_exp_quad_cov(dev(x), alpha, rho, jit))
        # CUDA exp vs libm exp differ by <= 2 ulp; everything else is exact
        assert np.all(np.abs(got - want) <= 4 * np.finfo(float).eps * np.abs(want) + 1e-300)
        assert np.array_equal(got, got.T)
        assert np.all(np.diag(got) == alpha * alpha + jit)


# --------------------------------------------------------------------- forward
@pytest.mark.parametrize("n", SIZES)
def test_cholesky_parity_se(sc, n):
    K = se(n)
    want = oracle.cholesky(K)
    got = host(sc.cholesky(dev(K)))
    assert relf(got, want) <= L_BAR_TOL
    up = got[np.triu_indices(n, 1)]
    assert np.all(up == 0) and not np.any(np.signbit(up))


@pytest.mark.parametrize("n", [3, 130, 700])
def test_cholesky_parity_toeplitz(sc, n):
    A = inputs.toeplitz(n)                       # the paper's benchmark matrix
    assert relf(host(sc.cholesky(dev(A))), oracle.cholesky(A)) <= 1e-14


@pytest.mark.parametrize("n", [64, 200, 1000, 1024, 2048])
def test_cholesky_integer_exact(sc, n):
    L0 = inputs.unit_lower_pm1(n, seed=n)
    A = inputs.gram_exact(L0)
    assert np.array_equal(host(sc.cholesky(dev(A))), L0)


@pytest.mark.parametrize("n", [300, 1000, 1024, 2048])
def test_cholesky_blocking_invariance(sc, n):
    # outer block 128 vs 256 (two-level): both within the bar of the oracle and of
    # each other (SPEC.md:490 blocking invariance)
    K = se(n)
    want = oracle.cholesky(K)
    lib = sc.load()
    outs = []
    try:
        for nb in (128, 256):
            assert lib.stan_cl_set_block_size(nb) == 0
            outs.append(host(sc.cholesky(dev(K))))
    finally:
        lib.stan_cl_set_block_size(0)
    for o in outs:
        assert relf(o, want) <= L_BAR_TOL
    assert relf(outs[0], outs[1]) <= L_BAR_TOL
    L0 = inputs.unit_lower_pm1(n, seed=n + 1)
    A = inputs.gram_exact(L0)
    for nb in (128, 256):
        lib.stan_cl_set_block_size(nb)
        try:
            assert np.array_equal(host(sc.cholesky(dev(A))), L0)
        finally:
            lib.stan_cl_set_block_size(0)


@pytest.mark.parametrize("n", [256, 700])
def test_cholesky_power_of_two_scaling(sc, n):
    """chol(D A D) = D chol(A) for D = diag(2^e_i): with power-of-two scales every
    product, sum, square root and quotient of the algorithm scales exactly, so
    the GPU result must be D times its unscaled result BIT FOR BIT.  The scales
    put pivots at 2^+-800, outside [2^-600, 2^600], which exercises the exact
    rescaling of the call-free sqrt/reciprocal (R12).  The paper's
    Toeplitz matrix keeps every intermediate normal under these scales (SE
    entries down to 1e-87 would underflow)."""
    A = inputs.toeplitz(n)
    e = np.random.default_rng(n).integers(-400, 401, n).astype(np.float64)
    e[:3] = [400, -400, 0]
    d = np.exp2(e)
    As = A * d[:, None] * d[None, :]
    L = host(sc.cholesky(dev(A)))
    Ls = host(sc.cholesky(dev(As)))
    assert np.array_equal(Ls, L * d[:, None])
    assert relf(L, oracle.cholesky(A)) <= L_BAR_TOL


def test_cholesky_in_place_and_upper_garbage(sc):
    n = 384
    K = se(n)
    want = oracle.cholesky(K)
    G = K.copy()
    G[np.triu_indices(n, 1)] = np.nan
    t = dev(G)
    sc.cholesky(t, out=t)                         # A == L
    assert relf(host(t), want) <= L_BAR_TOL
    assert np.all(host(t)[np.triu_indices(n, 1)] == 0)
    t2 = dev(G[:300, :300].copy())                # ragged (padded) path, in place
    sc.cholesky(t2, out=t2)
    assert relf(host(t2), oracle.cholesky(K[:300, :300])) <= L_BAR_TOL


def test_cholesky_not_pd(sc):
    for A, info in [(np.array([[1.0, 2.0], [2.0, 1.0]]), 2), (np.array([[-1.0]]), 1)]:
        with pytest.raises(sc.NotPositiveDefinite) as e:
            sc.cholesky(dev(A))
        assert e.value.info == info
    for n, r in [(64, 10), (300, 200), (1024, 1000), (1024, 128), (512, 0)]:
        A = inputs.toeplitz(n)
        A[r, r] = -1e12
        with pytest.raises(sc.NotPositiveDefinite) as e:
            sc.cholesky(dev(A))
        assert e.value.info == r + 1 == oracle.cholesky_info(A)[1]
        A = inputs.toeplitz(n)
        A[r, r] = np.nan
        with pytest.raises(sc.NotPositiveDefinite) as e:
            sc.cholesky(dev(A))
        assert e.value.info == r + 1


def test_cholesky_empty_and_errors(sc):
    lib = sc.load()
    assert lib.stan_cl_cholesky(0, None, None) == 0
    assert lib.stan_cl_cholesky(-1, None, None) == -1
    assert lib.stan_cl_cholesky(4, None, None) == -1
    t = torch.zeros(8, 8, dtype=torch.float64, device="cuda")
    # partial overlap of A and L is rejected
    assert lib.stan_cl_cholesky(4, t.data_ptr(), t.data_ptr() + 8) == -1
    assert lib.stan_cl_gp_exp_quad_cov(4, t.data_ptr(), 1.0, 0.0, 0.0, t.data_ptr()) == -1


def test_cholesky_non_default_stream(sc):
    n = 512
    K = se(n)
    want = oracle.cholesky(K)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        A = dev(K)
        L = sc.cholesky(A)
    s.synchronize()
    assert relf(host(L), want) <= L_BAR_TOL


@pytest.mark.parametrize("n", [1024, 4096])
def test_deterministic(sc, n):
    # fixed reduction orders everywhere (no atomics in the arithmetic): repeated
    # runs are bit-identical; also catches ordering races
    K = dev(se(n))
    Ls = [sc.cholesky(K) for _ in range(3)]
    assert all(torch.equal(Ls[0], x) for x in Ls[1:])
    W = dev(inputs.lbar(n))
    As = [sc.cholesky_adjoint(Ls[0], W) for _ in range(3)]
    assert all(torch.equal(As[0], x) for x in As[1:])


# --------------------------------------------------------------------- adjoint
@pytest.mark.parametrize("n", SIZES)
def test_adjoint_parity_se(sc, n):
    L = oracle.cholesky(se(n))                    # same L bits on both sides
    W = inputs.lbar(n)
    want = oracle.cholesky_adjoint(L, W)
    got = host(sc.cholesky_adjoint(dev(L), dev(W)))
    assert relf(got, want) <= A_BAR_TOL
    up = got[np.triu_indices(n, 1)]
    assert np.all(up == 0) and not np.any(np.signbit(up))


@pytest.mark.parametrize("n", [130, 512])
def test_adjoint_parity_toeplitz(sc, n):
    L = oracle.cholesky(inputs.toeplitz(n))
    W = inputs.lbar(n, seed=5)
    assert relf(host(sc.cholesky_adjoint(dev(L), dev(W))), oracle.cholesky_adjoint(L, W)) <= 1e-12


@pytest.mark.parametrize("n,band", [(256, 1), (256, 2), (1024, 2), (1000, 1)])
def test_adjoint_integer_exact(sc, n, band):
    L = inputs.unit_lower_pm1(n, seed=3, band=band)
    W = inputs.int_lbar(n, seed=4)
    want = oracle.cholesky_adjoint(L, W)
    assert np.array_equal(host(sc.cholesky_adjoint(dev(L), dev(W))), want)


@pytest.mark.parametrize("n", [300, 1024, 2048])
def test_adjoint_blocking_invariance(sc, n):
    # adjoint block 128 vs 256: both within the bar of the oracle and of each other
    # (SPEC.md:492); the integer-exact banded family is bit-identical across both
    L = oracle.cholesky(se(n))
    W = inputs.lbar(n)
    want = oracle.cholesky_adjoint(L, W)
    Li = inputs.unit_lower_pm1(n, seed=3, band=2)
    Wi = inputs.int_lbar(n, seed=4)
    want_i = oracle.cholesky_adjoint(Li, Wi)
    lib = sc.load()
    outs = []
    try:
        for nb in (128, 256):
            assert lib.stan_cl_set_adjoint_block_size(nb) == 0
            outs.append(host(sc.cholesky_adjoint(dev(L), dev(W))))
            assert np.array_equal(host(sc.cholesky_adjoint(dev(Li), dev(Wi))), want_i)
    finally:
        lib.stan_cl_set_adjoint_block_size(0)
    for o in outs:
        assert relf(o, want) <= A_BAR_TOL
    assert relf(outs[0], outs[1]) <= 1e-10


def test_adjoint_in_place_and_upper_garbage(sc):
    n = 384
    L = oracle.cholesky(se(n))
    W = inputs.lbar(n)
    want = oracle.cholesky_adjoint(L, W)
    Lg, Wg = L.copy(), W.copy()
    Lg[np.triu_indices(n, 1)] = np.nan
    Wg[np.triu_indices(n, 1)] = np.nan
    t = dev(Wg)
    sc.cholesky_adjoint(dev(Lg), t, out=t)
    assert relf(host(t), want) <= A_BAR_TOL
    assert np.all(host(t)[np.triu_indices(n, 1)] == 0)


def test_adjoint_bad_diagonal_and_errors(sc):
    lib = sc.load()
    L = np.eye(300)
    L[150, 150] = 0.0
    with pytest.raises(ValueError):
        sc.cholesky_adjoint(dev(L), dev(np.eye(300)))
    Ld = dev(L)
    out = torch.empty_like(Ld)
    assert lib.stan_cl_cholesky_adjoint(300, Ld.data_ptr(), Ld.data_ptr(), out.data_ptr()) == 151
    assert lib.stan_cl_cholesky_adjoint(300, Ld.data_ptr(), out.data_ptr(), Ld.data_ptr()) == -1  # A_bar == L
    assert lib.stan_cl_cholesky_adjoint(0, None, None, None) == 0


def test_adjoint_zero_seed(sc):
    n = 256
    L = oracle.cholesky(se(n))
    got = host(sc.cholesky_adjoint(dev(L), dev(np.zeros((n, n)))))
    assert np.array_equal(got, np.zeros((n, n)))


# ----------------------------------------------------------- host-buffer API
def _check_host_output(out, want, tol, n):
    lo = np.tril_indices(n)
    assert relf(out[lo], want[lo]) <= tol
    # the whole strict upper triangle is +0.0: the sentinel 7.0
    # is gone everywhere and no zero carries a sign bit
    up = out[np.triu_indices(n, 1)]
    assert np.all(up == 0.0) and not np.any(np.signbit(up))


@pytest.mark.parametrize("n", [100, 300, 640, 1024, 2048])
def test_host_entry_points(sc, n):
    # packed (lower-triangle) streamed transfers through the host-buffer C ABI
    K = se(n)
    G = K.copy()
    G[np.triu_indices(n, 1)] = np.nan                       # upper of the host input is ignored
    A = torch.from_numpy(G).pin_memory()
    L = torch.full((n, n), 7.0, dtype=torch.float64).pin_memory()
    assert sc.cholesky_host(A, L) == 0
    Lo = oracle.cholesky(K)
    _check_host_output(L.numpy(), Lo, L_BAR_TOL, n)
    W = inputs.lbar(n)
    Wg = W.copy()
    Wg[np.triu_indices(n, 1)] = np.nan
    Lg = Lo.copy()
    Lg[np.triu_indices(n, 1)] = np.nan
    Ab = torch.full((n, n), 7.0, dtype=torch.float64).pin_memory()
    assert sc.cholesky_adjoint_host(torch.from_numpy(Lg), torch.from_numpy(Wg), Ab) == 0
    _check_host_output(Ab.numpy(), oracle.cholesky_adjoint(Lo, W), A_BAR_TOL, n)


@pytest.mark.parametrize("n", [4096, 5000])
def test_host_matches_device(sc, n):
    """The streamed host entry points (packed transfers on copy streams, per-block
    D^-1 computed on the copy stream while the sweep already runs) reproduce the
    device-resident calls at sizes with many 256-wide adjoint blocks (the device
    path is pinned to the oracle elsewhere; the oracle is too slow here)."""
    K = inputs.gp_x(n)
    K = oracle.se_cov(K, 1.0, 1.0, 1e-6)
    W = inputs.lbar(n)
    Ld = sc.cholesky(torch.from_numpy(K).cuda())
    Ad = sc.cholesky_adjoint(Ld, torch.from_numpy(W).cuda())
    Lh = torch.empty((n, n), dtype=torch.float64).pin_memory()
    assert sc.cholesky_host(torch.from_numpy(K).pin_memory(), Lh) == 0
    Ah = torch.empty((n, n), dtype=torch.float64).pin_memory()
    assert sc.cholesky_adjoint_host(Ld.cpu().pin_memory(), torch.from_numpy(W).pin_memory(), Ah) == 0
    lo = np.tril_indices(n)
    assert relf(Lh.numpy()[lo], Ld.cpu().numpy()[lo]) <= 1e-14
    assert relf(Ah.numpy()[lo], Ad.cpu().numpy()[lo]) <= 1e-13


def test_host_entry_points_errors(sc):
    n = 400
    A = inputs.toeplitz(n)
    A[250, 250] = -1e12
    L = torch.empty((n, n), dtype=torch.float64).pin_memory()
    assert sc.cholesky_host(torch.from_numpy(A).pin_memory(), L) == 251
    Lb = np.eye(n)
    Lb[333, 333] = 0.0
    out = torch.empty((n, n), dtype=torch.float64).pin_memory()
    assert sc.cholesky_adjoint_host(torch.from_numpy(Lb), torch.from_numpy(np.eye(n)), out) == 334


def test_kernel_launch_counter(sc):
    before = sc.kernel_launches()
    sc.cholesky(dev(se(256)))
    assert sc.kernel_launches() > before


@pytest.mark.parametrize("n", [300, 1024])
def test_graph_replay_same_buffers(sc, n):
    # the 2nd call with the same buffers captures a CUDA graph, later calls replay
    # it: results must follow the buffer CONTENTS of every call
    A = torch.empty((n, n), dtype=torch.float64, device="cuda")
    L = torch.empty_like(A)
    W = torch.empty_like(A)
    Ab = torch.empty_like(A)
    before = sc.kernel_launches()
    for it in range(4):
        K = se(n, seed=100 + it)
        A.copy_(torch.from_numpy(K))
        sc.cholesky(A, out=L)
        Lo = oracle.cholesky(K)
        assert relf(host(L), Lo) <= L_BAR_TOL, it
        Wn = inputs.lbar(n, seed=200 + it)
        L.copy_(torch.from_numpy(Lo))
        W.copy_(torch.from_numpy(Wn))
        sc.cholesky_adjoint(L, W, out=Ab)
        assert relf(host(Ab), oracle.cholesky_adjoint(Lo, Wn)) <= A_BAR_TOL, it
    assert sc.kernel_launches() > before      # replays are counted
    Ah = torch.empty((n, n), dtype=torch.float64).pin_memory()
    Lh = torch.empty_like(Ah).pin_memory()
    for it in range(3):
        K = se(n, seed=300 + it)
        Ah.copy_(torch.from_numpy(K))
        assert sc.cholesky_host(Ah, Lh) == 0
        lo = np.tril_indices(n)
        assert relf(Lh.numpy()[lo], oracle.cholesky(K)[lo]) <= L_BAR_TOL, it


def test_host_adjoint_repeatable_fullsize(sc):
    """The streamed host adjoint against the device adjoint, bit for bit, over
    repeated calls at n = 16384: with its per-block kernels (tile zeroing,
    diagonal check, D^-1) on the copy stream beside the sweep it returned wrong
    entries in ~1 of 12 calls (round-2 stress test); they now run
    in stream order with the sweep."""
    n = 16384
    x = torch.from_numpy(inputs.gp_x(n)).cuda()
    L = sc.cholesky(sc.gp_exp_quad_cov(x, 1.0, 1.0, 1e-6))
    W = torch.from_numpy(inputs.lbar(n)).cuda()
    A0 = torch.tril(sc.cholesky_adjoint(L, W)).cpu()
    Lh, Wh = L.cpu().pin_memory(), W.cpu().pin_memory()
    Ah = torch.empty_like(Lh).pin_memory()
    for it in range(16):
        assert sc.cholesky_adjoint_host(Lh, Wh, Ah) == 0
        assert torch.equal(torch.tril(Ah), A0), it


def _forward_subprocess(env_extra, n, nb, exact=False):
    """L of the SE problem (or of the integer-exact family) at order n from a
    fresh process with the given environment."""
    import os
    import subprocess
    import sys
    import tempfile
    make = (f"L0 = inputs.unit_lower_pm1(n, seed=11); K = inputs.gram_exact(L0)" if exact
            else "K = oracle.se_cov(inputs.gp_x(n), 1.0, 1.0, 1e-6)")
    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, '.');"
        "import oracle, paper_1907_01063_b200 as sc; from paper_1907_01063_b200 import inputs;"
        f"n = {n}; {make}; lib = sc.load(); assert lib.stan_cl_set_block_size({nb}) == 0;"
        "L = sc.cholesky(torch.from_numpy(K).cuda());"
        "np.save(sys.argv[1], L.cpu().numpy())")
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "l.npy")
        env = dict(os.environ, **env_extra)
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        r = subprocess.run([sys.executable, "-c", code, out], env=env, cwd=root, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        return np.load(out)


@pytest.mark.parametrize("n,nb", [(1024, 128), (2048, 256), (3000, 128)])
def test_forward_schedules(n, nb):
    """The forward's lookahead schedules (STAN_CL_LA_SIDE = 0: lookahead column
    on the main stream; 1: on the side stream; 2: depth 2, the column block
    k+2 taking panels k and k+1 in one product; 3: split, the next diagonal
    tile alone on the side stream, the rows below on a third stream) at 128- and 256-wide outer
    blocks: each within the L tolerance of the oracle, the integer-exact family
    bit for bit."""
    K = se(n)
    want = oracle.cholesky(K)
    lo = np.tril_indices(n)
    L0 = inputs.unit_lower_pm1(n, seed=11)
    for m in ("0", "1", "2", "3"):
        env = {"STAN_CL_LA_SIDE": m}
        got = _forward_subprocess(env, n, nb)
        assert relf(got[lo], want[lo]) <= L_BAR_TOL, m
        assert np.all(np.triu(got, 1) == 0)
        assert np.array_equal(_forward_subprocess(env, n, nb, exact=True), L0), m


def _adjoint_bits_subprocess(env_extra, n):
    """A_bar of the SE problem at order n from a fresh process with the given
    environment (the schedule switches are read once per process)."""
    import os
    import subprocess
    import sys
    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, '.');"
        "import oracle, paper_1907_01063_b200 as sc; from paper_1907_01063_b200 import inputs;"
        f"n = {n}; K = oracle.se_cov(inputs.gp_x(n), 1.0, 1.0, 1e-6); L = oracle.cholesky_par(K);"
        "W = inputs.lbar(n); A = sc.cholesky_adjoint(torch.from_numpy(L).cuda(), torch.from_numpy(W).cuda());"
        "np.save(sys.argv[1], A.cpu().numpy())")
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "a.npy")
        env = dict(os.environ, **env_extra)
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        r = subprocess.run([sys.executable, "-c", code, out], env=env, cwd=root, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        return np.load(out)


@pytest.mark.parametrize("n", [1024, 3072])
def test_adjoint_schedules_bit_identical(n):
    """The three adjoint schedules (sequential, two-stream pipeline, merged
    single stream -- STAN_CL_ADJ_PIPE=0/1/2) give the same bits:
    every element receives the same updates from the same kernels in the same
    order; and they match the oracle."""
    got = {m: _adjoint_bits_subprocess({"STAN_CL_ADJ_PIPE": str(m)}, n) for m in (0, 1, 2)}
    assert np.array_equal(got[0].view(np.int64), got[2].view(np.int64))
    assert np.array_equal(got[1].view(np.int64), got[2].view(np.int64))
    K = se(n)
    want = oracle.cholesky_adjoint(oracle.cholesky_par(K), inputs.lbar(n))
    assert relf(got[2], want) <= A_BAR_TOL
