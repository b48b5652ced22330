"""NEXT-4: batched small matrices (stan_cl_cholesky_batched /
stan_cl_cholesky_adjoint_batched, n <= 128) against the oracle per matrix,
the single-matrix entry points, and the integer-exact families."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_1907_01063_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sc():
    import paper_1907_01063_b200 as m
    m.load()
    return m


def se_batch(batch, n, seed0=100):
    return np.stack([oracle.se_cov(inputs.gp_x(n, seed0 + b), 1.0, 1.0, 1e-6) for b in range(batch)])


def relf(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("batch,n", [(1, 1), (3, 2), (7, 5), (1001, 17), (64, 32), (5, 33), (99, 48), (257, 64),
                                     (33, 100), (20, 128)])
def test_cholesky_batched_parity(sc, batch, n):
    A = se_batch(batch, n)
    L, info = sc.cholesky_batched(torch.from_numpy(A).cuda())
    L = L.cpu().numpy()
    assert int(info.abs().sum()) == 0
    for b in range(batch):
        assert relf(L[b], oracle.cholesky(A[b])) <= 1e-11
        assert np.all(L[b][np.triu_indices(n, 1)] == 0.0)
    # same kernel as the single-matrix path: bit-identical
    for b in (0, batch - 1):
        assert torch.equal(sc.cholesky(torch.from_numpy(A[b]).cuda()).cpu(), torch.from_numpy(L[b]))


def test_cholesky_batched_integer_exact_in_place_and_failures(sc):
    n, batch = 128, 6
    L0 = np.stack([inputs.unit_lower_pm1(n, seed=b) for b in range(batch)])
    A = np.einsum("bij,bkj->bik", L0, L0)
    A[2, 70, 70] = -1.0  # matrix 2 fails (info 71 or earlier)
    A[4, 5, 5] = -1e9    # matrix 4 fails at row 5
    t = torch.from_numpy(A).cuda()
    lib = sc.load()
    info = torch.zeros(batch, dtype=torch.int32, device="cuda")
    rc = lib.stan_cl_cholesky_batched(batch, n, t.data_ptr(), t.data_ptr(), info.data_ptr())
    assert rc == 3  # first failing matrix is 2
    info = info.cpu().numpy()
    assert info[4] == 6 and 0 < info[2] <= 71
    assert all(info[b] == 0 for b in (0, 1, 3, 5))
    got = t.cpu().numpy()
    for b in (0, 1, 3, 5):
        assert np.array_equal(got[b], L0[b])


@pytest.mark.parametrize("batch,n", [(1, 1), (5, 3), (999, 20), (64, 32), (7, 33), (101, 50), (300, 64), (9, 100),
                                     (17, 128)])
def test_cholesky_adjoint_batched_parity(sc, batch, n):
    A = se_batch(batch, n, seed0=500)
    Ls = np.stack([oracle.cholesky(a) for a in A])
    W = np.stack([inputs.lbar(n, seed=900 + b) for b in range(batch)])
    Ab, info = sc.cholesky_adjoint_batched(torch.from_numpy(Ls).cuda(), torch.from_numpy(W).cuda())
    Ab = Ab.cpu().numpy()
    assert int(info.abs().sum()) == 0
    for b in range(batch):
        want = oracle.cholesky_adjoint(Ls[b], W[b])
        assert relf(Ab[b], want) <= 1e-9
        assert np.all(Ab[b][np.triu_indices(n, 1)] == 0.0)
    single = sc.cholesky_adjoint(torch.from_numpy(Ls[0]).cuda(), torch.from_numpy(W[0]).cuda()).cpu().numpy()
    assert relf(Ab[0], single) <= 1e-13


@pytest.mark.parametrize("n", [16, 48])
def test_cholesky_adjoint_batched_integer_exact_inplace_chunks(sc, n):
    # integer-exact banded family, a batch larger than one 4096 chunk (n = 48:
    # the padded path), in place; n = 16 runs one warp per matrix
    batch = 4100
    L1 = inputs.unit_lower_pm1(n, seed=3, band=2)
    W1 = inputs.int_lbar(n, seed=4)
    want = oracle.cholesky_adjoint(L1, W1)
    Lt = torch.from_numpy(np.broadcast_to(L1, (batch, n, n)).copy()).cuda()
    Wt = torch.from_numpy(np.broadcast_to(W1, (batch, n, n)).copy()).cuda()
    info = torch.zeros(batch, dtype=torch.int32, device="cuda")
    lib = sc.load()
    assert lib.stan_cl_cholesky_adjoint_batched(batch, n, Lt.data_ptr(), Wt.data_ptr(), Wt.data_ptr(),
                                                info.data_ptr()) == 0
    got = Wt.cpu().numpy()
    for b in (0, 1, 4095, 4096, 4099):
        assert np.array_equal(got[b], want)


def test_batched_errors(sc):
    lib = sc.load()
    t = torch.zeros(1, dtype=torch.float64, device="cuda")
    assert lib.stan_cl_cholesky_batched(2, 129, t.data_ptr(), t.data_ptr(), None) == -1
    assert lib.stan_cl_cholesky_batched(-1, 4, t.data_ptr(), t.data_ptr(), None) == -1
    assert lib.stan_cl_cholesky_batched(0, 4, None, None, None) == 0
    assert lib.stan_cl_cholesky_adjoint_batched(1, 129, t.data_ptr(), t.data_ptr(), t.data_ptr(), None) == -1
    Lb = torch.from_numpy(np.stack([np.eye(4), np.diag([1.0, 0.0, 1.0, 1.0])])).cuda()
    info = torch.zeros(2, dtype=torch.int32, device="cuda")
    rc = lib.stan_cl_cholesky_adjoint_batched(2, 4, Lb.data_ptr(), Lb.data_ptr(),
                                              torch.empty_like(Lb).data_ptr(), info.data_ptr())
    assert rc == 2 and info.cpu().tolist() == [0, 2]


@pytest.mark.parametrize("n", [40, 64])
def test_batched_w64_failures_and_in_place(sc, n):
    """32 < n <= 64 (two warps per matrix): per-matrix info of the first failing
    pivot, bit-exact integer family, in place."""
    batch = 9
    L0 = np.stack([inputs.unit_lower_pm1(n, seed=b) for b in range(batch)])
    A = np.einsum("bij,bkj->bik", L0, L0)
    A[3, n - 1, n - 1] = -1.0
    A[7, 10, 10] = -1e9
    t = torch.from_numpy(A).cuda()
    info = torch.zeros(batch, dtype=torch.int32, device="cuda")
    assert sc.load().stan_cl_cholesky_batched(batch, n, t.data_ptr(), t.data_ptr(), info.data_ptr()) == 4
    info = info.cpu().numpy()
    assert info[7] == 11 and info[3] == n
    got = t.cpu().numpy()
    for b in (0, 1, 2, 4, 5, 6, 8):
        assert info[b] == 0 and np.array_equal(got[b], L0[b])
    # adjoint: integer banded family bit for bit, in place over L_bar
    L1 = inputs.unit_lower_pm1(n, seed=3, band=2)
    W1 = inputs.int_lbar(n, seed=4)
    want = oracle.cholesky_adjoint(L1, W1)
    Lt = torch.from_numpy(np.broadcast_to(L1, (batch, n, n)).copy()).cuda()
    Wt = torch.from_numpy(np.broadcast_to(W1, (batch, n, n)).copy()).cuda()
    assert sc.load().stan_cl_cholesky_adjoint_batched(batch, n, Lt.data_ptr(), Wt.data_ptr(), Wt.data_ptr(),
                                                      None) == 0
    got = Wt.cpu().numpy()
    for b in range(batch):
        assert np.array_equal(got[b], want)
