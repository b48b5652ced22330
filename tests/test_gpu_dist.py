"""Multi-GPU path (block-cyclic by 256-wide block columns).

On a one-GPU box the distributed algorithms run with G simulated ranks in one
process (stan_cl_dist_sim_*: the same code, broadcasts become device copies)
and are checked against the oracle and the integer-exact families.  The NCCL
transport itself is exercised by test_nccl_ranks when >= 2 GPUs are visible.
"""
from __future__ import annotations

import ctypes
import os
import socket

import numpy as np
import pytest
import torch

import oracle
from paper_1907_01063_b200 import inputs

pytestmark = pytest.mark.gpu
B = 256


@pytest.fixture(scope="module")
def sc():
    import paper_1907_01063_b200 as m
    m.load()
    return m


def se(n, seed=inputs.X_SEED, jitter=1e-6):
    return oracle.se_cov(inputs.gp_x(n, seed), 1.0, 1.0, jitter)


def relf(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def scatter_padded(sc, A: np.ndarray, G: int):
    n = A.shape[0]
    At = torch.from_numpy(np.ascontiguousarray(A)).cuda()
    width = max(sc.dist_owned_blocks(n, G, q) for q in range(G)) * B
    outs = []
    for q in range(G):
        loc = sc.dist_scatter(At, G, q)
        pad = torch.zeros((n, width), dtype=torch.float64, device="cuda")
        pad[:, :loc.shape[1]] = loc
        outs.append(pad.contiguous())
    return outs


def check_lower_and_tiles(got: np.ndarray, want: np.ndarray, tol: float):
    n = want.shape[0]
    lo = np.tril_indices(n)
    assert relf(got[lo], want[lo]) <= tol
    i, j = np.triu_indices(n, 1)
    in_tile = (i // B) == (j // B)
    assert np.all(got[i[in_tile], j[in_tile]] == 0.0)


@pytest.mark.parametrize("n,G", [(256, 1), (768, 2), (1024, 3), (1536, 4), (1024, 4)])
def test_dist_sim_cholesky(sc, n, G):
    K = se(n)
    locs = scatter_padded(sc, K, G)
    assert sc.dist_sim_cholesky(locs, n) == 0
    got = sc.dist_gather(locs, n).cpu().numpy()
    check_lower_and_tiles(got, oracle.cholesky(K), 1e-11)
    # integer-exact family: bit-for-bit
    L0 = inputs.unit_lower_pm1(n, seed=n + G)
    locs = scatter_padded(sc, inputs.gram_exact(L0), G)
    assert sc.dist_sim_cholesky(locs, n) == 0
    got = sc.dist_gather(locs, n).cpu().numpy()
    assert np.array_equal(np.tril(got), L0)


@pytest.mark.parametrize("n,G", [(256, 1), (768, 2), (1024, 3), (1536, 4)])
def test_dist_sim_adjoint(sc, n, G):
    L = oracle.cholesky(se(n))
    W = inputs.lbar(n)
    Ls = scatter_padded(sc, L, G)
    Ws = scatter_padded(sc, W, G)
    assert sc.dist_sim_cholesky_adjoint(Ls, Ws, n) == 0
    got = sc.dist_gather(Ws, n).cpu().numpy()
    check_lower_and_tiles(got, oracle.cholesky_adjoint(L, W), 1e-9)
    Li = inputs.unit_lower_pm1(n, seed=3, band=2)
    Wi = inputs.int_lbar(n, seed=4)
    Ls = scatter_padded(sc, Li, G)
    Ws = scatter_padded(sc, Wi, G)
    assert sc.dist_sim_cholesky_adjoint(Ls, Ws, n) == 0
    assert np.array_equal(np.tril(sc.dist_gather(Ws, n).cpu().numpy()), oracle.cholesky_adjoint(Li, Wi))


@pytest.mark.parametrize("n,G", [(768, 2), (1024, 3)])
def test_se_cov_cols(sc, n, G):
    x = torch.from_numpy(inputs.gp_x(n)).cuda()
    K = sc.gp_exp_quad_cov(x, 1.3, 0.7, 1e-6)
    for q in range(G):
        w = sc.dist_owned_blocks(n, G, q) * B
        loc = torch.empty((n, w), dtype=torch.float64, device="cuda")
        sc.gp_exp_quad_cov_cols(x, loc, G, q, 1.3, 0.7, 1e-6)
        assert torch.equal(loc, sc.dist_scatter(K, G, q))


def test_dist_not_pd_and_errors(sc):
    n, G = 768, 2
    A = inputs.toeplitz(n)
    A[600, 600] = -1e12
    locs = scatter_padded(sc, A, G)
    assert sc.dist_sim_cholesky(locs, n) == 601
    lib = sc.load()
    t = torch.zeros(300, 512, dtype=torch.float64, device="cuda")
    assert lib.stan_cl_dist_cholesky(300, 0, t.data_ptr(), 512) == -1      # no communicator
    assert lib.stan_cl_dist_init(2, 0, None, 1, 2) == -1                    # no id
    idb = (ctypes.c_char * 128)()
    assert lib.stan_cl_dist_init(2, 0, ctypes.cast(idb, ctypes.c_void_p), 2, 2) == -1   # P*Q != nranks
    assert lib.stan_cl_dist_init(2, 0, ctypes.cast(idb, ctypes.c_void_p), 0, 2) == -1   # P < 1


# ---- 2-D block-cyclic grids (P > 1): row/column broadcasts, column reductions
GRIDS = [(1280, 2, 1), (1792, 2, 2), (1280, 3, 2), (2304, 2, 4), (1536, 2, 3), (768, 4, 1)]


def scatter2(sc, A: np.ndarray, P: int, Q: int):
    n = A.shape[0]
    At = torch.from_numpy(np.ascontiguousarray(A)).cuda()
    width = max(sc.dist_local_shape(n, P, Q, 0, q)[1] for q in range(Q))
    return [sc.dist_scatter2(At, P, Q, r // Q, r % Q, width).contiguous() for r in range(P * Q)]


@pytest.mark.parametrize("n,P,Q", GRIDS)
def test_dist_sim2_cholesky(sc, n, P, Q):
    K = se(n)
    locs = scatter2(sc, K, P, Q)
    assert sc.dist_sim2_cholesky(locs, n, P, Q) == 0
    got = sc.dist_gather2(locs, n, P, Q).cpu().numpy()
    check_lower_and_tiles(got, oracle.cholesky(K), 1e-11)
    L0 = inputs.unit_lower_pm1(n, seed=n + P * Q)       # integer-exact family: bit for bit
    locs = scatter2(sc, inputs.gram_exact(L0), P, Q)
    assert sc.dist_sim2_cholesky(locs, n, P, Q) == 0
    assert np.array_equal(np.tril(sc.dist_gather2(locs, n, P, Q).cpu().numpy()), L0)


@pytest.mark.parametrize("n,P,Q", GRIDS)
def test_dist_sim2_adjoint(sc, n, P, Q):
    L = oracle.cholesky(se(n))
    W = inputs.lbar(n)
    Ls, Ws = scatter2(sc, L, P, Q), scatter2(sc, W, P, Q)
    assert sc.dist_sim2_cholesky_adjoint(Ls, Ws, n, P, Q) == 0
    check_lower_and_tiles(sc.dist_gather2(Ws, n, P, Q).cpu().numpy(), oracle.cholesky_adjoint(L, W), 1e-9)
    Li = inputs.unit_lower_pm1(n, seed=3, band=2)       # integer-exact adjoint family: bit for bit
    Wi = inputs.int_lbar(n, seed=4)
    Ls, Ws = scatter2(sc, Li, P, Q), scatter2(sc, Wi, P, Q)
    assert sc.dist_sim2_cholesky_adjoint(Ls, Ws, n, P, Q) == 0
    assert np.array_equal(np.tril(sc.dist_gather2(Ws, n, P, Q).cpu().numpy()), oracle.cholesky_adjoint(Li, Wi))


@pytest.mark.parametrize("n,P,Q", [(4096, 2, 4), (4096, 4, 2), (3072, 3, 3)])
def test_dist_sim2_large(sc, n, P, Q):
    """More steps and wider column exchanges than the oracle-sized cases: the
    distributed results against the single-GPU device path (itself pinned to the
    oracle) and the integer-exact families bit for bit."""
    K = se(n)
    Kt = torch.from_numpy(K).cuda()
    L1 = sc.cholesky(Kt)
    W = inputs.lbar(n)
    A1 = sc.cholesky_adjoint(L1, torch.from_numpy(W).cuda())
    locs = scatter2(sc, K, P, Q)
    assert sc.dist_sim2_cholesky(locs, n, P, Q) == 0
    Ld = sc.dist_gather2(locs, n, P, Q).cpu().numpy()
    check_lower_and_tiles(Ld, L1.cpu().numpy(), 1e-11)
    L1n = L1.cpu().numpy()
    Ls, Ws = scatter2(sc, L1n, P, Q), scatter2(sc, W, P, Q)
    assert sc.dist_sim2_cholesky_adjoint(Ls, Ws, n, P, Q) == 0
    check_lower_and_tiles(sc.dist_gather2(Ws, n, P, Q).cpu().numpy(), A1.cpu().numpy(), 1e-9)
    L0 = inputs.unit_lower_pm1(n, seed=n + 7)
    locs = scatter2(sc, inputs.gram_exact(L0), P, Q)
    assert sc.dist_sim2_cholesky(locs, n, P, Q) == 0
    assert np.array_equal(np.tril(sc.dist_gather2(locs, n, P, Q).cpu().numpy()), L0)
    Li = inputs.unit_lower_pm1(n, seed=5, band=2)
    Wi = inputs.int_lbar(n, seed=6)
    Ls, Ws = scatter2(sc, Li, P, Q), scatter2(sc, Wi, P, Q)
    assert sc.dist_sim2_cholesky_adjoint(Ls, Ws, n, P, Q) == 0
    Ai = sc.cholesky_adjoint(torch.from_numpy(Li).cuda(), torch.from_numpy(Wi).cuda()).cpu().numpy()
    assert np.array_equal(np.tril(sc.dist_gather2(Ws, n, P, Q).cpu().numpy()), np.tril(Ai))


def test_dist_sim2_matches_single_gpu_layout(sc):
    """P = 1 of the 2-D code is the block-column layout: same bits as dist_sim on 1 x G."""
    n = 1280
    K = se(n)
    a = scatter2(sc, K, 1, 3)
    b = scatter_padded(sc, K, 3)
    assert sc.dist_sim2_cholesky(a, n, 1, 3) == 0 and sc.dist_sim_cholesky(b, n) == 0
    assert torch.equal(sc.dist_gather2(a, n, 1, 3), sc.dist_gather(b, n))


@pytest.mark.parametrize("n,P,Q", [(1280, 2, 2), (1536, 3, 2)])
def test_se_cov_tiles(sc, n, P, Q):
    x = torch.from_numpy(inputs.gp_x(n)).cuda()
    K = sc.gp_exp_quad_cov(x, 1.3, 0.7, 1e-6)
    for r in range(P * Q):
        p, q = divmod(r, Q)
        rows, cols = sc.dist_local_shape(n, P, Q, p, q)
        loc = torch.empty((rows, cols), dtype=torch.float64, device="cuda")
        sc.gp_exp_quad_cov_tiles(x, loc, P, Q, p, q, 1.3, 0.7, 1e-6)
        assert torch.equal(loc, sc.dist_scatter2(K, P, Q, p, q))


def test_dist_sim2_not_pd(sc):
    n, P, Q = 1280, 2, 2
    A = inputs.toeplitz(n)
    A[1000, 1000] = -1e12
    assert sc.dist_sim2_cholesky(scatter2(sc, A, P, Q), n, P, Q) == 1001


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _nccl_worker(rank, world, port, n, P, Q, q):
    """One rank of a real NCCL run on a P x Q grid: forward on the SE covariance,
    adjoint on the ORACLE's L (the A_bar bar is for the same L bits on both sides;
    no oracle input comes from the CUDA path)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    import paper_1907_01063_b200 as sc
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        sc.dist_init_from_torch(None, P, Q)
        p_, q_ = divmod(rank, Q)
        K = torch.from_numpy(se(n)).cuda()
        loc = sc.dist_scatter2(K, P, Q, p_, q_).contiguous()
        rc = sc.dist_cholesky(loc, n)
        Lo = torch.from_numpy(oracle.cholesky(se(n))).cuda()
        Lloc = sc.dist_scatter2(Lo, P, Q, p_, q_).contiguous()
        W = sc.dist_scatter2(torch.from_numpy(inputs.lbar(n)).cuda(), P, Q, p_, q_).contiguous()
        rca = sc.dist_cholesky_adjoint(Lloc, W, n)
        gl, gw = [None] * world, [None] * world
        dist.all_gather_object(gl, loc.cpu())
        dist.all_gather_object(gw, W.cpu())
        q.put((rank, rc, rca, [g.numpy() for g in gl] if rank == 0 else None,
               [g.numpy() for g in gw] if rank == 0 else None))
    except Exception as e:  # noqa: BLE001
        q.put((rank, "error", repr(e), None, None))
    finally:
        sc.load().stan_cl_dist_finalize()
        dist.destroy_process_group()


def _nccl_single_worker(port, n, q):
    """world_size 1: the real NCCL path (dlopen, ncclCommInitRank, two ncclCommSplit,
    the status all-reduce, finalize) on one device, forward + adjoint."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    import paper_1907_01063_b200 as sc
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        grid = sc.dist_init_from_torch()
        K = torch.from_numpy(se(n)).cuda()
        loc = sc.dist_scatter2(K, 1, 1, 0, 0).contiguous()
        rc = sc.dist_cholesky(loc, n)
        L = loc.cpu().numpy()
        Lo = torch.from_numpy(oracle.cholesky(se(n))).cuda()
        Lloc = sc.dist_scatter2(Lo, 1, 1, 0, 0).contiguous()
        W = torch.from_numpy(inputs.lbar(n)).cuda().contiguous()
        rca = sc.dist_cholesky_adjoint(Lloc, W, n)
        A = sc.load().stan_cl_dist_init(1, 0, None, 1, 1)        # already initialised / bad id
        q.put((grid, rc, rca, L, W.cpu().numpy(), A))
    except Exception as e:  # noqa: BLE001
        q.put(("error", repr(e)))
    finally:
        sc.load().stan_cl_dist_finalize()
        dist.destroy_process_group()


def test_nccl_single_rank(sc):
    import torch.multiprocessing as mp
    n = 768
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_single_worker, args=(_free_port(), n, q))
    p.start()
    res = q.get(timeout=300)
    p.join(timeout=60)
    assert res[0] != "error", res
    grid, rc, rca, L, Ab, again = res
    assert grid == (1, 1) and rc == 0 and rca == 0 and again == -1
    K = se(n)
    Lo = oracle.cholesky(K)
    check_lower_and_tiles(L, Lo, 1e-11)
    check_lower_and_tiles(Ab, oracle.cholesky_adjoint(Lo, inputs.lbar(n)), 1e-9)


@pytest.mark.parametrize("P,Q", [(1, 2), (2, 1), (2, 2)])
def test_nccl_ranks(sc, P, Q):
    """Real ncclBroadcast / ncclReduce on P x Q ranks (one GPU each): forward and
    adjoint against the oracle."""
    import torch.multiprocessing as mp
    world, n = P * Q, 1536
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_nccl_worker, args=(r, world, port, n, P, Q, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        r, rc, rca, gl, gw = q.get(timeout=300)
        res[r] = (rc, rca, gl, gw)
    for p in ps:
        p.join(timeout=60)
    assert all(v[0] == 0 and v[1] == 0 for v in res.values()), res
    L = sc.dist_gather2([torch.from_numpy(g) for g in res[0][2]], n, P, Q).numpy()
    Ab = sc.dist_gather2([torch.from_numpy(g) for g in res[0][3]], n, P, Q).numpy()
    K = se(n)
    Lo = oracle.cholesky(K)
    check_lower_and_tiles(L, Lo, 1e-11)
    check_lower_and_tiles(Ab, oracle.cholesky_adjoint(Lo, inputs.lbar(n)), 1e-9)


def _trace_all(sc, n, P, Q, adjoint):
    """Every rank's recorded NCCL sequence (stan_cl_dist_trace), run one rank at a
    time on this device through the real per-rank code path."""
    out = {}
    for r in range(P * Q):
        p, q = divmod(r, Q)
        rows, cols = sc.dist_local_shape(n, P, Q, p, q)
        A = torch.zeros((max(rows, 1), max(cols, B)), dtype=torch.float64, device="cuda")
        L = torch.zeros_like(A) if adjoint else None
        out[(p, q)] = sc.dist_trace(n, P, Q, p, q, adjoint, A, L)
    return out


@pytest.mark.parametrize("P,Q", [(1, 2), (2, 1), (2, 2), (2, 4), (4, 2), (3, 3)])
@pytest.mark.parametrize("adjoint", [False, True])
def test_collective_schedule_consistent(sc, P, Q, adjoint):
    """Deadlock / count check of the multi-GPU schedule:
    every member of each row, column and world communicator must issue the same
    sequence of (op, root, count, stream) on it, as NCCL requires; roots are
    members; every broadcast moves whole 256 x 256 tiles."""
    n = 256 * 11                                       # 11 block rows: ragged over every grid
    tr = _trace_all(sc, n, P, Q, adjoint)
    ranks = sorted(tr)
    seqs = {}
    for (p, q) in ranks:
        for kind, idx, op, root, cnt, st in tr[(p, q)]:
            if kind == 0:
                assert idx == p
                assert 0 <= root < Q
            elif kind == 1:
                assert idx == q
                assert 0 <= root < P
            seqs.setdefault((kind, idx), {}).setdefault((p, q), []).append((op, root, cnt, st))
            if op == 0:
                assert cnt > 0 and cnt % B == 0
    # every member of a communicator appears with an identical sequence
    for (kind, idx), per in seqs.items():
        members = [(idx, q) for q in range(Q)] if kind == 0 else \
                  [(p, idx) for p in range(P)] if kind == 1 else ranks
        assert sorted(per) == sorted(members), (kind, idx, sorted(per))
        first = per[members[0]]
        for m in members[1:]:
            assert per[m] == first, (kind, idx, m)
    # there is real traffic: forward broadcasts panels on both kinds of
    # communicator when both grid dimensions exceed 1; the adjoint reduces over
    # process columns when P > 1
    ops = [e for v in tr.values() for e in v]
    if Q > 1:
        assert any(e[0] == 0 and e[2] == 0 for e in ops)
    if P > 1:
        assert any(e[0] == 1 and e[2] == 0 for e in ops)
        if adjoint:
            assert any(e[2] == 1 for e in ops)
    assert sum(1 for e in ops if e[0] == 2) == P * Q   # one status all-reduce per rank
