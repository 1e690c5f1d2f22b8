"""Partitioned (multi-GPU) PLUQ on one GPU: every slice of a virtual world computed locally,
optionally through the exchange's pack/unpack staging (loopback).  Outputs must be bit-identical
to the oracle and to the unpartitioned GPU run."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ctx(G, world, loopback, min_work):
    ctx = G.Context(0)
    ctx.dist_init_virtual(world, loopback)
    ctx.dist_set_min_work(min_work)
    return ctx


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("loopback", [False, True])
def test_virtual_world_matches_oracle(gpu, oracle_lib, world, loopback):
    G, _ = gpu
    O = oracle_lib
    p = 131071
    ctx = _ctx(G, world, loopback, 1)  # partition every Schur operation, however small
    try:
        info = ctx.dist_info()
        assert info["world"] == world and info["virtual"]
        rng = np.random.default_rng(world * 10 + loopback)
        for t in range(6):
            m, n = int(rng.integers(130, 420)), int(rng.integers(130, 420))
            if t % 2 == 0:
                A = O.random_mat(p, m, n, 500 + t)
            else:
                N = max(m, n)
                M, _, _ = O.lru_matrix(N, N // 3, p, 40 + t)
                A = M[:m, :n].copy()
            for thr in (8, 32):
                a_o, P_o, Q_o, r_o = O.pluq_tile_recursive(p, A, thr)
                a_g = A.copy()
                res = G.pluq_tile_recursive(p, a_g, thr, ctx=ctx)
                assert res.rank == r_o
                assert np.array_equal(res.P, P_o) and np.array_equal(res.Q, Q_o)
                assert np.array_equal(a_g, a_o)
    finally:
        ctx.close()


@pytest.mark.parametrize("p", [251, 131071])
def test_virtual_world_matches_single_gpu_large(gpu, p, monkeypatch):
    """n = 2048 rank-deficient and full-rank inputs: partitioned (4 virtual ranks, loopback,
    default min_work and a small one) vs the single-GPU path, bit for bit."""
    import torch

    G, ctx1 = gpu
    n = 2048
    # generic (split) node GEMMs above 256: corner nodes' deferred GEMMs stay replicated
    monkeypatch.setenv("FFG_CORNER_MAX", "256")
    for gen in ("iid", "lru"):
        d = torch.empty((n, n), dtype=torch.int32, device="cuda")
        if gen == "iid":
            G.random_mat_dev(p, d, 77, ctx=ctx1)
        else:
            G.lru_matrix_dev(p, d, n // 2, 78, ctx=ctx1)
        ctx1.synchronize()
        A = d.cpu().numpy().view(np.uint32).copy()
        a1 = A.copy()
        r1 = G.pluq_tile_recursive(p, a1, 64, ctx=ctx1)
        for min_work in (1 << 28, 1 << 20):
            ctx = _ctx(G, 4, True, min_work)
            try:
                a4 = A.copy()
                r4 = G.pluq_tile_recursive(p, a4, 64, ctx=ctx)
                assert r4.rank == r1.rank
                assert np.array_equal(r4.P, r1.P) and np.array_equal(r4.Q, r1.Q)
                assert np.array_equal(a4, a1)
                if min_work == 1 << 20:
                    assert ctx.dist_info()["exchanges"] > 0  # loopback staged the slices
            finally:
                ctx.close()


def test_world_one_is_plain(gpu, oracle_lib):
    G, _ = gpu
    O = oracle_lib
    ctx = G.Context(0)
    try:
        ctx.dist_init_virtual(1)
        assert ctx.dist_info()["world"] == 1 and not ctx.dist_info()["virtual"]
        ctx.dist_init(1, 0, G.dist_unique_id())  # a one-rank world needs no communicator
        A = O.random_mat(131071, 300, 300, 9)
        a_o, P_o, Q_o, r_o = O.pluq_tile_recursive(131071, A, 32)
        res = G.pluq_tile_recursive(131071, A, 32, ctx=ctx)
        assert res.rank == r_o and np.array_equal(A, a_o)
        ctx.dist_finalize()
    finally:
        ctx.close()


@pytest.mark.parametrize("world,loopback", [(2, True), (4, False), (8, True)])
@pytest.mark.parametrize("n,ks", [(1024, []), (2048, [100, 700]), (1500, [5, 64, 1400])])
def test_virtual_world_panel_schedule(gpu, oracle_lib, world, loopback, n, ks, monkeypatch):
    """Square full-rank input on a partitioned context: the speculative panel schedule runs on
    one stream, its large node GEMMs split over the (virtual) ranks and all-gathered, column
    pivots included -- bit-exact against the oracle through the device and host entries."""
    import torch

    from test_gpu_parity import _zero_schur_pivot

    G, _ = gpu
    O = oracle_lib
    p = 131071
    A = _zero_schur_pivot(O.random_mat(p, n, n, 21 + n), p, [k for k in ks if k < n])
    a_o, P_o, Q_o, r_o = O.pluq_tile_recursive(p, A, 64)
    # nodes above 256 take the generic node branch, whose GEMMs are split (corner nodes stay
    # replicated: their wide GEMMs run on side streams, and only the critical stream may
    # issue collectives)
    monkeypatch.setenv("FFG_CORNER_MAX", "256")
    ctx = _ctx(G, world, loopback, 1 << 20)
    try:
        d = torch.from_numpy(A.view(np.int32).copy()).cuda()
        res = G.pluq_tile_recursive(p, d, 64, ctx=ctx)
        ctx.synchronize()
        assert res.rank == r_o
        assert np.array_equal(res.P, P_o) and np.array_equal(res.Q, Q_o)
        assert np.array_equal(d.cpu().numpy().view(np.uint32), a_o)
        h = A.copy()
        res = G.pluq_tile_recursive(p, h, 64, ctx=ctx)
        assert res.rank == r_o and np.array_equal(h, a_o)
        assert np.array_equal(res.P, P_o) and np.array_equal(res.Q, Q_o)
        assert ctx.dist_info()["exchanges"] > 0 or not loopback
    finally:
        ctx.close()
