"""The pipelined host entry (ffg_pluq_tile_recursive: spine-first upload, early download of
the root's top rows) against the device entry on the same inputs, at sizes where the spine
has several levels, on full-rank and rank-deficient inputs (where R's permutations and the
pivot-gather rotations reach back into the early-downloaded rows), with lda > n."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape", [(3000, 3000), (4500, 2600), (2600, 4500)])
@pytest.mark.parametrize("gen", ["iid", "lru", "lowrank"])
def test_host_entry_matches_device_entry(gpu, oracle_lib, shape, gen):
    import torch

    G, ctx = gpu
    O = oracle_lib
    p = 131071
    m, n = shape
    N = max(m, n)
    if gen == "iid":
        A = O.random_mat(p, m, n, m + n)
    elif gen == "lru":
        d = torch.empty((N, N), dtype=torch.int32, device="cuda")
        G.lru_matrix_dev(p, d, N // 3, 5, ctx=ctx)
        ctx.synchronize()
        A = d.cpu().numpy().view(np.uint32)[:m, :n].copy()
    else:  # rank 700 product: every block rank deficient, nontrivial permutations everywhere
        L = O.random_mat(p, m, 700, 1).astype(np.uint64)
        R = O.random_mat(p, 700, n, 2).astype(np.uint64)
        A = np.zeros((m, n), np.uint32)
        for k0 in range(0, 700, 64):
            A = ((A.astype(np.uint64) + L[:, k0:k0 + 64] @ R[k0:k0 + 64, :]) % p).astype(np.uint32)
    # device entry
    d = torch.from_numpy(A.view(np.int32).copy()).cuda()
    rd = G.pluq_tile_recursive(p, d, 64, ctx=ctx)
    ctx.synchronize()
    want = d.cpu().numpy().view(np.uint32)
    # host entry, with a padded leading dimension
    ld = n + 37
    buf = np.full((m, ld), 0xDEADBEEF, np.uint32)
    buf[:, :n] = A
    view = buf[:, :n]
    rh = G.pluq_tile_recursive(p, view, 64, ctx=ctx)
    assert rh.rank == rd.rank
    assert np.array_equal(rh.P, rd.P) and np.array_equal(rh.Q, rd.Q)
    assert np.array_equal(view, want)
    assert np.all(buf[:, n:] == 0xDEADBEEF)  # padding untouched


@pytest.mark.parametrize("threads", ["0", "4"])
def test_concurrent_subtrees_match_oracle(gpu, oracle_lib, threads, monkeypatch):
    """Rank-deficient L*R*U input with many E/G forks (thr 16): the concurrent-subtree driver
    (E || G on separate host threads / streams / mailboxes) is bit-identical to the oracle."""
    import torch

    G, ctx = gpu
    O = oracle_lib
    p = 131071
    n = 1024
    d = torch.empty((n, n), dtype=torch.int32, device="cuda")
    G.lru_matrix_dev(p, d, n // 2, 11, ctx=ctx)
    ctx.synchronize()
    A = d.cpu().numpy().view(np.uint32).copy()
    a_o, P_o, Q_o, r_o = O.pluq_tile_recursive(p, A, 16)
    monkeypatch.setenv("FFG_SUBTREE_THREADS", threads)
    a_g = A.copy()
    res = G.pluq_tile_recursive(p, a_g, 16, ctx=ctx)
    assert res.rank == r_o == n // 2
    assert np.array_equal(res.P, P_o) and np.array_equal(res.Q, Q_o)
    assert np.array_equal(a_g, a_o)


@pytest.mark.parametrize("n,dup", [(2048, None), (1500, None), (2048, (1900, 5)), (2048, (200, 7)), (777, None)])
def test_streamed_speculative_host_entry(gpu, oracle_lib, n, dup):
    """Square input through the host entry takes the streamed speculative path (bands upload,
    factor and download concurrently).  A duplicated row makes a late (1900) or early (200) base
    case rank deficient: the guess fails after earlier bands already reached the host buffer, and
    the exact rerun from the HBM backup must still produce the oracle's outputs."""
    G, _ = gpu
    O = oracle_lib
    p = 131071
    A = O.random_mat(p, n, n, 40 + n)
    if dup:
        A[dup[0], :] = A[dup[1], :]
    a_o, P_o, Q_o, r_o = O.pluq_tile_recursive(p, A, 64)
    ctx = G.Context(0)  # fresh: no rest period from an earlier failed guess
    try:
        ld = n + 5
        buf = np.full((n, ld), 0xDEADBEEF, np.uint32)
        buf[:, :n] = A
        view = buf[:, :n]
        res = G.pluq_tile_recursive(p, view, 64, ctx=ctx)
        assert res.rank == r_o
        assert np.array_equal(res.P, P_o) and np.array_equal(res.Q, Q_o)
        assert np.array_equal(view, a_o)
        assert np.all(buf[:, n:] == 0xDEADBEEF)
    finally:
        ctx.close()
