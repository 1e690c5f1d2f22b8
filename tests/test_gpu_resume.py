"""GPU: a failed full-rank guess resumes tile_rec at the failed block (Driver::recover / resume,
DESIGN.md "Resume") -- bit-exact against the oracle (rankrev.hpp:85-183) on inputs whose leading
a x a block is generic and full rank and whose Schur complement is rank deficient, so the
speculative panel schedule succeeds on exactly the first a / 64 base cases and fails on the next;
plus small fields where guesses fail often, at every depth (nested node-level resumes)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _mat(rng, p, r, c):
    return rng.integers(0, p, size=(r, c), dtype=np.int64)


def prefix_then_deficient(n, a, p, seed, tail_rank):
    """A = [[Lx Ux, Lx Y], [Z Ux, S + Z Y]] mod p: leading block Lx Ux (unit lower x upper, generic),
    Schur complement S of rank tail_rank (a product of random (n-a) x r and r x (n-a) factors)."""
    rng = np.random.default_rng(seed)
    Lx = np.tril(_mat(rng, p, a, a), -1) + np.eye(a, dtype=np.int64)
    Ux = np.triu(_mat(rng, p, a, a), 1) + np.diag(rng.integers(1, p, size=a))
    Y = _mat(rng, p, a, n - a)
    Z = _mat(rng, p, n - a, a)
    S = (_mat(rng, p, n - a, tail_rank) @ _mat(rng, p, tail_rank, n - a)) % p
    top = np.hstack([(Lx @ Ux) % p, (Lx @ Y) % p])
    bot = np.hstack([(Z @ Ux) % p, (S + (Z @ Y) % p) % p])
    return np.vstack([top, bot]).astype(np.uint32)


def _check(G, ctx, O, A, p, thr=64):
    import torch
    want = O.pluq_tile_recursive(p, A, thr)
    d = torch.from_numpy(A.view(np.int32).copy()).cuda()
    res = G.pluq_tile_recursive(p, d, thr, ctx=ctx)  # device entry
    ctx.synchronize()
    got = d.cpu().numpy().view(np.uint32)
    assert res.rank == want[3]
    assert np.array_equal(res.P, want[1]) and np.array_equal(res.Q, want[2])
    assert np.array_equal(got, want[0])
    h = A.copy()
    rh = G.pluq_tile_recursive(p, h, thr, ctx=ctx)  # host entry (streamed bands)
    assert rh.rank == want[3] and np.array_equal(rh.P, want[1]) and np.array_equal(rh.Q, want[2])
    assert np.array_equal(h, want[0])


@pytest.mark.parametrize("n,a", [(512, 64), (512, 192), (512, 256), (512, 448), (1024, 320), (1024, 640)])
@pytest.mark.parametrize("tail", ["one_short", "half"])
def test_resume_after_failed_block_matches_oracle(gpu, oracle_lib, n, a, tail):
    G, ctx = gpu
    p = 131071
    r = (n - a - 1) if tail == "one_short" else (n - a) // 2
    A = prefix_then_deficient(n, a, p, 100 + n + a, r)
    _check(G, ctx, oracle_lib, A, p)


@pytest.mark.parametrize("p,n,seed", [(251, 2048, 1), (251, 2048, 2), (251, 2048, 3), (251, 2048, 5),
                                      (5, 512, 1), (3, 640, 2), (65521, 700, 4)])
def test_small_fields_resume_matches_oracle(gpu, oracle_lib, p, n, seed):
    """Random input over small fields: guesses fail at random depths (whole matrix and nodes)."""
    G, ctx = gpu
    A = oracle_lib.random_mat(p, n, n, seed)
    _check(G, ctx, oracle_lib, A, p)


def test_resume_with_deficient_leading_factor(gpu, oracle_lib):
    """Two zero pivots of the leading factor U (positions 70 and 150): blocks 1 and 2 fail inside what
    would be the prefix, the trailing Schur complement is deficient too -- nested resumes."""
    G, ctx = gpu
    p = 131071
    n, a = 512, 256
    A = prefix_then_deficient(n, a, p, 7, (n - a) // 3)
    rng = np.random.default_rng(8)
    Lx = np.tril(rng.integers(0, p, size=(a, a)), -1) + np.eye(a, dtype=np.int64)
    d = rng.integers(1, p, size=a)
    d[70] = 0
    d[150] = 0
    Ux = np.triu(rng.integers(0, p, size=(a, a)), 1) + np.diag(d)
    A[:a, :a] = ((Lx @ Ux) % p).astype(np.uint32)
    _check(G, ctx, oracle_lib, A, p)
