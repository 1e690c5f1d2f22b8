"""Profile-first exact path on the B200 (csrc/profile.cu) against the oracle (reference-pinned).

  * ffg_rank_profile_dev (phase 1: the cluster slab search + tensor-core trailing updates) must
    return rr_base's pivots P[:r], Q[:r] in discovery order (rankrev.hpp:40-57);
  * ffg_pluq_from_profile_dev (phases 2 + 3) must return tile_rec's packed L\\U, P, Q, rank;
  * the whole path through ffg_pluq_tile_recursive[_dev] (FFG_PROFILE_FIRST=2 forces it) must
    equal pluq_tile_recursive bit for bit -- rank-deficient, full-rank, small fields, ragged
    shapes, several slabs and several cluster CTAs.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cases(O):
    rng = np.random.default_rng(2024)
    out = []
    for (m, n) in ((1, 1), (1, 77), (90, 1), (33, 33), (64, 100), (130, 70), (257, 300), (300, 257), (700, 650),
                   (96, 2000), (520, 1500)):
        for p in (3, 251, 131071):
            rk = int(rng.integers(0, min(m, n) + 1))
            out.append((f"gen p={p} {m}x{n} r={rk}", p, O.generate_matrix(p, m, n, rk, int(rng.integers(1 << 30)))[0]))
        out.append((f"iid p=2 {m}x{n}", 2, O.random_mat(2, m, n, 5)))
        out.append((f"iid p=131071 {m}x{n}", 131071, O.random_mat(131071, m, n, 6)))
    for (n, r, s) in ((256, 128, 1), (600, 300, 2), (1000, 999, 3), (512, 0, 4)):
        out.append((f"lru n={n} r={r}", 131071, O.lru_matrix(n, r, 131071, s)[0]))
    out.append(("zero 100x140", 65521, np.zeros((100, 140), np.uint32)))
    out.append(("identity 200", 67108859, np.eye(200, dtype=np.uint32)))
    return out


def _to_dev(A):
    import torch
    return torch.from_numpy(A.astype(np.int32)).cuda()


@pytest.mark.parametrize("smem_kernel", [False, True])
def test_rank_profile_equals_rr_base_pivots(gpu, oracle_lib, smem_kernel, monkeypatch):
    """Both slab kernels: the register-resident one (<= 1024 columns per cluster CTA, the default)
    and the shared-memory one (wider matrices; FFG_RP_SMEM=1 forces it at every width)."""
    G, ctx = gpu
    O = oracle_lib
    if smem_kernel:
        monkeypatch.setenv("FFG_RP_SMEM", "1")
    for name, p, A in _cases(O):
        _, Pb, Qb, rb = O.rr_base(p, A.copy())
        d = _to_dev(A)
        rows, cols = G.rank_profile_dev(p, d, ctx=ctx)
        assert rows.size == rb, (name, rows.size, rb)
        assert np.array_equal(rows, Pb[:rb]) and np.array_equal(cols, Qb[:rb]), name
        assert np.array_equal(d.cpu().numpy().astype(np.uint32), A), f"{name}: input modified"


def test_pluq_from_profile_matches_tile_rec(gpu, oracle_lib):
    G, ctx = gpu
    O = oracle_lib
    for name, p, A in _cases(O)[::2]:
        _, Pb, Qb, rb = O.rr_base(p, A.copy())
        for thr in (1, 8, 64):
            want = O.pluq_tile_recursive(p, A.copy(), thr)
            d = _to_dev(A)
            res = G.pluq_from_profile_dev(p, d, thr, Pb[:rb], Qb[:rb], ctx=ctx)
            assert res.rank == want[3], name
            assert np.array_equal(res.P, want[1]) and np.array_equal(res.Q, want[2]), (name, thr)
            assert np.array_equal(d.cpu().numpy().astype(np.uint32), want[0]), (name, thr)


@pytest.mark.parametrize("entry", ["dev", "host"])
def test_profile_first_path_matches_reference(gpu, oracle_lib, entry, monkeypatch):
    G, ctx = gpu
    O = oracle_lib
    monkeypatch.setenv("FFG_PROFILE_FIRST", "2")
    for name, p, A in _cases(O)[1::2]:
        for thr in (4, 64):
            want = O.pluq_tile_recursive(p, A.copy(), thr)
            if entry == "dev":
                d = _to_dev(A)
                res = G.pluq_tile_recursive(p, d, thr, ctx=ctx)
                got = d.cpu().numpy().astype(np.uint32)
            else:
                got = A.copy()
                res = G.pluq_tile_recursive(p, got, thr, ctx=ctx)
            assert res.rank == want[3], name
            assert np.array_equal(res.P, want[1]) and np.array_equal(res.Q, want[2]), (name, thr)
            assert np.array_equal(got, want[0]), (name, thr)


def test_profile_first_default_policy_lru_2048(gpu, oracle_lib):
    """Default policy: the whole-matrix guess fails at the first block of an L*R*U input, the
    profile-first path takes over."""
    G, ctx = gpu
    O = oracle_lib
    p = 131071
    A, rows, cols = O.lru_matrix(2048, 1024, p, 9)
    want = O.pluq_tile_recursive(p, A.copy(), 64)
    d = _to_dev(A)
    res = G.pluq_tile_recursive(p, d, 64, ctx=ctx)
    assert res.rank == 1024
    assert np.array_equal(res.P, want[1]) and np.array_equal(res.Q, want[2])
    assert np.array_equal(d.cpu().numpy().astype(np.uint32), want[0])
    assert set(zip(res.P[:1024].tolist(), res.Q[:1024].tolist())) == set(zip(rows.tolist(), cols.tolist()))
