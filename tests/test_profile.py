"""tile_rec's permutations from the rank profile matrix alone (csrc/rpsim.cu, ffg_tile_rec_perms).

The profile-first exact path rests on three facts, each checked here against the
reference's algorithm (the oracle, itself pinned to oracle/_ref's outputs):
  1. every rank-profile-revealing elimination finds the same pivot set R_A:
     rr_base (rankrev.hpp:29-78) and tile_rec (:85-183) agree on it;
  2. tile_rec's P and Q depend on R_A only: tile_rec run on the 0/1 matrix R_A
     returns the same arrays -- and ffg_tile_rec_perms computes them without
     touching a matrix;
  3. given P, Q and the rank, the packed L\\U is the unique LU without pivoting of
     A[P][:, Q] on its leading rank x rank block, with a zero trailing block.
At full size the config-4 profile is known (R's support) and the reference's P/Q
hashes are pinned in tests/golden/full_size.json.
"""
import json
import os

import numpy as np
import pytest

from golden_util import fnv_u32

FULL = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "full_size.json")


def _cases(O, seed):
    rng = np.random.default_rng(seed)
    out = []
    for p in (2, 3, 5, 251, 65521, 131071):
        for t in range(6):
            m, n = int(rng.integers(1, 160)), int(rng.integers(1, 160))
            rk = int(rng.integers(0, min(m, n) + 1))
            if t % 3 == 0:
                A = O.random_mat(p, m, n, 50 + t)  # i.i.d. (small p: accidental deficiency)
            else:
                A = O.generate_matrix(p, m, n, rk, 500 + 7 * t + p % 97)[0]
            out.append((p, A))
    for (n, r, s) in ((256, 128, 1), (300, 100, 2), (200, 199, 3), (130, 0, 4)):
        out.append((131071, O.lru_matrix(n, r, 131071, s)[0]))
    return out


def test_profile_determines_tile_rec_perms(oracle_lib):
    import paper_1402_3501_b200 as G
    O = oracle_lib
    checked = 0
    for p, A in _cases(O, 7):
        m, n = A.shape
        _, Pb, Qb, rb = O.rr_base(p, A.copy())
        for thr in (1, 3, 8, 64):
            packed, P, Q, r = O.pluq_tile_recursive(p, A.copy(), thr)
            assert r == rb
            # 1: same pivot set as rr_base
            assert set(zip(P[:r].tolist(), Q[:r].tolist())) == set(zip(Pb[:rb].tolist(), Qb[:rb].tolist()))
            # 2: the simulation from the profile alone (pivots handed over in rr_base's order)
            Ps, Qs, rs = G.tile_rec_perms(m, n, thr, Pb[:rb], Qb[:rb])
            assert rs == r and np.array_equal(Ps, P) and np.array_equal(Qs, Q), (p, m, n, thr)
            checked += 1
    assert checked > 100


def _lu_from_pq(p, A, P, Q, r):
    B = A[P.astype(np.int64)][:, Q.astype(np.int64)].astype(object)
    m, n = B.shape
    for k in range(r):
        inv = pow(int(B[k, k]), p - 2, p)
        for i in range(k + 1, m):
            lik = (int(B[i, k]) * inv) % p
            B[i, k] = lik
            if lik:
                B[i, k + 1:] = (B[i, k + 1:] - lik * B[k, k + 1:]) % p
    out = np.array(B % p, dtype=np.uint32)
    out[r:, r:] = 0
    return out


def test_packed_output_is_lu_of_permuted_input(oracle_lib):
    O = oracle_lib
    for p, A in _cases(O, 11)[::3]:
        for thr in (1, 8):
            packed, P, Q, r = O.pluq_tile_recursive(p, A.copy(), thr)
            assert np.array_equal(_lu_from_pq(p, A, P, Q, r), packed)


def test_tile_rec_perms_edge_cases():
    import paper_1402_3501_b200 as G
    P, Q, r = G.tile_rec_perms(0, 5, 8, [], [])
    assert r == 0 and P.size == 0 and np.array_equal(Q, np.arange(5))
    P, Q, r = G.tile_rec_perms(7, 9, 2, [], [])
    assert r == 0 and np.array_equal(P, np.arange(7)) and np.array_equal(Q, np.arange(9))
    with pytest.raises(G.FfgError):
        G.tile_rec_perms(4, 4, 1, [0, 0], [1, 2])  # two pivots in one row: not a rank profile


@pytest.mark.parametrize("name", ["c4m", "c4"])
def test_config4_perms_full_size_from_profile(oracle_lib, name):
    """Config 4's rank profile is R's support; the reference's P/Q at full size (hashes) follow
    from it alone."""
    import paper_1402_3501_b200 as G
    c = json.load(open(FULL))[name]
    assert c["profile_is_R"]
    rows, cols = oracle_lib.lru_positions(c["n"], c["r"], c["p"], c["seed"])
    P, Q, r = G.tile_rec_perms(c["n"], c["n"], c["thr"], rows, cols)
    assert r == c["rank"]
    assert fnv_u32(P) == c["P_fnv"] and fnv_u32(Q) == c["Q_fnv"]
