"""CPU: the oracle restatement (oracle/oracle.c) against the reference's own outputs.

tests/golden/golden.json was produced by running the reference headers
compiled unchanged (oracle/_ref, scripts/make_golden.py).  Each case is
regenerated from its seed here, its input checksum checked, then run through
the ORACLE and compared with the reference's output hashes.  This is what
pins the oracle; the GPU tests then compare against both.
"""
import numpy as np
import pytest

from golden_util import fnv_u32, load, make_input

GOLD = load()
CASES = GOLD["cases"]


def _ids(c):
    return f"{c['kind']}-p{c['p']}-{c.get('note', '')[:30]}"


def _check_inputs(O, c, mats):
    want = c["in_ck"] if isinstance(c["in_ck"], list) else [c["in_ck"]]
    got = [O.checksum(a, c["p"]) for a in mats]
    assert got == want, "regenerated input differs from the reference's"


def run_oracle(O, c):
    p = c["p"]
    if c["kind"] == "fgemm":
        A, B, C0 = make_input(c["A"]), make_input(c["B"]), make_input(c["C"])
        _check_inputs(O, c, [A, B, C0])
        out = O.fgemm(p, c["alpha"], A, B, c["beta"], C0, acc_bits=c.get("acc_bits", 53))
        return {"out_ck": O.checksum(out, p), "out": out}
    if c["kind"] == "ftrsm":
        A, B = make_input(c["A"]), make_input(c["B"])
        _check_inputs(O, c, [A, B])
        try:
            out = O.ftrsm(p, c["side"], c["uplo"], c["diag"], A, B)
        except O.OracleError as e:
            return {"error": O.ERRORS[e.code], "index": e.index}
        return {"out_ck": O.checksum(out, p), "out": out}
    A = make_input(c["A"])
    _check_inputs(O, c, [A])
    if c["kind"] == "rr_base":
        a, P, Q, r = O.rr_base(p, A)
    else:
        a, P, Q, r = O.pluq_tile_recursive(p, A, c["thr"], fix_j=c.get("variant") != "as_written")
    return {"out_ck": O.checksum(a, p), "P_h": fnv_u32(P), "Q_h": fnv_u32(Q), "rank": r, "out": a, "P": P, "Q": Q}


def compare(c, got):
    if "error" in c:
        assert got.get("error") == c["error"] and got.get("index") == c["index"]
        return
    assert "error" not in got, got
    assert got["out_ck"] == c["out_ck"]
    if "out" in c:
        assert np.array_equal(np.asarray(got["out"]).ravel(), np.array(c["out"], dtype=np.uint32))
    if c["kind"] in ("rr_base", "tile_rec"):
        assert got["rank"] == c["rank"]
        assert got["P_h"] == c["P_h"] and got["Q_h"] == c["Q_h"]


FAST = [c for c in CASES if not (c["kind"] == "tile_rec" and c["A"].get("m", 0) * c["A"].get("n", 0) > 300 * 300)]
BIG = [c for c in CASES if c not in FAST]


@pytest.mark.parametrize("case", FAST, ids=_ids)
def test_oracle_matches_reference(oracle_lib, case):
    compare(case, run_oracle(oracle_lib, case))


@pytest.mark.parametrize("case", BIG, ids=_ids)
def test_oracle_matches_reference_n1024(oracle_lib, case):
    compare(case, run_oracle(oracle_lib, case))


def test_golden_has_reference_known_answers():
    notes = {c.get("note", "") for c in CASES}
    for must in ("blas_test.cpp:9-16 hand computed", "rankrev_test.cpp:61-71 rank-2 example",
                 "blas_test.cpp:223-233 SingularDiagonal index 1", "BASELINE config 1: n=1024 iid GF(131071)"):
        assert must in notes
    hand = next(c for c in CASES if c["note"] == "blas_test.cpp:9-16 hand computed")
    assert hand["out"] == [2, 1, 4, 3]  # blas_test.cpp:15
    rank2 = next(c for c in CASES if c["note"] == "rankrev_test.cpp:61-71 rank-2 example")
    assert rank2["rank"] == 2 and sorted(rank2["P"][:2]) == [0, 2] and sorted(rank2["Q"][:2]) == [0, 1]


def test_as_written_reference_bug_is_documented():
    """rankrev.hpp:146: the unmodified reference does not reconstruct L*R*U inputs."""
    aw = [c for c in CASES if c.get("variant") == "as_written"]
    assert aw and sum(1 for c in aw if c["reconstructs"] is False) > len(aw) // 2


def test_rr_base_equals_slab_iterative(oracle_lib):
    """The GPU base case relies on rr_base == slab-iterative for every slab size (rankrev.hpp:244-282)."""
    O = oracle_lib
    rng = np.random.default_rng(3)
    for t in range(40):
        m, n = int(rng.integers(1, 90)), int(rng.integers(1, 30))
        N = max(m, n)
        M, _, _ = O.lru_matrix(N, N // 2, 131071 if t % 2 else 5, t)
        A = M[:m, :n].copy()
        p = 131071 if t % 2 else 5
        want = O.rr_base(p, A)
        for k in (1, 3, 8, 32):
            got = O.pluq_slab_iterative(p, A, k)
            assert all(np.array_equal(x, y) for x, y in zip(want[:3], got[:3])) and want[3] == got[3]


def test_lru_profiles_are_R(oracle_lib):
    """Config-4 known answer: the rank profile matrix of L*R*U is R (size-independent)."""
    O = oracle_lib
    for p, n in ((251, 40), (131071, 64)):
        M, rows, cols = O.lru_matrix(n, n // 2, p, 9)
        a, P, Q, r = O.pluq_tile_recursive(p, M, 4)
        assert r == n // 2
        assert np.array_equal(np.sort(P[:r]), np.sort(rows)) and np.array_equal(np.sort(Q[:r]), np.sort(cols))
        pairs = set(zip(P[:r].tolist(), Q[:r].tolist()))
        assert pairs == set(zip(rows.tolist(), cols.tolist()))
        assert np.array_equal(O.reconstruct(p, a, P, Q, r), M)
