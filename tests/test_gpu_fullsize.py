"""Full-size bit-exact parity at the BASELINE configurations, against the REFERENCE.

tests/golden/full_size.json holds, for configs 2-5, the input checksum and the
reference's own outputs at full size -- packed L\\U (or C) checksum
(matrix.hpp:53-68), FNV hashes of P and Q (PermSeq::to_array(), perm.hpp:88-95)
and the rank -- produced by scripts/make_golden_full.py from oracle/_ref (the
reference headers compiled, rankrev.hpp:146 temp-J fix).  Here the same inputs
are regenerated on the device from their seeds (ffg_random_mat_dev = the
reference's random_mat; ffg_lru_matrix_dev = the config-4 generator), their
checksums checked against the fixture, factored through the C ABI (device entry
and host entry) and the four hashes compared.  Nothing here reads /root/reference.
"""
import json
import os

import numpy as np
import pytest

from golden_util import fnv_u32

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

FULL = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "full_size.json")
GOLD = json.load(open(FULL)) if os.path.exists(FULL) else {}


def _case(name):
    if name not in GOLD:
        pytest.fail(f"{name} missing from {FULL} (run scripts/make_golden_full.py)")
    return GOLD[name]


def _input_dev(G, ctx, c):
    import torch
    n, p = c["n"], c["p"]
    d = torch.empty((n, n), dtype=torch.int32, device="cuda")
    if c["gen"] == "iid":
        G.random_mat_dev(p, d, c["seed"], ctx=ctx)
        rc = None
    else:
        rc = G.lru_matrix_dev(p, d, c["r"], c["seed"], ctx=ctx)
    ctx.synchronize()
    return d, rc


def _check(O, c, packed, res):
    assert res.rank == c["rank"], (res.rank, c["rank"])
    assert fnv_u32(res.P) == c["P_fnv"], "P differs from the reference"
    assert fnv_u32(res.Q) == c["Q_fnv"], "Q differs from the reference"
    assert O.checksum(packed, c["p"]) == c["out_ck"], "packed L\\U differs from the reference"


PLUQ_CASES = ["c3", "c4", "c5", "c4m", "c5m"]


@pytest.mark.parametrize("name", PLUQ_CASES)
def test_pluq_device_entry_matches_reference_full_size(gpu, oracle_lib, name):
    """ffg_pluq_tile_recursive_dev on the resident BASELINE input (the bench's path)."""
    G, ctx = gpu
    O = oracle_lib
    c = _case(name)
    d, rc = _input_dev(G, ctx, c)
    assert O.checksum(d.cpu().numpy().view(np.uint32), c["p"]) == c["in_ck"], "input generator drifted"
    res = G.pluq_tile_recursive(c["p"], d, c["thr"], ctx=ctx)
    ctx.synchronize()
    packed = d.cpu().numpy().view(np.uint32)
    del d
    _check(O, c, packed, res)
    if rc is not None:  # L*R*U: the rank profile matrix is R
        rows, cols = rc
        assert set(zip(res.P[:res.rank].tolist(), res.Q[:res.rank].tolist())) == set(zip(rows.tolist(),
                                                                                          cols.tolist()))


@pytest.mark.parametrize("name", PLUQ_CASES)
def test_pluq_host_entry_matches_reference_full_size(gpu, oracle_lib, name):
    """ffg_pluq_tile_recursive (host buffers: the drop-in for the reference call), and for
    p <= 256 also the byte-storage entry ffg_pluq_tile_recursive_u8."""
    import torch
    G, ctx = gpu
    O = oracle_lib
    c = _case(name)
    d, _ = _input_dev(G, ctx, c)
    A = d.cpu().numpy().view(np.uint32).copy()
    A8 = d.to(torch.uint8).cpu().numpy() if c["p"] <= 256 else None
    del d
    torch.cuda.empty_cache()
    assert O.checksum(A, c["p"]) == c["in_ck"]
    res = G.pluq_tile_recursive(c["p"], A, c["thr"], ctx=ctx)
    _check(O, c, A, res)
    if A8 is not None:
        res8 = G.pluq_tile_recursive(c["p"], A8, c["thr"], ctx=ctx)
        _check(O, c, A8.astype(np.uint32), res8)


def test_fgemm_config2_matches_reference_full_size(gpu, oracle_lib):
    """BASELINE config 2: C <- C - A*B mod 131071 at 8192^3, checksum of C vs the reference's pfgemm,
    through the device entry and the host entry."""
    import torch
    G, ctx = gpu
    O = oracle_lib
    c = _case("c2")
    n, p = c["n"], c["p"]
    mats = []
    for s in c["seeds"]:
        t = torch.empty((n, n), dtype=torch.int32, device="cuda")
        G.random_mat_dev(p, t, s, ctx=ctx)
        mats.append(t)
    ctx.synchronize()
    host = [t.cpu().numpy().view(np.uint32).copy() for t in mats]
    assert [O.checksum(h, p) for h in host] == c["in_ck"]
    dA, dB, dC = mats
    G.fgemm(p, c["alpha"], dA, dB, c["beta"], dC, ctx=ctx)
    ctx.synchronize()
    assert O.checksum(dC.cpu().numpy().view(np.uint32), p) == c["out_ck"]
    del mats, dA, dB, dC
    torch.cuda.empty_cache()
    A, B, Cm = host
    G.fgemm(p, c["alpha"], A, B, c["beta"], Cm, ctx=ctx)
    assert O.checksum(Cm, p) == c["out_ck"]
