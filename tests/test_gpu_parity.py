"""GPU parity: the B200 library (through the C ABI) against the reference's
golden outputs (tests/golden/golden.json, produced by the reference itself)
and against the oracle, bit-exact, plus full-size property checks.
"""
import numpy as np
import pytest

from golden_util import fnv_u32, load, make_input
from verify import gemm_ok, pluq_ok

pytestmark = pytest.mark.gpu

GOLD = load()
CASES = [c for c in GOLD["cases"] if c.get("variant") != "as_written"]


def _ids(c):
    return f"{c['kind']}-p{c['p']}-{c.get('note', '')[:24]}"


def run_gpu(G, ctx, c):
    p = c["p"]
    if c["kind"] == "fgemm":
        A, B, C0 = make_input(c["A"]), make_input(c["B"]), make_input(c["C"])
        out = C0.copy()
        G.fgemm(p, c["alpha"], A, B, c["beta"], out, ctx=ctx)
        return {"out": out}
    if c["kind"] == "ftrsm":
        A, B = make_input(c["A"]), make_input(c["B"])
        out = B.copy()
        try:
            G.ftrsm(p, c["side"], c["uplo"], c["diag"], A, out, ctx=ctx)
        except G.SingularDiagonal as e:
            return {"error": "SingularDiagonal", "index": e.index}
        return {"out": out}
    A = make_input(c["A"]).copy()
    res = G.rr_base(p, A, ctx=ctx) if c["kind"] == "rr_base" else G.pluq_tile_recursive(p, A, c["thr"], ctx=ctx)
    return {"out": A, "P": res.P, "Q": res.Q, "rank": res.rank}


@pytest.mark.parametrize("case", CASES, ids=_ids)
def test_gpu_matches_reference_golden(gpu, oracle_lib, case):
    G, ctx = gpu
    got = run_gpu(G, ctx, case)
    if "error" in case:
        assert got.get("error") == case["error"] and got.get("index") == case["index"]
        return
    assert "error" not in got
    assert oracle_lib.checksum(got["out"], case["p"]) == case["out_ck"]
    if "out" in case:
        assert np.array_equal(got["out"].ravel(), np.array(case["out"], dtype=np.uint32))
    if case["kind"] in ("rr_base", "tile_rec"):
        assert got["rank"] == case["rank"]
        assert fnv_u32(got["P"]) == case["P_h"] and fnv_u32(got["Q"]) == case["Q_h"]


# ------------------------------------------------------------------ random + edge cases vs oracle
PRIMES = (2, 3, 5, 251, 65521, 131071, 16777213, 67108859)


@pytest.mark.parametrize("p", PRIMES)
def test_fgemm_random_vs_oracle(gpu, oracle_lib, p):
    G, ctx = gpu
    O = oracle_lib
    rng = np.random.default_rng(p)
    for t in range(8):
        m, k, n = (int(x) for x in rng.integers(1, 400, 3))
        A, B, C0 = O.random_mat(p, m, k, t), O.random_mat(p, k, n, t + 1), O.random_mat(p, m, n, t + 2)
        for alpha, beta in ((p - 1, 1), (1, 0), (3 % p, 2 % p), (0, 1), (0, 0)):
            want = O.fgemm(p, alpha, A, B, beta, C0)
            got = C0.copy()
            G.fgemm(p, alpha, A, B, beta, got, ctx=ctx)
            assert np.array_equal(want, got), (m, k, n, alpha, beta)


def test_fgemm_strided_views(gpu, oracle_lib):
    """Sub-views with lda > cols and unaligned offsets (tile_rec hands such views to fgemm)."""
    G, ctx = gpu
    O = oracle_lib
    p = 131071
    big = O.random_mat(p, 300, 301, 3)
    A = big[1:130, 3:200]
    B = big[5:202, 7:90]
    C = O.random_mat(p, 130, 300, 4)[1:130, 11:94]
    want = O.fgemm(p, p - 1, A, B, 1, C)
    got = C.copy()
    G.fgemm(p, p - 1, A, B, 1, got, ctx=ctx)
    assert np.array_equal(want, got)


def test_fgemm_empty_and_k0(gpu, oracle_lib):
    G, ctx = gpu
    O = oracle_lib
    p = 65521
    for (m, k, n) in ((0, 5, 3), (4, 0, 3), (4, 5, 0), (1, 1, 1)):
        A, B, C0 = O.random_mat(p, m, k, 1), O.random_mat(p, k, n, 2), O.random_mat(p, m, n, 3)
        for beta in (0, 1, 7):
            got = C0.copy()
            G.fgemm(p, 5, A, B, beta, got, ctx=ctx)
            assert np.array_equal(got, O.fgemm(p, 5, A, B, beta, C0))


def test_fgemm_kmax_chunking(gpu, oracle_lib):
    """K beyond the exact s32 bound: the kernel folds mod p once per kmax chunk (blas.hpp:85-88)."""
    G, ctx = gpu
    O = oracle_lib
    for p in (251, 131071):
        kmax = G.field_info(p)["kmax"]
        k = kmax + 300
        A, B, C0 = O.random_mat(p, 3, k, 1), O.random_mat(p, k, 5, 2), O.random_mat(p, 3, 5, 3)
        got = C0.copy()
        G.fgemm(p, p - 1, A, B, 1, got, ctx=ctx)
        assert np.array_equal(got, O.fgemm(p, p - 1, A, B, 1, C0))
        # all-(p-1) operands: the worst case for the accumulator bound
        A = np.full((2, k), p - 1, np.uint32)
        B = np.full((k, 3), p - 1, np.uint32)
        got = np.zeros((2, 3), np.uint32)
        G.fgemm(p, 1, A, B, 0, got, ctx=ctx)
        assert np.all(got == (k % p) * 1 % p)  # (p-1)^2 = 1 mod p


def test_ftrsm_errors(gpu):
    G, ctx = gpu
    U = np.array([[2, 1, 0], [0, 3, 1], [0, 0, 0]], np.uint32)
    B = np.ones((4, 3), np.uint32)
    with pytest.raises(G.SingularDiagonal) as ei:
        G.ftrsm(5, 1, 1, 1, U, B, ctx=ctx)
    assert ei.value.index == 2
    with pytest.raises(G.DimMismatch):
        G.ftrsm(5, 0, 0, 0, U, B, ctx=ctx)
    # empty B: no check, no error (blas.hpp:393)
    G.ftrsm(5, 1, 1, 1, np.zeros((0, 0), np.uint32), np.zeros((4, 0), np.uint32), ctx=ctx)


@pytest.mark.parametrize("p", (2, 5, 251, 131071))
def test_pluq_random_vs_oracle(gpu, oracle_lib, p):
    G, ctx = gpu
    O = oracle_lib
    rng = np.random.default_rng(p + 17)
    for t in range(10):
        m, n = int(rng.integers(1, 320)), int(rng.integers(1, 320))
        kind = t % 3
        if kind == 0:
            A = O.random_mat(p, m, n, 100 + t)
        else:
            N = max(m, n)
            M, _, _ = O.lru_matrix(N, N // (2 if kind == 1 else 3), p, t)
            A = M[:m, :n].copy()
        for thr in (1, 3, 8, 32, 100):
            if thr == 1 and max(m, n) > 160:
                continue
            a_o, P_o, Q_o, r_o = O.pluq_tile_recursive(p, A, thr)
            a_g = A.copy()
            res = G.pluq_tile_recursive(p, a_g, thr, ctx=ctx)
            assert r_o == res.rank
            assert np.array_equal(P_o, res.P) and np.array_equal(Q_o, res.Q)
            assert np.array_equal(a_o, a_g)


def test_pluq_edge_shapes(gpu, oracle_lib):
    G, ctx = gpu
    O = oracle_lib
    p = 131071
    for (m, n) in ((0, 5), (5, 0), (1, 1), (1, 300), (300, 1), (2, 257), (257, 2)):
        for fill in ("zero", "rand"):
            A = np.zeros((m, n), np.uint32) if fill == "zero" else O.random_mat(p, m, n, m * 7 + n)
            a_o, P_o, Q_o, r_o = O.pluq_tile_recursive(p, A, 8)
            a_g = A.copy()
            res = G.pluq_tile_recursive(p, a_g, 8, ctx=ctx)
            assert (r_o, P_o.tolist(), Q_o.tolist()) == (res.rank, res.P.tolist(), res.Q.tolist())
            assert np.array_equal(a_o, a_g)


def test_rr_base_large_block_global_path(gpu, oracle_lib):
    """Blocks larger than shared memory take the global-scratch path of the base kernel."""
    G, ctx = gpu
    O = oracle_lib
    for p in (5, 131071):
        M, _, _ = O.lru_matrix(400, 150, p, 3)
        A = M[:, :300].copy()
        a_o, P_o, Q_o, r_o = O.rr_base(p, A)
        a_g = A.copy()
        res = G.rr_base(p, a_g, ctx=ctx)
        assert r_o == res.rank and np.array_equal(P_o, res.P) and np.array_equal(Q_o, res.Q)
        assert np.array_equal(a_o, a_g)


# ------------------------------------------------------------------ device generators
def test_device_generators_match_cpu(gpu, oracle_lib):
    import torch
    G, ctx = gpu
    O = oracle_lib
    for p in (251, 131071):
        d = torch.empty((37, 53), dtype=torch.int32, device="cuda")
        G.random_mat_dev(p, d, 99, ctx=ctx)
        ctx.synchronize()
        assert np.array_equal(d.cpu().numpy().view(np.uint32), O.random_mat(p, 37, 53, 99))
        M = torch.empty((70, 70), dtype=torch.int32, device="cuda")
        rows, cols = G.lru_matrix_dev(p, M, 30, 5, ctx=ctx)
        ctx.synchronize()
        Mo, ro, co = O.lru_matrix(70, 30, p, 5)
        assert np.array_equal(M.cpu().numpy().view(np.uint32), Mo)
        assert np.array_equal(rows, ro) and np.array_equal(cols, co)


# ------------------------------------------------------------------ larger sizes: properties
def test_fgemm_8192_config2_freivalds(gpu, oracle_lib):
    """BASELINE config 2 shape (8192^3, GF(131071), C <- C - A*B) via random projections."""
    import torch
    G, ctx = gpu
    p, N = 131071, 8192
    dA = torch.empty((N, N), dtype=torch.int32, device="cuda")
    dB = torch.empty_like(dA)
    dC = torch.empty_like(dA)
    G.random_mat_dev(p, dA, 11, ctx=ctx)
    G.random_mat_dev(p, dB, 12, ctx=ctx)
    G.random_mat_dev(p, dC, 13, ctx=ctx)
    ctx.synchronize()
    A, B, C0 = (t.cpu().numpy().view(np.uint32) for t in (dA, dB, dC))
    G.fgemm(p, p - 1, dA, dB, 1, dC, ctx=ctx)
    ctx.synchronize()
    assert gemm_ok(p, p - 1, A, B, 1, C0, dC.cpu().numpy().view(np.uint32))


@pytest.mark.parametrize("p,n,thr,kind", [(131071, 2048, 64, "iid"), (131071, 4096, 64, "iid"),
                                          (251, 4096, 64, "iid"), (131071, 2048, 64, "lru"),
                                          (251, 1024, 8, "lru")])
def test_pluq_properties(gpu, oracle_lib, p, n, thr, kind):
    """Factorization identity P A Q = L U, rank, profiles; bit-exact vs the oracle where it is fast."""
    import torch
    G, ctx = gpu
    O = oracle_lib
    d = torch.empty((n, n), dtype=torch.int32, device="cuda")
    if kind == "iid":
        G.random_mat_dev(p, d, 1, ctx=ctx)
        rows = cols = None
    else:
        rows, cols = G.lru_matrix_dev(p, d, n // 2, 4, ctx=ctx)
    ctx.synchronize()
    A = d.cpu().numpy().view(np.uint32).copy()
    res = G.pluq_tile_recursive(p, d, thr, ctx=ctx)
    ctx.synchronize()
    packed = d.cpu().numpy().view(np.uint32)
    assert pluq_ok(p, A, packed, res.P, res.Q, res.rank)
    if kind == "lru":
        assert res.rank == n // 2
        assert set(zip(res.P[:res.rank].tolist(), res.Q[:res.rank].tolist())) == set(zip(rows.tolist(), cols.tolist()))
    if n <= 2048:
        a_o, P_o, Q_o, r_o = O.pluq_tile_recursive(p, A, thr)
        assert r_o == res.rank and np.array_equal(P_o, res.P) and np.array_equal(Q_o, res.Q)
        assert np.array_equal(a_o, packed)


def test_simt_path_still_exact(gpu, oracle_lib, monkeypatch):
    """The CUDA-core small-GEMM kernel (off by default, FFG_SIMT_MACS) stays bit-exact."""
    G, _ = gpu
    O = oracle_lib
    p = 131071
    monkeypatch.setenv("FFG_SIMT_MACS", str(1 << 24))
    ctx = G.Context(0)  # the threshold is read at context creation
    try:
        rng = np.random.default_rng(5)
        for (m, n, k) in ((1, 1, 1), (64, 64, 64), (100, 37, 250), (130, 70, 33)):
            A = O.random_mat(p, m, k, int(rng.integers(1 << 30)))
            B = O.random_mat(p, k, n, int(rng.integers(1 << 30)))
            C0 = O.random_mat(p, m, n, int(rng.integers(1 << 30)))
            want = O.fgemm(p, p - 1, A, B, 1, C0.copy())
            got = C0.copy()
            G.fgemm(p, p - 1, A, B, 1, got, ctx=ctx)
            assert np.array_equal(got, want)
    finally:
        ctx.close()
        monkeypatch.setenv("FFG_SIMT_MACS", "0")
        G.Context(0).close()  # restore the default threshold


@pytest.mark.parametrize("path", ["slab", "register", "smem"])
def test_every_base_kernel_matches_oracle(gpu, oracle_lib, path, monkeypatch):
    """The three base-case kernels (blocked slab, register right-looking, shared-memory
    right-looking) each reproduce rr_base bit for bit: full-rank, rank-deficient, ragged."""
    G, ctx = gpu
    O = oracle_lib
    env = {"slab": {}, "register": {"FFG_BASE_NO_SLAB": "1"}, "smem": {"FFG_BASE_SMEM": "1"}}[path]
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(404)
    for p in (2, 251, 131071):
        for t in range(12):
            m, n = int(rng.integers(1, 65)), int(rng.integers(1, 65))
            if t % 3 == 0:
                A = O.random_mat(p, m, n, 900 + t)
            elif t % 3 == 1:
                N = max(m, n)
                M, _, _ = O.lru_matrix(N, max(1, N // 3), p, t)
                A = M[:m, :n].copy()
            else:
                A = (O.random_mat(p, m, n, 700 + t) * (rng.random((m, n)) < 0.1)).astype(np.uint32)
            a_o, P_o, Q_o, r_o = O.rr_base(p, A)
            a_g = A.copy()
            res = G.rr_base(p, a_g, ctx=ctx)
            assert res.rank == r_o
            assert np.array_equal(res.P, P_o) and np.array_equal(res.Q, Q_o)
            assert np.array_equal(a_g, a_o)
            # the same block as the base case of a tile_rec call
            a_t = A.copy()
            res_t = G.pluq_tile_recursive(p, a_t, 64, ctx=ctx)
            assert res_t.rank == r_o and np.array_equal(a_t, a_o)


@pytest.mark.parametrize("case", ["full", "late_deficient", "zero_last_row"])
@pytest.mark.parametrize("n", [333, 1000])
def test_panel_mode_matches_oracle(gpu, oracle_lib, case, n, monkeypatch):
    """Speculative square runs take the panel schedule (every base case solves its whole right
    and bottom panels, every node updates [H | right panel] and the bottom panel): bit-exact
    against the oracle, and a guess that fails only at the last base cases (after the panel
    updates have overwritten the input) restores the HBM backup and reruns exactly."""
    G, ctx = gpu
    O = oracle_lib
    p = 131071
    A = O.random_mat(p, n, n, 77 + n)
    if case == "late_deficient":  # last column = sum of the first two: rank n-1
        A[:, n - 1] = ((A[:, 0].astype(np.uint64) + A[:, 1]) % p).astype(np.uint32)
    elif case == "zero_last_row":
        A[n - 1, :] = 0
    a_o, P_o, Q_o, r_o = O.pluq_tile_recursive(p, A, 16)
    outs = []
    for no_panel in ("0", "1"):
        monkeypatch.setenv("FFG_NO_PANEL", no_panel)
        import torch

        d = torch.from_numpy(A.view(np.int32).copy()).cuda()
        res = G.pluq_tile_recursive(p, d, 16, ctx=ctx)
        ctx.synchronize()
        got = d.cpu().numpy().view(np.uint32)
        assert res.rank == r_o
        assert np.array_equal(res.P, P_o) and np.array_equal(res.Q, Q_o)
        assert np.array_equal(got, a_o)
        outs.append(got)


@pytest.mark.parametrize("la", ["0", "128", "256", "1024"])
@pytest.mark.parametrize("n,thr", [(1000, 16), (2048, 64), (1537, 64)])
def test_panel_lookahead_pieces_match_oracle(gpu, oracle_lib, la, n, thr, monkeypatch):
    """Panel mode with the trailing update of every node >= FFG_PANEL_LA cut into look-ahead
    pieces (R's bands of doubling width, the first on the critical stream, the rest on a
    low-priority stream whose events R's recursion waits for): bit-exact against the oracle
    through the device entry and the streamed host entry."""
    import torch

    G, _ = gpu
    O = oracle_lib
    p = 131071
    A = O.random_mat(p, n, n, 9 + n)
    a_o, P_o, Q_o, r_o = O.pluq_tile_recursive(p, A, thr)
    monkeypatch.setenv("FFG_PANEL_LA", la)
    ctx = G.Context(0)
    try:
        d = torch.from_numpy(A.view(np.int32).copy()).cuda()
        res = G.pluq_tile_recursive(p, d, thr, ctx=ctx)
        ctx.synchronize()
        assert res.rank == r_o
        assert np.array_equal(res.P, P_o) and np.array_equal(res.Q, Q_o)
        assert np.array_equal(d.cpu().numpy().view(np.uint32), a_o)
        h = A.copy()
        res = G.pluq_tile_recursive(p, h, thr, ctx=ctx)
        assert res.rank == r_o and np.array_equal(h, a_o)
        assert np.array_equal(res.P, P_o) and np.array_equal(res.Q, Q_o)
    finally:
        ctx.close()


@pytest.mark.parametrize("la,end", [("256", "0.5"), ("512", "1"), ("1024", "0.5")])
@pytest.mark.parametrize("n,pivots", [(2048, False), (1537, False), (2048, True)])
def test_host_entry_lookahead_matches_oracle(gpu, oracle_lib, la, end, n, pivots, monkeypatch):
    """Streamed host entry with look-ahead pieces in the nodes of >= FFG_HOST_LA ending before
    FFG_HOST_LA_END * n (each piece waits only for the bands it touches): bit-exact against the
    oracle, column pivots inside and at the end of blocks included."""
    G, _ = gpu
    O = oracle_lib
    p, thr = 131071, 64
    A = O.random_mat(p, n, n, 31 + n)
    if pivots:
        A = _zero_schur_pivot(A, p, [70, 300, 700, 1100, 1400])
    a_o, P_o, Q_o, r_o = O.pluq_tile_recursive(p, A, thr)
    monkeypatch.setenv("FFG_HOST_LA", la)
    monkeypatch.setenv("FFG_HOST_LA_END", end)
    monkeypatch.setenv("FFG_BAND_MAX", "256")
    ctx = G.Context(0)
    try:
        h = A.copy()
        res = G.pluq_tile_recursive(p, h, thr, ctx=ctx)
        assert res.rank == r_o and np.array_equal(h, a_o)
        assert np.array_equal(res.P, P_o) and np.array_equal(res.Q, Q_o)
    finally:
        ctx.close()


def _zero_schur_pivot(A, p, ks, seed=5):
    """Row k's first k+1 entries become a combination of rows 0..k-1 (the rest stays random): the
    Schur diagonal at k is zero and row k pivots on a later column -- a column rotation inside its
    base block when k % 64 < 63, a rank-deficient block when k is its last row."""
    rng = np.random.default_rng(seed)
    A = A.copy()
    for k in ks:
        c = rng.integers(0, p, size=k, dtype=np.uint64)
        comb = np.zeros(k + 1, np.uint64)
        for i in range(k):
            comb = (comb + c[i] * A[i, :k + 1].astype(np.uint64)) % p
        A[k, :k + 1] = comb.astype(np.uint32)
    return A


@pytest.mark.parametrize("ks", [[0], [100], [127], [100, 700], [5, 64, 65, 300, 1000]])
@pytest.mark.parametrize("n", [1000, 2048])
def test_panel_column_pivots_match_oracle(gpu, oracle_lib, ks, n):
    """Speculative panel runs guess only full rank: a zero Schur diagonal inside a base block
    pivots on a later column (rr_base's rotation), the column pivots are gathered into the bottom
    panel, applied to the rows above the block at the end, and returned in Q -- bit-exact against
    the oracle through both entries; a rank-deficient block (k = 127) falls back to the exact path."""
    import torch

    G, _ = gpu
    O = oracle_lib
    p = 131071
    ks = [k for k in ks if k < n]
    A = _zero_schur_pivot(O.random_mat(p, n, n, 3 + n), p, ks)
    a_o, P_o, Q_o, r_o = O.pluq_tile_recursive(p, A, 64)
    for entry in ("dev", "host"):
        ctx = G.Context(0)
        try:
            if entry == "dev":
                d = torch.from_numpy(A.view(np.int32).copy()).cuda()
                res = G.pluq_tile_recursive(p, d, 64, ctx=ctx)
                ctx.synchronize()
                got = d.cpu().numpy().view(np.uint32)
            else:
                got = A.copy()
                res = G.pluq_tile_recursive(p, got, 64, ctx=ctx)
            assert res.rank == r_o
            assert np.array_equal(res.P, P_o) and np.array_equal(res.Q, Q_o), entry
            assert np.array_equal(got, a_o), entry
        finally:
            ctx.close()


@pytest.mark.parametrize("p,m,n", [(251, 300, 300), (251, 1000, 1000), (251, 333, 700), (2, 257, 190), (5, 64, 64),
                                   (251, 0, 5)])
def test_u8_host_entry_matches_oracle(gpu, oracle_lib, p, m, n):
    """Byte storage (p <= 256, BASELINE config 5's "stored as uint8"): the same outputs as the
    oracle on the u32 matrix, with a padded leading dimension left untouched."""
    G, ctx = gpu
    O = oracle_lib
    A = O.random_mat(p, m, n, 11 + m + n) if m and n else np.zeros((m, n), np.uint32)
    a_o, P_o, Q_o, r_o = O.pluq_tile_recursive(p, A, 64)
    buf = np.full((m, n + 9), 0xAB, np.uint8)
    buf[:, :n] = A.astype(np.uint8)
    view = buf[:, :n]
    res = G.pluq_tile_recursive(p, view, 64, ctx=ctx)
    assert res.rank == r_o
    assert np.array_equal(res.P, P_o[:m]) and np.array_equal(res.Q, Q_o[:n])
    assert np.array_equal(view.astype(np.uint32), a_o)
    assert np.all(buf[:, n:] == 0xAB)


def test_u8_host_entry_rejects_large_p(gpu):
    G, ctx = gpu
    with pytest.raises(Exception):
        G.pluq_tile_recursive(131071, np.zeros((4, 4), np.uint8), 64, ctx=ctx)


@pytest.mark.parametrize("n,thr,seed", [(1100, 16, 1), (1100, 16, 2), (1300, 16, 3)])
def test_node_level_speculation_small_field(gpu, oracle_lib, n, thr, seed):
    """GF(251) with many blocks: the whole-matrix guess is skipped, square nodes of the exact
    recursion try the speculative panel schedule on their own (some fail and rerun exactly)
    -- bit-exact against the oracle."""
    import torch

    G, _ = gpu
    O = oracle_lib
    p = 251
    A = O.random_mat(p, n, n, seed)
    a_o, P_o, Q_o, r_o = O.pluq_tile_recursive(p, A, thr)
    ctx = G.Context(0)
    try:
        d = torch.from_numpy(A.view(np.int32).copy()).cuda()
        res = G.pluq_tile_recursive(p, d, thr, ctx=ctx)
        ctx.synchronize()
        assert res.rank == r_o
        assert np.array_equal(res.P, P_o) and np.array_equal(res.Q, Q_o)
        assert np.array_equal(d.cpu().numpy().view(np.uint32), a_o)
    finally:
        ctx.close()


@pytest.mark.slow
def test_node_level_speculation_matches_exact_at_config5_blocks(gpu, monkeypatch):
    """n = 4096, GF(251), thr 64 (config 5's block size): node-level speculation on vs off,
    bit for bit."""
    import torch

    G, _ = gpu
    p, n = 251, 4096
    outs = []
    for ns in ("1024", "0"):
        monkeypatch.setenv("FFG_NODE_SPEC", ns)
        ctx = G.Context(0)
        try:
            d = torch.empty((n, n), dtype=torch.int32, device="cuda")
            G.random_mat_dev(p, d, 5, ctx=ctx)
            res = G.pluq_tile_recursive(p, d, 64, ctx=ctx)
            ctx.synchronize()
            outs.append((res.rank, res.P.copy(), res.Q.copy(), d.cpu().numpy().copy()))
        finally:
            ctx.close()
    assert outs[0][0] == outs[1][0]
    for i in (1, 2, 3):
        assert np.array_equal(outs[0][i], outs[1][i])


@pytest.mark.parametrize("trial", range(40))
def test_panel_schedule_random_sweep(gpu, oracle_lib, trial):
    """Random square sizes, thresholds (odd leaf sizes, two-leaf nodes of unequal leaves),
    primes up to 2^26 and injected zero Schur diagonals through the speculative schedules
    (device and host entries), against the oracle."""
    import torch

    G, _ = gpu
    O = oracle_lib
    rng = np.random.default_rng(1000 + trial)
    p = int(rng.choice([65521, 131071, 16777213, 67108859]))
    thr = int(rng.choice([8, 16, 33, 48, 64]))
    n = int(rng.integers(150, 900))
    ks = sorted(set(int(k) for k in rng.integers(0, n - 1, size=int(rng.integers(0, 4)))))
    A = _zero_schur_pivot(O.random_mat(p, n, n, 77 * trial + 1), p, ks)
    a_o, P_o, Q_o, r_o = O.pluq_tile_recursive(p, A, thr)
    ctx = G.Context(0)
    try:
        d = torch.from_numpy(A.view(np.int32).copy()).cuda()
        res = G.pluq_tile_recursive(p, d, thr, ctx=ctx)
        ctx.synchronize()
        assert res.rank == r_o, (p, thr, n, ks)
        assert np.array_equal(res.P, P_o) and np.array_equal(res.Q, Q_o), (p, thr, n, ks)
        assert np.array_equal(d.cpu().numpy().view(np.uint32), a_o), (p, thr, n, ks)
        h = A.copy()
        res = G.pluq_tile_recursive(p, h, thr, ctx=ctx)
        assert res.rank == r_o and np.array_equal(h, a_o), (p, thr, n, ks)
        assert np.array_equal(res.P, P_o) and np.array_equal(res.Q, Q_o), (p, thr, n, ks)
    finally:
        ctx.close()


@pytest.mark.parametrize("knobs", [{"FFG_PROG_MIN": "256"}, {"FFG_PROG_MIN": "512", "FFG_PROG_CHUNKS": "2"},
                                   {"FFG_CORNER_MAX": "0"}, {"FFG_NO_CORNER": "1"}, {"FFG_APPLY_CTAS": "7"}])
def test_panel_schedule_variants_match_oracle(gpu, oracle_lib, knobs, monkeypatch):
    """The panel schedule's off-by-default variants (progressive K-chunked trailing updates,
    no corner deferral, no two-leaf corner, capped strip-looping applies) stay bit-exact."""
    import torch

    G, _ = gpu
    O = oracle_lib
    p, n = 131071, 1300
    A = _zero_schur_pivot(O.random_mat(p, n, n, 606), p, [40, 700])
    a_o, P_o, Q_o, r_o = O.pluq_tile_recursive(p, A, 64)
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    ctx = G.Context(0)
    try:
        d = torch.from_numpy(A.view(np.int32).copy()).cuda()
        res = G.pluq_tile_recursive(p, d, 64, ctx=ctx)
        ctx.synchronize()
        assert res.rank == r_o
        assert np.array_equal(res.P, P_o) and np.array_equal(res.Q, Q_o)
        assert np.array_equal(d.cpu().numpy().view(np.uint32), a_o)
    finally:
        ctx.close()


@pytest.mark.parametrize("n,thr,seed,lead", [(1100, 16, 4, 0), (1300, 16, 5, 7), (1200, 8, 6, 3)])
def test_small_field_host_pipeline_matches_oracle(gpu, oracle_lib, n, thr, seed, lead):
    """GF(251) with many blocks through the host entries: u32 (the pipelined exact recursion:
    spine uploads, right-spine early downloads) and bytes (widened / narrowed in HBM, node-level
    speculation inside) -- bit-exact against the oracle, padding untouched."""
    G, _ = gpu
    O = oracle_lib
    p = 251
    A = O.random_mat(p, n, n, seed)
    a_o, P_o, Q_o, r_o = O.pluq_tile_recursive(p, A, thr)
    ctx = G.Context(0)
    try:
        buf = np.full((n, n + lead), 0xCD, np.uint32)
        buf[:, :n] = A
        res = G.pluq_tile_recursive(p, buf[:, :n], thr, ctx=ctx)
        assert res.rank == r_o and np.array_equal(buf[:, :n], a_o)
        assert np.array_equal(res.P, P_o) and np.array_equal(res.Q, Q_o)
        assert np.all(buf[:, n:] == 0xCD)
        b8 = np.full((n, n + lead), 0xEE, np.uint8)
        b8[:, :n] = A.astype(np.uint8)
        res = G.pluq_tile_recursive(p, b8[:, :n], thr, ctx=ctx)
        assert res.rank == r_o and np.array_equal(b8[:, :n].astype(np.uint32), a_o)
        assert np.array_equal(res.P, P_o) and np.array_equal(res.Q, Q_o)
        assert np.all(b8[:, n:] == 0xEE)
    finally:
        ctx.close()
