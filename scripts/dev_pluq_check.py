"""Dev check: GPU ftrsm / rr_base / pluq vs oracle."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
import paper_1402_3501_b200 as G
ctx = G.Context(0)
rng = np.random.default_rng(0)
def same(a, b): return all(np.array_equal(x, y) for x, y in zip(a, b))
bad = 0; n = 0
for p in [2, 5, 251, 65521, 131071]:
    for t in range(10):
        m = int(rng.integers(1, 300)); w = int(rng.integers(1, 300))
        T = O.random_mat(p, m, m, t); T[np.arange(m), np.arange(m)] = np.maximum(T[np.arange(m), np.arange(m)], 1)
        B = O.random_mat(p, m, w, t + 1); Bt = O.random_mat(p, w, m, t + 2)
        for uplo in (0, 1):
            for diag in (0, 1):
                n += 2
                want = O.ftrsm(p, 0, uplo, diag, T, B); got = B.copy(); G.ftrsm(p, 0, uplo, diag, T, got, ctx=ctx)
                if not np.array_equal(want, got): bad += 1; print("trsm L mismatch", p, m, w, uplo, diag)
                want = O.ftrsm(p, 1, uplo, diag, T, Bt); got = Bt.copy(); G.ftrsm(p, 1, uplo, diag, T, got, ctx=ctx)
                if not np.array_equal(want, got): bad += 1; print("trsm R mismatch", p, m, w, uplo, diag)
print("trsm cases", n, "bad", bad, flush=True)
ref = O.Ref(True) if os.path.exists(os.path.join('oracle','_ref','libffref_fixed.so')) else None
bad = 0; n = 0
for p in [2, 3, 5, 251, 131071]:
    for t in range(12):
        m = int(rng.integers(1, 120)); w = int(rng.integers(1, 120))
        if t % 3 == 0: A = O.random_mat(p, m, w, 77 + t)
        else:
            N = max(m, w); M_, _, _ = O.lru_matrix(N, N // 2, p, t); A = M_[:m, :w].copy()
        a_o, P_o, Q_o, r_o = O.rr_base(p, A)
        a_g = A.copy(); res = G.rr_base(p, a_g, ctx=ctx); n += 1
        if not (np.array_equal(a_o, a_g) and np.array_equal(P_o, res.P) and np.array_equal(Q_o, res.Q) and r_o == res.rank):
            bad += 1; print("rr_base mismatch", p, m, w, r_o, res.rank)
print("rr_base cases", n, "bad", bad, flush=True)
bad = 0; n = 0
for p in [2, 3, 251, 65521, 131071]:
    for t in range(10):
        m = int(rng.integers(1, 400)); w = int(rng.integers(1, 400))
        kind = t % 3
        if kind == 0: A = O.random_mat(p, m, w, 99 + t)
        elif kind == 1:
            N = max(m, w); M_, _, _ = O.lru_matrix(N, N // 2, p, t); A = M_[:m, :w].copy()
        else:
            N = max(m, w); M_, _, _ = O.lru_matrix(N, N // 3, p, t + 50); A = M_[:m, :w].copy()
        for thr in [1, 4, 16, 64]:
            if thr == 1 and max(m, w) > 150: continue
            a_o, P_o, Q_o, r_o = O.pluq_tile_recursive(p, A, thr, True)
            a_g = A.copy(); res = G.pluq_tile_recursive(p, a_g, thr, ctx=ctx); n += 1
            if not (np.array_equal(a_o, a_g) and np.array_equal(P_o, res.P) and np.array_equal(Q_o, res.Q) and r_o == res.rank):
                bad += 1; print("pluq mismatch", p, m, w, thr, kind, r_o, res.rank, np.array_equal(P_o, res.P), np.array_equal(Q_o, res.Q), (a_o != a_g).sum())
print("pluq cases", n, "bad", bad, flush=True)
for p, N, thr in [(131071, 2048, 64), (131071, 4096, 64), (251, 4096, 64)]:
    A = O.random_mat(p, N, N, 5)
    t0 = time.time(); a_g = A.copy(); res = G.pluq_tile_recursive(p, a_g, thr, ctx=ctx); t1 = time.time()
    a_g = A.copy(); t2 = time.time(); res = G.pluq_tile_recursive(p, a_g, thr, ctx=ctx); t3 = time.time()
    print(f"p={p} N={N} thr={thr}: rank {res.rank}, first {t1-t0:.3f}s, second {t3-t2:.3f}s (host API incl copies)", flush=True)
    if N <= 2048:
        a_o, P_o, Q_o, r_o = O.pluq_tile_recursive(p, A, thr, True)
        print("  bit-exact:", np.array_equal(a_o, a_g) and np.array_equal(P_o, res.P) and np.array_equal(Q_o, res.Q))
