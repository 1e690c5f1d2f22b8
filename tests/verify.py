"""Size-independent checks for full-size parity (numpy, int64, chunked).

Freivalds-style random projections: a wrong answer passes with probability
<= 1/p per projection; two projections are used.
"""
from __future__ import annotations

import numpy as np

CH = 1024


def _matvec(A, x, p):
    out = np.empty(A.shape[0], np.int64)
    for i in range(0, A.shape[0], CH):
        out[i:i + CH] = (A[i:i + CH].astype(np.int64) @ x) % p
    return out


def gemm_ok(p, alpha, A, B, beta, C0, C1, reps=2, seed=0):
    """C1 == alpha*A*B + beta*C0 mod p."""
    rng = np.random.default_rng(seed)
    for _ in range(reps):
        x = rng.integers(0, p, C1.shape[1]).astype(np.int64)
        want = (alpha * _matvec(A, _matvec(B, x, p), p) + beta * _matvec(C0, x, p)) % p
        if not np.array_equal(want, _matvec(C1, x, p)):
            return False
    return True


def pluq_ok(p, A, packed, P, Q, r, reps=2, seed=0):
    """P A Q == L U for the packed factors (oracle.hpp:198-215 semantics) and a zero trailing block."""
    m, n = A.shape
    rng = np.random.default_rng(seed)
    P = np.asarray(P, np.int64)
    Q = np.asarray(Q, np.int64)
    if sorted(P.tolist()) != list(range(m)) or sorted(Q.tolist()) != list(range(n)):
        return False
    for _ in range(reps):
        x = rng.integers(0, p, n).astype(np.int64)
        # U x (U = rows [0, r) of packed, upper incl. diagonal)
        ux = np.zeros(r, np.int64)
        for i in range(0, r, CH):
            blk = packed[i:min(i + CH, r)].astype(np.int64)
            rows = np.arange(i, min(i + CH, r))
            mask = np.arange(n)[None, :] >= rows[:, None]
            ux[i:i + CH] = ((blk * mask) @ x) % p
        # L (U x): L[t][k] = packed[t][k] for k < min(t, r), 1 on the diagonal for t < r
        y1 = np.zeros(m, np.int64)
        for i in range(0, m, CH):
            blk = packed[i:i + CH, :r].astype(np.int64)
            rows = np.arange(i, min(i + CH, m))
            mask = np.arange(r)[None, :] < rows[:, None]
            y1[i:i + CH] = ((blk * mask) @ ux) % p
        diag = np.arange(min(m, r))
        y1[diag] = (y1[diag] + ux[diag]) % p
        # (P A Q) x = (A z)[P] with z[Q[u]] = x[u]
        z = np.empty(n, np.int64)
        z[Q] = x
        y2 = _matvec(A, z, p)[P]
        if not np.array_equal(y1, y2):
            return False
    # trailing block rows r.., cols r.. must be zero (rankrev_test.cpp:275-286)
    if r < m and r < n:
        for i in range(r, m, CH):
            if np.any(packed[i:i + CH, r:]):
                return False
    return True
