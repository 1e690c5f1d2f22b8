"""Small end-to-end runs (sanitizer-sized; compute-sanitizer is closed on this pool): the
speculative panel schedule (with column pivots), the exact recursion (rank deficient), the
byte entry, permutations and fgemm, all checked against the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import paper_1402_3501_b200 as G  # noqa: E402
from oracle import oracle as O  # noqa: E402
from test_gpu_parity import _zero_schur_pivot  # noqa: E402

p = 131071
ctx = G.Context(0)
cases = [("iid", O.random_mat(p, 300, 300, 1), 64), ("pivots", _zero_schur_pivot(O.random_mat(p, 260, 260, 2), p, [5, 70]), 64),
         ("lru", O.lru_matrix(200, 90, p, 7)[0], 16)]
for name, A, thr in cases:
    want = O.pluq_tile_recursive(p, A, thr)
    got = A.copy()
    res = G.pluq_tile_recursive(p, got, thr, ctx=ctx)
    assert res.rank == want[3] and np.array_equal(got, want[0]), name
    assert np.array_equal(res.P, want[1]) and np.array_equal(res.Q, want[2]), name
B8 = O.random_mat(251, 200, 200, 3)
want = O.pluq_tile_recursive(251, B8, 64)
g8 = B8.astype(np.uint8)
res = G.pluq_tile_recursive(251, g8, 64, ctx=ctx)
assert np.array_equal(g8.astype(np.uint32), want[0])
X, Y, Z = O.random_mat(p, 130, 140, 4), O.random_mat(p, 140, 150, 5), O.random_mat(p, 130, 150, 6)
out = Z.copy()
G.fgemm(p, p - 1, X, Y, 1, out, ctx=ctx)
assert np.array_equal(out, O.fgemm(p, p - 1, X, Y, 1, Z))
ctx.close()
print("sanitize_small ok")
