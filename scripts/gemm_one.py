"""One small fgemm shape, repeated (for ncu).  python scripts/gemm_one.py M N K [compact]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1402_3501_b200 as G  # noqa: E402

m, n, k = (int(x) for x in sys.argv[1:4])
compact = len(sys.argv) > 4 and sys.argv[4] == "compact"
p = int(os.environ.get("P", "131071"))
ctx = G.Context(0)
if compact:
    A = torch.empty((m, k), dtype=torch.int32, device="cuda")
    B = torch.empty((k, n), dtype=torch.int32, device="cuda")
    C_ = torch.empty((m, n), dtype=torch.int32, device="cuda")
    for i, t in enumerate((A, B, C_)):
        G.random_mat_dev(p, t, i + 1, ctx=ctx)
else:
    NB = int(os.environ.get("BIG", "16384"))
    big = torch.empty((NB, NB), dtype=torch.int32, device="cuda")
    G.random_mat_dev(p, big, 5, ctx=ctx)
    A, B, C_ = big[:m, :k], big[:k, 8192:8192 + n], big[8192:8192 + m, 4096:4096 + n]
for _ in range(10):
    G.fgemm(p, p - 1, A, B, 1, C_, ctx=ctx)
ctx.synchronize()
