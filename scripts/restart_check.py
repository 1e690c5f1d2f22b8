"""Small-field PLUQs through the speculative base kernel (column-pivot restarts) vs the oracle."""
import os
import sys
import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1402_3501_b200 as G  # noqa: E402
from oracle import build_ref  # noqa: E402
build_ref.build_oracle()
from oracle import oracle as O  # noqa: E402

ctx = G.Context(0)
for p, n, seed in [(131071, 64, 1), (5, 64, 1), (251, 64, 2), (251, 128, 3), (3, 128, 4), (251, 512, 5), (251, 2048, 6)]:
    A = O.random_mat(p, n, n, seed)
    want = O.pluq_tile_recursive(p, A, 64)
    d = torch.from_numpy(A.view(np.int32).copy()).cuda()
    print("run", p, n, seed, flush=True)
    res = G.pluq_tile_recursive(p, d, 64, ctx=ctx)
    ctx.synchronize()
    got = d.cpu().numpy().view(np.uint32)
    ok = res.rank == want[3] and np.array_equal(res.P, want[1]) and np.array_equal(res.Q, want[2]) and np.array_equal(got, want[0])
    print(p, n, seed, "rank", res.rank, want[3], "ok" if ok else "MISMATCH", flush=True)
