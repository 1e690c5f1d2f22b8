"""A few back-to-back PLUQs on fresh seeded matrices (for env-driven diagnostics)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1402_3501_b200 as G  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
p = 131071
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = G.Context(0, stream=st.cuda_stream)
d = torch.empty((n, n), dtype=torch.int32, device="cuda")
for i in range(reps):
    G.random_mat_dev(p, d, 10 + i, ctx=ctx)
    ctx.synchronize()
    t = time.perf_counter()
    r = G.pluq_tile_recursive(p, d, 64, ctx=ctx)
    ctx.synchronize()
    print(f"pluq n={n} rank={r.rank} {1e3 * (time.perf_counter() - t):.2f} ms", flush=True)
