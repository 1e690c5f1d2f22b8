"""One warm + one measured fgemm (BASELINE config 2: 8192^3, C <- C - A*B mod 131071) for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_3501_b200 as G
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
p = 131071
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
ctx = G.Context(0, stream=st.cuda_stream)
A, B, C = (torch.empty((n, n), dtype=torch.int32, device="cuda") for _ in range(3))
for x, s in ((A, 11), (B, 12), (C, 13)):
    G.random_mat_dev(p, x, s, ctx=ctx)
for _ in range(2):
    G.fgemm(p, p - 1, A, B, 1, C, ctx=ctx)
ctx.synchronize()
print("ok")
