"""Per-seed device time of one PLUQ (config 5 by default) with the speculation outcome logged
(FFG_SPEC_LOG=1 prints 'SPEC ok / failed / resumed at offset')."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1402_3501_b200 as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--p", type=int, default=251)
ap.add_argument("--seeds", type=str, default="1,2,3,4,5,6")
ap.add_argument("--lru", action="store_true")
a = ap.parse_args()
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = G.Context(0, stream=st.cuda_stream)
d = torch.empty((a.n, a.n), dtype=torch.int32, device="cuda")
for i, s in enumerate([int(x) for x in a.seeds.split(",")]):
    if a.lru:
        G.lru_matrix_dev(a.p, d, a.n // 2, s, ctx=ctx)
    else:
        G.random_mat_dev(a.p, d, s, ctx=ctx)
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    r = G.pluq_tile_recursive(a.p, d, 64, ctx=ctx)
    e1.record(st)
    torch.cuda.synchronize()
    print(f"seed {s}: {e0.elapsed_time(e1):.2f} ms rank {r.rank}", file=sys.stderr, flush=True)
