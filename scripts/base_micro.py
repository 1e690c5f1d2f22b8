"""Isolated device time of the panel schedule's base-case kernels (CUPTI), one 64 x 64 block.

    python scripts/base_micro.py [--n 64] [--reps 50]
"""
import argparse
import collections
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1402_3501_b200 as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=64)
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--p", type=int, default=131071)
a = ap.parse_args()
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = G.Context(0, stream=st.cuda_stream)
src = torch.empty((a.n, a.n), dtype=torch.int32, device="cuda")
G.random_mat_dev(a.p, src, 5, ctx=ctx)
d = torch.empty_like(src)


def once():
    d.copy_(src)
    G.pluq_tile_recursive(a.p, d, 64, ctx=ctx)


for _ in range(5):
    once()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(a.reps):
        once()
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type.name != "CUDA" or e.device_time_total <= 0:
        continue
    nm = re.sub(r"\(.*", "", e.name).replace("void ", "").replace("ffg::", "")
    if nm.startswith("Memcpy") or nm.startswith("Memset"):
        continue
    agg[nm][0] += 1
    agg[nm][1] += e.time_range.end - e.time_range.start
for k, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:50s} {c // a.reps:3d}/call {us / c:8.2f} us")
