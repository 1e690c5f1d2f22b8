"""CUPTI timeline window of one PLUQ: every kernel whose start falls in [--t0, --t1) ms.

    python scripts/trace_window.py --lru --n 16384 --t0 20 --t1 20.8
"""
import argparse
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1402_3501_b200 as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--p", type=int, default=131071)
ap.add_argument("--thr", type=int, default=64)
ap.add_argument("--lru", action="store_true")
ap.add_argument("--t0", type=float, default=20.0)
ap.add_argument("--t1", type=float, default=20.8)
a = ap.parse_args()
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = G.Context(0, stream=st.cuda_stream)
mats = []
for i in range(2):
    d = torch.empty((a.n, a.n), dtype=torch.int32, device="cuda")
    if a.lru:
        G.lru_matrix_dev(a.p, d, a.n // 2, 3 + i, ctx=ctx)
    else:
        G.random_mat_dev(a.p, d, 3 + i, ctx=ctx)
    mats.append(d)
ctx.synchronize()
G.pluq_tile_recursive(a.p, mats[0], a.thr, ctx=ctx)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    G.pluq_tile_recursive(a.p, mats[1], a.thr, ctx=ctx)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA" and e.device_time_total > 0]
ks = sorted((e.time_range.start, e.time_range.end, re.sub(r"^void ", "", re.sub(r"\(.*", "", e.name))[:40]) for e in evs)
base = ks[0][0]
print(f"kernels {len(ks)}, span {(ks[-1][1] - base) / 1e3:.2f} ms")
for s, t, nm in ks:
    ms = (s - base) / 1e3
    if a.t0 <= ms < a.t1:
        print(f"  +{(s - base) - a.t0 * 1e3:9.1f} us  {t - s:8.1f} us  {nm}")
