"""CUPTI kernel summary of one PLUQ for a given seed (config 5 default): busy vs idle, per kernel."""
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
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--p", type=int, default=251)
ap.add_argument("--seed", type=int, default=3)
ap.add_argument("--lru", action="store_true")
a = ap.parse_args()
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = G.Context(0, stream=st.cuda_stream)
d = torch.empty((a.n, a.n), dtype=torch.int32, device="cuda")
for warm in (True, False):
    if a.lru:
        G.lru_matrix_dev(a.p, d, a.n // 2, a.seed, ctx=ctx)
    else:
        G.random_mat_dev(a.p, d, a.seed, ctx=ctx)
    ctx.synchronize()
    if warm:
        G.pluq_tile_recursive(a.p, d, 64, ctx=ctx)
        torch.cuda.synchronize()
        continue
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        G.pluq_tile_recursive(a.p, d, 64, ctx=ctx)
        e1.record(st)
        torch.cuda.synchronize()
ks = []
for e in prof.events():
    if e.device_type.name != "CUDA" or e.device_time_total <= 0:
        continue
    nm = re.sub(r"^void ", "", re.sub(r"\(.*", "", e.name))[:40]
    ks.append((e.time_range.start, e.time_range.end, nm))
ks.sort()
busy, last = 0.0, None
for s, t, _ in ks:
    if last is None or s >= last:
        busy += t - s
        last = t
    elif t > last:
        busy += t - last
        last = t
span = (ks[-1][1] - ks[0][0]) / 1e3
print(f"event {e0.elapsed_time(e1):.2f} ms, span {span:.2f} ms, busy {busy / 1e3:.2f} ms, launches {len(ks)}")
agg = collections.defaultdict(lambda: [0, 0.0])
for s, t, nm in ks:
    agg[nm][0] += 1
    agg[nm][1] += (t - s) / 1e3
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
    print(f"  {k:40s} {v[0]:6d} {v[1]:9.3f} ms")
# idle gaps > 50 us
gaps = []
last = None
for s, t, nm in ks:
    if last is not None and s > last + 50_000 / 1e3 * 1e3:
        gaps.append((s - last) / 1e3)
    last = t if last is None else max(last, t)
print(f"gaps > 50 us: {len(gaps)}, total {sum(gaps):.2f} ms")
