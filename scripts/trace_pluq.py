"""In-situ kernel timeline of one PLUQ via CUPTI (torch.profiler), no serialization.

    python scripts/trace_pluq.py --n 16384 --thr 64 [--lru] [--json out.json]

Prints per-kernel-name count / busy ms / share, GPU busy vs idle (gaps between
kernels on the timeline), and the busy time per recursion size bucket.
"""
import argparse
import collections
import json
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
ap.add_argument("--json", default=None)
ap.add_argument("--chrome", default=None, help="also export the raw chrome trace here")
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
G.pluq_tile_recursive(a.p, mats[0], a.thr, ctx=ctx)  # warm
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    G.pluq_tile_recursive(a.p, mats[1], a.thr, ctx=ctx)
    e1.record(st)
    torch.cuda.synchronize()
wall = e0.elapsed_time(e1)
if a.chrome:
    prof.export_chrome_trace(a.chrome)
evs = [e for e in prof.events() if e.device_type.name == "CUDA" and e.device_time_total > 0]
ks = []
for e in evs:
    name = re.sub(r"\(.*", "", e.name)
    name = re.sub(r"^void ", "", name)[:44]
    if name.startswith("Memcpy") or name.startswith("Memset"):
        continue
    ks.append((e.time_range.start, e.time_range.end, name))
ks.sort()
agg = collections.defaultdict(lambda: [0, 0.0])
for s, t, nm in ks:
    agg[nm][0] += 1
    agg[nm][1] += (t - s) / 1e3
busy = 0.0
last = None
for s, t, _ in ks:
    if last is None or s >= last:
        busy += (t - s) / 1e3
        last = t
    elif t > last:
        busy += (t - last) / 1e3
        last = t
span = (ks[-1][1] - ks[0][0]) / 1e3 if ks else 0
print(f"n={a.n} thr={a.thr} {'lru' if a.lru else 'iid'}: event time {wall:.2f} ms, kernel span {span:.2f} ms, "
      f"GPU busy {busy:.2f} ms ({busy / span:.0%}), idle {span - busy:.2f} ms, launches {len(ks)}")
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':44s} {'n':>6s} {'busy ms':>9s} {'avg us':>8s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:44s} {v[0]:6d} {v[1]:9.3f} {1e3 * v[1] / v[0]:8.2f} {v[1] / tot:6.1%}")
if a.json:
    json.dump({"n": a.n, "thr": a.thr, "event_ms": wall, "busy_ms": busy, "span_ms": span, "launches": len(ks),
               "kernels": {k: {"count": v[0], "ms": v[1]} for k, v in agg.items()}}, open(a.json, "w"), indent=1)

# ---- per-step view (panel mode): kernels between consecutive base cases, grouped by the size of
# the node whose GEMMs follow base k (k's trailing one bits)
bases = [k for k in ks if "rr_base" in k[2]]
if len(bases) > 2:
    byt = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i in range(len(bases) - 1):
        t = 0
        while (i >> t) & 1:
            t += 1
        gap = (bases[i + 1][0] - bases[i][0]) / 1e3
        byt[t][0] += 1
        byt[t][1] += gap
        byt[t][2] += (bases[i][1] - bases[i][0]) / 1e3
    print("step type (node size after base k) | steps | avg base-to-base us | avg base us | total ms")
    for t in sorted(byt):
        c, g, b = byt[t]
        print(f"  node {64 << (t + 1):6d} | {c:5d} | {1e3 * g / c:9.1f} | {1e3 * b / c:7.1f} | {g:8.2f}")
    for i in list(range(100, 104)) + [126, 127]:
        if i + 1 >= len(bases):
            break
        b0 = bases[i][0]
        print(f"step {i}:")
        for s, t_, nm in ks:
            if b0 <= s < bases[i + 1][0] + 1:
                print(f"   +{(s - b0) / 1e3 * 1e3:8.1f} us  {((t_ - s) / 1e3) * 1e3:7.1f} us  {nm}")

# ---- long gaps between consecutive base cases (resumes, top-level GEMMs, host round trips)
if len(bases) > 2:
    print("long base-to-base gaps (> 150 us): base index, start ms, gap us, idle us, top kernels in the gap")
    t00 = ks[0][0]
    nlong = 0
    tot_long = 0.0
    for i in range(len(bases) - 1):
        s0, s1 = bases[i][0], bases[i + 1][0]
        gap = (s1 - s0) / 1e3
        if gap * 1e3 <= 150:
            continue
        nlong += 1
        tot_long += gap
        inside = [(s, t_, nm) for s, t_, nm in ks if s0 <= s < s1]
        by = collections.defaultdict(float)
        for s, t_, nm in inside:
            by[nm] += (t_ - s) / 1e3
        # idle: parts of the gap with no kernel running
        cov, last = 0.0, s0
        for s, t_, _ in sorted(inside):
            if t_ > last:
                cov += (t_ - max(s, last)) / 1e3
                last = t_
        top = ", ".join(f"{k.split('::')[-1][:22]} {1e3 * v:.0f}" for k, v in sorted(by.items(), key=lambda x: -x[1])[:4])
        print(f"  base {i:5d} at {(s0 - t00) / 1e3:8.2f} ms: gap {1e3 * gap:8.1f} us, idle {1e3 * (gap - cov):7.1f} us | {top}")
    print(f"  {nlong} long gaps, {tot_long:.2f} ms total")
