"""Per-kernel device times (CUPTI via torch.profiler) for small TRSM / base / GEMM calls."""
import collections
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1402_3501_b200 as G  # noqa: E402

p = 131071
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = G.Context(0, stream=st.cuda_stream)


def kernel_times(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in prof.events():
        if e.device_type.name != "CUDA" or e.device_time_total <= 0:
            continue
        nm = re.sub(r"\(.*", "", e.name).replace("void ", "").replace("ffg::", "")[:40]
        if nm.startswith("Memcpy") or nm.startswith("Memset"):
            continue
        agg[nm][0] += 1
        agg[nm][1] += (e.time_range.end - e.time_range.start)
    return {k: (v[0] // reps, v[1] / v[0]) for k, v in agg.items()}


def show(tag, d):
    print(f"{tag:28s} " + "  ".join(f"{k}: {n}x {us:.1f}us" for k, (n, us) in sorted(d.items())))


for t in (64, 128, 256):
    for w in (64, 1024, 8192):
        T = torch.empty((t, t), dtype=torch.int32, device="cuda")
        G.random_mat_dev(p, T, 2, ctx=ctx)
        B = torch.empty((t, w), dtype=torch.int32, device="cuda")
        G.random_mat_dev(p, B, 3, ctx=ctx)
        show(f"trsm L lower unit t={t} w={w}", kernel_times(lambda: G.ftrsm(p, 0, 0, 0, T, B, ctx=ctx)))
for n in (32, 64, 128):
    d = torch.empty((n, n), dtype=torch.int32, device="cuda")
    src = torch.empty_like(d)
    G.random_mat_dev(p, src, 1, ctx=ctx)

    def f():
        d.copy_(src)
        G.pluq_tile_recursive(p, d, n, ctx=ctx)
    show(f"base n={n}", kernel_times(f))
for (m, k, n) in ((128, 128, 128), (128, 128, 1024), (1024, 128, 1024), (4096, 128, 4096), (1024, 1024, 1024),
                  (4096, 4096, 4096)):
    A = torch.empty((m, k), dtype=torch.int32, device="cuda")
    B = torch.empty((k, n), dtype=torch.int32, device="cuda")
    C = torch.empty((m, n), dtype=torch.int32, device="cuda")
    for x, s in ((A, 4), (B, 5), (C, 6)):
        G.random_mat_dev(p, x, s, ctx=ctx)
    show(f"gemm {m}x{k}x{n}", kernel_times(lambda: G.fgemm(p, p - 1, A, B, 1, C, ctx=ctx)))
