"""Latency of the small/medium fgemm shapes the PLUQ recursion issues (device buffers, CUDA
events, warm).  Usage: [FFG_NO_DIRECT=1] [FFG_SIMT_MACS=0] python scripts/gemm_small.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time  # noqa: E402

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1402_3501_b200 as G  # noqa: E402

p = int(os.environ.get("P", "131071"))
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = G.Context(0, stream=st.cuda_stream)
NB = int(os.environ.get("BIG", "16384"))
H = NB // 2
big = torch.empty((NB, NB), dtype=torch.int32, device="cuda")
G.random_mat_dev(p, big, 5, ctx=ctx)
shapes = [(64, 64, 64), (64, 64, 128), (128, 128, 128), (128, 128, 256), (128, 1024, 128), (1024, 128, 128),
          (128, 8192, 128), (8192, 128, 128), (256, 8192, 256), (8192, 256, 256), (512, 512, 1024),
          (1024, 1024, 2048), (2048, 2048, 4096)]
if os.environ.get("SHAPES"):  # "m,n,k;m,n,k"
    shapes = [tuple(int(x) for x in t.split(",")) for t in os.environ["SHAPES"].split(";")]
for (m, n, k) in shapes:
    A = big[:m, :k]
    B = big[:k, H:H + n] if n <= H else big[:k, :n]
    C_ = big[H:H + m, H // 2:H // 2 + n] if m <= H else big[:m, H // 2:H // 2 + n]
    inplace = os.environ.get("INPLACE") == "1" and m <= 128
    if inplace:
        if m != k:
            continue
        C_ = B = big[:k, H:H + n]
        A = big[H:H + m, :k]
    for _ in range(3):
        G.fgemm(p, p - 1, A, B, 1, C_, ctx=ctx)
    reps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(st)
    for _ in range(reps):
        G.fgemm(p, p - 1, A, B, 1, C_, ctx=ctx)
    e1.record(st)
    host_us = (time.perf_counter() - t0) * 1e6 / reps
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / reps
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            G.fgemm(p, p - 1, A, B, 1, C_, ctx=ctx)
        torch.cuda.synchronize()
    ks = {}
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            nm = ev.name.split("(")[0].replace("void ", "").replace("ffg::", "")[:28]
            ks[nm] = ks.get(nm, 0.0) + ev.device_time_total / reps
    kern = " ".join(f"{k}={v:.1f}" for k, v in ks.items())
    print(f"{m:6d} {n:6d} {k:6d} {'inplace' if inplace else '':8s} event {us:7.1f} us  host {host_us:6.1f} us  "
          f"kernels: {kern}", flush=True)
