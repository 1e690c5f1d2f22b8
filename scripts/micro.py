"""Microbenchmarks of single small kernels through the device API (in situ, CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1402_3501_b200 as G  # noqa: E402

p = 131071
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = G.Context(0, stream=st.cuda_stream)


def timeit(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


print("base case (one rr_base kernel + rank readback) per call, us:")
for n in (16, 32, 64, 96, 128):
    d = torch.empty((n, n), dtype=torch.int32, device="cuda")
    src = torch.empty_like(d)
    G.random_mat_dev(p, src, 1, ctx=ctx)

    def f():
        d.copy_(src)
        G.pluq_tile_recursive(p, d, n, ctx=ctx)
    t_all = timeit(f)
    t_copy = timeit(lambda: d.copy_(src))
    print(f"  n={n:4d}: {t_all - t_copy:8.1f} us  ({(t_all - t_copy) / n:.2f} us/pivot)")

print("small trsm (direct kernel), us:")
for side in (0, 1):
    for (t, w) in ((16, 64), (64, 64), (64, 1024), (128, 128), (128, 4096)):
        T = torch.empty((t, t), dtype=torch.int32, device="cuda")
        G.random_mat_dev(p, T, 2, ctx=ctx)
        Td = T.clone()
        idx = torch.arange(t, device="cuda")
        Td[idx, idx] = Td[idx, idx].clamp(min=1)
        B = torch.empty((t, w) if side == 0 else (w, t), dtype=torch.int32, device="cuda")
        G.random_mat_dev(p, B, 3, ctx=ctx)
        us = timeit(lambda: G.ftrsm(p, side, 1 - side, 1 - side, Td, B, ctx=ctx))
        print(f"  side={side} t={t:4d} w={w:5d}: {us:8.1f} us")

print("gemm, us:")
for (m, k, n) in ((64, 64, 64), (128, 128, 128), (256, 256, 256), (512, 512, 512), (1024, 1024, 1024),
                  (2048, 2048, 2048), (4096, 4096, 4096), (128, 128, 4096), (4096, 128, 4096)):
    A = torch.empty((m, k), dtype=torch.int32, device="cuda")
    B = torch.empty((k, n), dtype=torch.int32, device="cuda")
    C = torch.empty((m, n), dtype=torch.int32, device="cuda")
    for x, s in ((A, 4), (B, 5), (C, 6)):
        G.random_mat_dev(p, x, s, ctx=ctx)
    us = timeit(lambda: G.fgemm(p, p - 1, A, B, 1, C, ctx=ctx), reps=20)
    print(f"  {m}x{k}x{n}: {us:9.1f} us  {2.0 * m * n * k / us / 1e6:9.1f} Top/s field")
