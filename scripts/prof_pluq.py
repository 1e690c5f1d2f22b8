"""Profiling driver: one warm PLUQ, then the measured one (for ncu launch lists / nsys-less timing).

    python scripts/prof_pluq.py --n 4096 --thr 64 [--p 131071] [--lru]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1402_3501_b200 as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--p", type=int, default=131071)
ap.add_argument("--thr", type=int, default=64)
ap.add_argument("--lru", action="store_true")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = G.Context(0, stream=st.cuda_stream)
mats = []
for i in range(a.reps):
    d = torch.empty((a.n, a.n), dtype=torch.int32, device="cuda")
    if a.lru:
        G.lru_matrix_dev(a.p, d, a.n // 2, 3 + i, ctx=ctx)
    else:
        G.random_mat_dev(a.p, d, 3 + i, ctx=ctx)
    mats.append(d)
ctx.synchronize()
for i, d in enumerate(mats):
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    r = G.pluq_tile_recursive(a.p, d, a.thr, ctx=ctx)
    e1.record(st)
    torch.cuda.synchronize()
    print(f"rep {i}: rank {r.rank} device {e0.elapsed_time(e1):.2f} ms wall {(time.perf_counter() - t0) * 1e3:.2f} ms "
          f"launches so far {ctx.launches}", flush=True)
