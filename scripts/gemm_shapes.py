"""Histogram of the fgemm shapes one PLUQ issues (reads FFG_GEMM lines from a log).

    FFG_GEMM_LOG=1 python scripts/gemm_shapes.py --run --n 16384 2> shapes.log
    python scripts/gemm_shapes.py shapes.log
"""
import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("log", nargs="?")
ap.add_argument("--run", action="store_true")
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--p", type=int, default=131071)
ap.add_argument("--thr", type=int, default=64)
a = ap.parse_args()

if a.run:
    import torch

    import paper_1402_3501_b200 as G

    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx = G.Context(0, stream=st.cuda_stream)
    d = torch.empty((a.n, a.n), dtype=torch.int32, device="cuda")
    G.random_mat_dev(a.p, d, 3, ctx=ctx)
    torch.cuda.synchronize()
    print("FFG_GEMM_BEGIN", file=sys.stderr, flush=True)
    G.pluq_tile_recursive(a.p, d, a.thr, ctx=ctx)
    torch.cuda.synchronize()
    sys.exit(0)

rows = []
on = False
for line in open(a.log):
    if line.startswith("FFG_GEMM_BEGIN"):
        on, rows = True, []
    elif on and line.startswith("FFG_GEMM "):
        m, n, k, simt = map(int, line.split()[1:])
        rows.append((m, n, k, simt))
by = collections.Counter()
macs = collections.Counter()
for m, n, k, simt in rows:
    key = ("simt" if simt else "tc", m, n, k)
    by[key] += 1
    macs[key] += m * n * k
tot = sum(macs.values())
print(f"{len(rows)} gemms, {tot / 1e12:.3f} T MACs")
print(f"{'path':5s} {'M':>6s} {'N':>6s} {'K':>6s} {'count':>6s} {'MAC share':>9s}")
for key, c in sorted(by.items(), key=lambda kv: -kv[1])[:60]:
    print(f"{key[0]:5s} {key[1]:6d} {key[2]:6d} {key[3]:6d} {c:6d} {macs[key] / tot:9.4f}")
