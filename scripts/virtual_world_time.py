"""Single-GPU "virtual world" timing of the partitioned PLUQ: one process computes every rank's
slice of each split Schur operation through the partition code (no exchange), so the difference to
world 1 is the partitioning overhead.  Prints one JSON line per world.

    python scripts/virtual_world_time.py [--n 16384] [--p 131071] [--worlds 1,2,4,8] [--reps 4]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1402_3501_b200 as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--p", type=int, default=131071)
ap.add_argument("--worlds", default="1,2,4,8")
ap.add_argument("--reps", type=int, default=4)
a = ap.parse_args()
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
d = torch.empty((a.n, a.n), dtype=torch.int32, device="cuda")
for world in [int(w) for w in a.worlds.split(",")]:
    ctx = G.Context(0, stream=st.cuda_stream)
    if world > 1:
        ctx.dist_init_virtual(world, False)
    ms = []
    for i in range(a.reps + 1):
        G.random_mat_dev(a.p, d, 1 + i, ctx=ctx)
        ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        G.pluq_tile_recursive(a.p, d, 64, ctx=ctx)
        e1.record(st)
        torch.cuda.synchronize()
        if i:
            ms.append(e0.elapsed_time(e1))
    info = ctx.dist_info()
    print(json.dumps({"n": a.n, "p": a.p, "virtual_world": world, "ms": [round(x, 2) for x in ms],
                      "mean_ms": round(sum(ms) / len(ms), 2), "exchanges": info["exchanges"]}), flush=True)
    ctx.close()
