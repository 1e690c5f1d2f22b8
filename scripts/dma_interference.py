"""Does a concurrent PCIe copy (unrelated buffers) slow the device-only PLUQ?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1402_3501_b200 as G  # noqa: E402

n, p = 16384, 131071
st = torch.cuda.Stream()
cs = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = G.Context(0, stream=st.cuda_stream)
d = torch.empty((n, n), dtype=torch.int32, device="cuda")
junk = torch.empty((n, n), dtype=torch.int32, device="cuda")
host = torch.empty((n, n), dtype=torch.int32).pin_memory()
for mode in ("alone", "d2h", "h2d", "alone"):
    for it in range(2):
        G.random_mat_dev(p, d, 5 + it, ctx=ctx)
        torch.cuda.synchronize()
        if mode != "alone":
            with torch.cuda.stream(cs):
                for _ in range(3):
                    if mode == "d2h":
                        host.copy_(junk, non_blocking=True)
                    else:
                        junk.copy_(host, non_blocking=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        G.pluq_tile_recursive(p, d, 64, ctx=ctx)
        e1.record(st)
        torch.cuda.synchronize()
        if it == 1:
            print(f"{mode:6s}: {e0.elapsed_time(e1):.2f} ms", flush=True)
