"""CUPTI timeline of one host-entry PLUQ (pinned host buffers): copies vs kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1402_3501_b200 as G  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
p = 131071
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = G.Context(0, stream=st.cuda_stream)
d = torch.empty((n, n), dtype=torch.int32, device="cuda")
G.random_mat_dev(p, d, 5, ctx=ctx)
ctx.synchronize()
H0 = d.cpu().pin_memory()
del d
torch.cuda.empty_cache()
H = torch.empty_like(H0).pin_memory()
Hn = H.numpy().view(np.uint32)
for it in range(2):
    H.copy_(H0)
    if it == 1:
        prof = profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU])
        prof.__enter__()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    G.pluq_tile_recursive(p, Hn, 64, ctx=ctx)
    e1.record(st)
    torch.cuda.synchronize()
    if it == 1:
        prof.__exit__(None, None, None)
    print(f"call {it}: {e0.elapsed_time(e1):.2f} ms", flush=True)
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in evs)
ks = [e for e in evs if "Memcpy" not in e.name and "Memset" not in e.name]
cps = [e for e in evs if "Memcpy" in e.name]
kspan = (min(e.time_range.start for e in ks) - t0, max(e.time_range.end for e in ks) - t0)
print(f"kernels: {len(ks)} from {kspan[0] / 1e3:.2f} to {kspan[1] / 1e3:.2f} ms")
for c in sorted(cps, key=lambda e: e.time_range.start):
    s, e = (c.time_range.start - t0) / 1e3, (c.time_range.end - t0) / 1e3
    if e - s > 0.05:
        print(f"  {c.name[:28]:28s} {s:8.2f} -> {e:8.2f} ms ({e - s:6.2f} ms)")
bases = sorted((e for e in ks if "rr_base" in e.name), key=lambda e: e.time_range.start)
if bases:
    print("base cases (every 16th): " + " ".join(
        f"{(b.time_range.start - t0) / 1e3:.1f}" for b in bases[::16]) + f" | last ends {(bases[-1].time_range.end - t0) / 1e3:.2f} ms")
end = max(e.time_range.end for e in evs) - t0
for lo in range(0, int(end / 1e3) + 5, 5):
    w0, w1 = lo * 1e3, (lo + 5) * 1e3

    def ov(e):
        s, t = e.time_range.start - t0, e.time_range.end - t0
        return max(0.0, min(t, w1) - max(s, w0))
    kb = sum(ov(e) for e in ks)
    h2d = sum(ov(e) for e in cps if "HtoD" in e.name)
    d2h = sum(ov(e) for e in cps if "DtoH" in e.name)
    print(f"  [{lo:3d},{lo + 5:3d}) ms: kernel-time {kb / 1e3:6.2f} ms  H2D busy {h2d / 1e3:5.2f}  D2H busy {d2h / 1e3:5.2f}")
