"""Dev check: GPU fgemm vs oracle (small) and Freivalds (large), timing of 8192^3."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
import paper_1402_3501_b200 as G

ctx = G.Context(0)
rng = np.random.default_rng(0)
bad = 0; n_cases = 0
for p in [2, 3, 5, 251, 65521, 131071, 16777213, 67108859]:
    for t in range(12):
        m, k, n = [int(x) for x in rng.integers(1, 300, 3)]
        if t == 0: m, k, n = 128, 128, 80
        A = O.random_mat(p, m, k, t); B = O.random_mat(p, k, n, t + 1); Cm = O.random_mat(p, m, n, t + 2)
        for al, be in [(p - 1, 1), (1, 0), (7 % p, 3 % p)]:
            want = O.fgemm(p, al, A, B, be, Cm)
            got = Cm.copy(); G.fgemm(p, al, A, B, be, got, ctx=ctx)
            n_cases += 1
            if not np.array_equal(want, got):
                bad += 1
                if bad < 5:
                    d = np.argwhere(want != got)
                    print("MISMATCH p", p, "mkn", m, k, n, "al be", al, be, "ndiff", len(d), "first", d[:3], want[tuple(d[0])], got[tuple(d[0])])
print(f"small cases: {n_cases}, bad {bad}", flush=True)

import torch
def freivalds(p, al, A, B, be, C0, C1, reps=2):
    for r in range(reps):
        x = np.random.default_rng(r).integers(0, p, C0.shape[1]).astype(np.int64)
        bx = (B.astype(np.int64) @ x) % p
        abx = (A.astype(np.int64) @ bx) % p
        want = (al * abx + be * ((C0.astype(np.int64) @ x) % p)) % p
        got = (C1.astype(np.int64) @ x) % p
        if not np.array_equal(want, got): return False
    return True

for p, N in [(131071, 8192), (251, 8192), (65521, 4096)]:
    A = O.random_mat(p, N, N, 11); B = O.random_mat(p, N, N, 12); C0 = O.random_mat(p, N, N, 13)
    dA = torch.from_numpy(A.view(np.int32)).cuda(); dB = torch.from_numpy(B.view(np.int32)).cuda(); dC = torch.from_numpy(C0.view(np.int32)).cuda()
    ts = torch.cuda.Stream(); torch.cuda.set_stream(ts)
    ctx.set_stream(ts.cuda_stream)
    G.fgemm(p, p - 1, dA, dB, 1, dC, ctx=ctx); torch.cuda.synchronize()
    ok = freivalds(p, p - 1, A, B, 1, C0, dC.cpu().numpy().view(np.uint32))
    times = []
    for i in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); G.fgemm(p, p - 1, dA, dB, 1, dC, ctx=ctx); e1.record(); torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    t = min(times) / 1e3
    print(f"p={p} N={N}: freivalds ok={ok}  time {t*1e3:.3f} ms  field Gop/s {2*N**3/t/1e9:.0f}", flush=True)
    ctx.set_stream(None)
