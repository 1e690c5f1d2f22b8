import sys, time
sys.path.insert(0, '/root/repo')
import torch
import paper_1402_3501_b200 as G
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
for world in (1, 2, 8):
    ctx = G.Context(0, stream=st.cuda_stream)
    if world > 1:
        ctx.dist_init_virtual(world, False)
    n = 16384
    ms = []
    for i in range(4):
        d = torch.empty((n, n), dtype=torch.int32, device='cuda')
        G.random_mat_dev(131071, d, 1 + i, ctx=ctx); ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); G.pluq_tile_recursive(131071, d, 64, ctx=ctx); e1.record(st); torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    print('virtual world', world, 'ms', [round(x, 1) for x in ms], flush=True)
    ctx.close()
