"""PCIe copy rates on this box: 1 GiB H2D / D2H alone and concurrently, and 2-D copies of short
rows (the column strips of the host entry's L-shaped bands)."""
import torch

n = 16384
H = torch.empty((n, n), dtype=torch.int32).pin_memory()
H2 = torch.empty((n, n), dtype=torch.int32).pin_memory()
D = torch.empty((n, n), dtype=torch.int32, device="cuda")
D2 = torch.empty((n, n), dtype=torch.int32, device="cuda")
up, down = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        for s in (up, down):
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


gb = n * n * 4 / 1e9


def h2d():
    with torch.cuda.stream(up):
        D.copy_(H, non_blocking=True)


def d2h():
    with torch.cuda.stream(down):
        H2.copy_(D2, non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn in (("H2D", h2d), ("D2H", d2h), ("both", both)):
    t = timed(fn)
    print(f"{name:5s} {t:7.2f} ms  {gb / t * 1e3:6.1f} GB/s per direction")
import ctypes
import glob
import os

import nvidia.cuda_runtime as _cr  # the runtime torch loads

rt = ctypes.CDLL(glob.glob(os.path.join(list(_cr.__path__)[0], "lib", "libcudart.so*"))[0])
rt.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                 ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
for w in (256, 1024, 4096):
    def strips():
        for c0 in range(0, n, w):
            rc = rt.cudaMemcpy2DAsync(D.data_ptr() + c0 * 4, n * 4, H.data_ptr() + c0 * 4, n * 4, w * 4, n, 1,
                                      up.cuda_stream)
            assert rc == 0, rc
    t = timed(strips, 2)
    print(f"H2D cudaMemcpy2D, {n // w} column strips of {w * 4} B rows: {t:7.2f} ms  {gb / t * 1e3:6.1f} GB/s")
    def strips_both():
        strips()
        d2h()
    t = timed(strips_both, 2)
    print(f"   ... with a 1 GiB D2H beside it: {t:7.2f} ms")
