"""Host logic of the partitioned PLUQ, on CPU: the library's partition function, the NCCL id
rendezvous over a torch process group, and the slice decomposition of the Schur operations
(world_size 2, gloo on 127.0.0.1; the oracle computes each rank's slice, gloo gathers them)."""
import os
import socket

import numpy as np
import pytest

import paper_1402_3501_b200 as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_partition_covers_disjoint_aligned():
    for world in (1, 2, 3, 4, 5, 8):
        for total in (0, 1, 127, 128, 129, 1000, 4096, 8191, 16384, 16385):
            for align in (1, 64, 128):
                sl = G.dist.plan(total, world, align)
                assert len(sl) == world
                pos = 0
                for r, (lo, hi) in enumerate(sl):
                    assert lo == pos and lo <= hi <= total
                    if hi < total and hi > lo:
                        assert lo % align == 0 and (hi - lo) % align == 0
                    pos = hi
                assert pos == total
                # no rank gets more than one aligned chunk beyond the even share
                chunk = -(-(-(-total // world)) // align) * align if total else 0
                assert all(hi - lo <= chunk for lo, hi in sl)


def test_partition_rejects_bad_rank():
    with pytest.raises(G.FfgError):
        G.dist_partition(10, 2, 2)
    with pytest.raises(G.FfgError):
        G.dist_partition(10, 0, 0)


def test_unique_id_is_128_bytes():
    uid = G.dist_unique_id()
    assert isinstance(uid, bytes) and len(uid) == 128


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port):
    import torch.distributed as dist

    from oracle import oracle as O

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        # 1. NCCL id rendezvous: every rank receives rank 0's id
        uid = G.dist.share_unique_id(rank)
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        assert all(i == ids[0] for i in ids) and len(ids[0]) == 128

        p = 131071
        align = 128

        def gather_rows(full_shape, lo, block):
            parts = [None] * world
            dist.all_gather_object(parts, (lo, block))
            out = np.zeros(full_shape, np.uint32)
            for plo, pb in parts:
                if pb is not None:
                    out[plo:plo + pb.shape[0], :] = pb
            return out

        def gather_cols(full_shape, lo, block):
            parts = [None] * world
            dist.all_gather_object(parts, (lo, block))
            out = np.zeros(full_shape, np.uint32)
            for plo, pb in parts:
                if pb is not None:
                    out[:, plo:plo + pb.shape[1]] = pb
            return out

        # 2. C -= A B split by rows of C and by columns of C
        m, k, n = 300, 140, 260
        A = O.random_mat(p, m, k, 1)
        B = O.random_mat(p, k, n, 2)
        C0 = O.random_mat(p, m, n, 3)
        want = O.fgemm(p, p - 1, A, B, 1, C0.copy())
        lo, hi = G.dist_partition(m, world, rank, align)
        blk = O.fgemm(p, p - 1, A[lo:hi], B, 1, C0[lo:hi].copy()) if hi > lo else None
        assert np.array_equal(gather_rows(C0.shape, lo, blk), want)
        lo, hi = G.dist_partition(n, world, rank, align)
        blk = O.fgemm(p, p - 1, A, B[:, lo:hi], 1, C0[:, lo:hi].copy()) if hi > lo else None
        assert np.array_equal(gather_cols(C0.shape, lo, blk), want)

        # 3. TRSMs of tile_rec: left unit-lower on column slices, right upper on row slices
        t = 150
        T = O.random_mat(p, t, t, 4)
        T[np.diag_indices(t)] = np.maximum(T[np.diag_indices(t)], 1)
        Bl = O.random_mat(p, t, 290, 5)
        want = O.ftrsm(p, 0, 0, 0, T, Bl.copy())
        lo, hi = G.dist_partition(Bl.shape[1], world, rank, align)
        blk = O.ftrsm(p, 0, 0, 0, T, Bl[:, lo:hi].copy()) if hi > lo else None
        assert np.array_equal(gather_cols(Bl.shape, lo, blk), want)
        Br = O.random_mat(p, 333, t, 6)
        want = O.ftrsm(p, 1, 1, 1, T, Br.copy())
        lo, hi = G.dist_partition(Br.shape[0], world, rank, align)
        blk = O.ftrsm(p, 1, 1, 1, T, Br[lo:hi].copy()) if hi > lo else None
        assert np.array_equal(gather_rows(Br.shape, lo, blk), want)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_decomposition(oracle_lib):
    import torch.multiprocessing as mp

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    mp.spawn(_worker, args=(2, _free_port()), nprocs=2, join=True)


def test_bench_relaunches_itself_under_torchrun_for_gpus_n():
    """`bench.py --gpus 2` outside torchrun re-executes itself with one process per rank (CPU check
    through the reference arm: rank 0 prints the line, rank 1 exits cleanly)."""
    import json
    import subprocess
    import sys
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--n", "256", "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                       timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["same_size_as_config"] is True


def test_bench_rejects_world_mismatch():
    import subprocess
    import sys
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--n", "256"], capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode != 0 and "WORLD_SIZE" in (r.stderr + r.stdout)
