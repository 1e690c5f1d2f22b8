"""GPU parity of the public entries on their own (not only as parts of the PLUQ):

* ffg_apply_perm_dev: forward and inverse, rows and columns, against the oracle's apply_perm
  (perm.hpp:167-193) of the same PermSeq move list (swaps and rotations);
* ffg_ftrsm at t in {513, 1024, 2048} for all 8 side/uplo/diag combinations against the
  oracle (blas.hpp:285-384), through the host entry and the device entry;
* a C++ program built on include/ffpluq_b200.hpp (the reference-shaped header) run on the
  B200 against a reference golden case (BASELINE config 1, n = 1024).
"""
import os
import shutil
import subprocess

import numpy as np
import pytest

from golden_util import SplitMix64, fnv_u32, load, make_input

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _moves(dim, count, seed):
    rng = SplitMix64(seed)
    out = []
    for _ in range(count):
        i, j = rng.below(dim), rng.below(dim)
        if i == j:
            continue
        t = rng.below(2)
        if t == 1 and i > j:
            i, j = j, i
        out.append((t, i, j))
    return out


@pytest.mark.parametrize("axis", [0, 1])
@pytest.mark.parametrize("inverse", [False, True])
@pytest.mark.parametrize("count", [1, 17, 400])
def test_apply_perm_dev_matches_oracle(gpu, oracle_lib, axis, inverse, count):
    import torch
    G, ctx = gpu
    O = oracle_lib
    p = 131071
    m, n, ld = 300, 257, 270
    A = O.random_mat(p, m, n, count + axis)
    dim = m if axis == 0 else n
    mv = _moves(dim, count, 1000 * count + 7 * axis + inverse)
    arr = O.moves_to_array(dim, mv)
    want = O.apply_moves(A, axis, mv, inverse)
    buf = torch.full((m, ld), -1, dtype=torch.int32, device="cuda")
    buf[:, :n] = torch.from_numpy(A.view(np.int32)).cuda()
    view = buf[:, :n]
    perm = torch.from_numpy(arr.view(np.int32)).cuda()
    G.apply_perm_dev(view, axis, perm, inverse, ctx=ctx)
    ctx.synchronize()
    got = buf.cpu().numpy().view(np.uint32)
    assert np.array_equal(got[:, :n], want)
    assert np.all(got[:, n:] == 0xFFFFFFFF)  # the padding is untouched


def _triangle(O, p, t, seed):
    a = O.random_mat(p, t, t, seed)
    d = np.arange(t)
    a[d, d] = np.where(a[d, d] == 0, 1, a[d, d])
    return a


@pytest.mark.parametrize("t", [513, 1024, 2048])
@pytest.mark.parametrize("side", [0, 1])
@pytest.mark.parametrize("uplo", [0, 1])
@pytest.mark.parametrize("diag", [0, 1])
def test_ftrsm_large_matches_oracle(gpu, oracle_lib, t, side, uplo, diag):
    import torch
    G, ctx = gpu
    O = oracle_lib
    p = 131071
    other = 96
    A = _triangle(O, p, t, t + 2 * side + uplo)
    B = O.random_mat(p, t, other, 5) if side == 0 else O.random_mat(p, other, t, 6)
    want = O.ftrsm(p, side, uplo, diag, A, B)
    got = B.copy()
    G.ftrsm(p, side, uplo, diag, A, got, ctx=ctx)  # host entry
    assert np.array_equal(got, want)
    dA = torch.from_numpy(A.view(np.int32).copy()).cuda()
    dB = torch.from_numpy(B.view(np.int32).copy()).cuda()
    G.ftrsm(p, side, uplo, diag, dA, dB, ctx=ctx)  # device entry
    ctx.synchronize()
    assert np.array_equal(dB.cpu().numpy().view(np.uint32), want)


CPP = r"""
#include <cstdio>
#include <vector>
#include "ffpluq_b200.hpp"
using namespace ffpluq_b200;
int main(int argc, char** argv) {
    size_t n = 0, thr = 0; unsigned long long p = 0;
    FILE* f = std::fopen(argv[1], "rb");
    if (!f || std::fread(&n, 8, 1, f) != 1 || std::fread(&thr, 8, 1, f) != 1 || std::fread(&p, 8, 1, f) != 1) return 2;
    std::vector<u32> a(n * n);
    if (std::fread(a.data(), 4, n * n, f) != n * n) return 2;
    std::fclose(f);
    MatView v{a.data(), n, n, n, p};
    PluqResult res = pluq_tile_recursive(v, thr);
    // the reference's PermSeq semantics: to_array() of the returned move lists
    std::vector<u32> P = res.P.to_array(), Q = res.Q.to_array();
    FILE* o = std::fopen(argv[2], "wb");
    size_t r = res.rank;
    std::fwrite(&r, 8, 1, o);
    std::fwrite(P.data(), 4, n, o);
    std::fwrite(Q.data(), 4, n, o);
    std::fwrite(a.data(), 4, n * n, o);
    std::fclose(o);
    std::printf("rank %zu\n", r);
    return 0;
}
"""


def test_cpp_header_program_on_b200_matches_reference_golden(gpu, oracle_lib, tmp_path):
    """include/ffpluq_b200.hpp: a C++ caller of the reference-shaped API, run on the GPU, against the
    reference's own output for BASELINE config 1 (tests/golden/golden.json)."""
    gxx = shutil.which("g++")
    assert gxx, "g++ is part of the image"
    O = oracle_lib
    case = next(c for c in load()["cases"] if c["kind"] == "tile_rec" and "BASELINE config 1" in c.get("note", "")
                and c.get("variant") != "as_written")
    p, thr = case["p"], case["thr"]
    A = make_input(case["A"])
    n = A.shape[0]
    src = tmp_path / "prog.cpp"
    src.write_text(CPP)
    libdir = os.path.join(ROOT, "paper_1402_3501_b200")
    exe = tmp_path / "prog"
    subprocess.check_call([gxx, "-std=c++17", "-O2", str(src), "-I", os.path.join(ROOT, "include"), "-L", libdir,
                           "-lffg_b200", f"-Wl,-rpath,{libdir}", "-o", str(exe)])
    inp, out = tmp_path / "in.bin", tmp_path / "out.bin"
    with open(inp, "wb") as f:
        f.write(np.array([n, thr, p], dtype=np.uint64).tobytes())
        f.write(A.astype(np.uint32).tobytes())
    r = subprocess.run([str(exe), str(inp), str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    raw = np.fromfile(out, dtype=np.uint8)
    rank = int(raw[:8].view(np.uint64)[0])
    rest = raw[8:].view(np.uint32)
    P, Q, packed = rest[:n], rest[n:2 * n], rest[2 * n:].reshape(n, n)
    assert rank == case["rank"]
    assert fnv_u32(P) == case["P_h"] and fnv_u32(Q) == case["Q_h"]
    assert O.checksum(packed, p) == case["out_ck"]


def test_device_entries_reject_bad_leading_dimension(gpu):
    """ld < cols on any entry is FFG_ERR_INVALID_DIM (never an out-of-bounds device access); the
    Python mirror refuses CPU / wrong-dtype / non-unit-stride tensors for the _dev entries."""
    import ctypes as C

    import torch
    G, ctx = gpu
    L = G.lib()
    d = torch.zeros((64, 64), dtype=torch.int32, device="cuda")
    ptr = d.data_ptr()
    assert L.ffg_fgemm_dev(ctx.handle, 131071, 1, ptr, 10, ptr, 64, 0, ptr, 64, 64, 64, 64) == 9
    assert L.ffg_ftrsm_dev(ctx.handle, 131071, 0, 0, 0, ptr, 64, ptr, 32, 64, 64) == 9
    r = C.c_size_t(0)
    P = (C.c_uint32 * 64)()
    assert L.ffg_pluq_tile_recursive_dev(ctx.handle, 131071, ptr, 64, 64, 63, 8, P, P, C.byref(r)) == 9
    assert L.ffg_apply_perm_dev(ctx.handle, ptr, 64, 64, 16, 0, 0, ptr) == 9
    assert L.ffg_random_mat_dev(ctx.handle, 131071, 1, ptr, 64, 64, 8) == 9
    with pytest.raises(TypeError):
        G.pluq_tile_recursive(131071, torch.zeros((8, 8), dtype=torch.int32), 8, ctx=ctx)  # CPU tensor
    with pytest.raises(TypeError):
        G.pluq_tile_recursive(131071, torch.zeros((8, 8), dtype=torch.int64, device="cuda"), 8, ctx=ctx)
    with pytest.raises(ValueError):
        G.pluq_tile_recursive(131071, torch.zeros((8, 8), dtype=torch.int32, device="cuda").t(), 8, ctx=ctx)
    ctx.synchronize()


def test_spec_stats_and_knob_snapshot(oracle_lib, monkeypatch):
    """ffg_spec_stats counts the full-rank guesses of a context; the FFG_* switches are a snapshot
    that ffg_knobs_reload() refreshes (conftest reloads after every monkeypatch change)."""
    import paper_1402_3501_b200 as G
    O = oracle_lib
    p = 131071
    ctx = G.Context(0)
    try:
        s0 = ctx.spec_stats()
        assert set(s0) == {"guesses", "guesses_failed", "node_guesses", "node_guesses_failed", "profile_first_runs"}
        A = O.random_mat(p, 640, 640, 5)  # full rank: the guess holds
        want = O.pluq_tile_recursive(p, A, 64)
        got = A.copy()
        r = G.pluq_tile_recursive(p, got, 64, ctx=ctx)
        assert r.rank == want[3] and np.array_equal(got, want[0])
        s1 = ctx.spec_stats()
        assert s1["guesses"] == s0["guesses"] + 1 and s1["guesses_failed"] == s0["guesses_failed"]
        B, _, _ = O.lru_matrix(640, 300, p, 9)  # deficient from the first block: the guess fails
        want = O.pluq_tile_recursive(p, B, 64)
        got = B.copy()
        r = G.pluq_tile_recursive(p, got, 64, ctx=ctx)
        assert r.rank == want[3] == 300 and np.array_equal(got, want[0])
        assert np.array_equal(r.P, want[1]) and np.array_equal(r.Q, want[2])
        s2 = ctx.spec_stats()
        # the failed whole-matrix guess, then the profile-first path's own (holding) guess on the
        # generic leading block
        assert s2["guesses"] == s1["guesses"] + 2 and s2["guesses_failed"] == s1["guesses_failed"] + 1
        assert s2["profile_first_runs"] == s1["profile_first_runs"] + 1
    finally:
        ctx.close()
    # a switch set after the first snapshot is seen once the snapshot is refreshed (conftest reloads
    # on monkeypatch): without the profile-first path the same input takes the exact recursion
    ctx = G.Context(0)
    try:
        monkeypatch.setenv("FFG_PROFILE_FIRST", "0")
        s0 = ctx.spec_stats()
        got = B.copy()
        r = G.pluq_tile_recursive(p, got, 64, ctx=ctx)
        want = O.pluq_tile_recursive(p, B, 64)
        assert r.rank == want[3] and np.array_equal(got, want[0])
        assert np.array_equal(r.P, want[1]) and np.array_equal(r.Q, want[2])
        assert ctx.spec_stats()["profile_first_runs"] == s0["profile_first_runs"]
    finally:
        ctx.close()
