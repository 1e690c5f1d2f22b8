"""Generate tests/golden/golden.json from the REFERENCE itself (oracle/_ref).

Run in the build container (needs /root/reference to have built oracle/_ref):

    python oracle/build_ref.py && python scripts/make_golden.py

Every output in the fixture comes from oracle/_ref/libffref_fixed.so or
libffref.so -- the reference headers compiled by oracle/build_ref.py -- never
from this repo's oracle or GPU code.  Inputs are regenerated from seeds by the
oracle's restatements of the reference generators (tests/golden_util.py) and
pinned by their checksums (matrix.hpp:53-68).

Case list (reference test that each block replicates):
  fgemm  : blas_test.cpp:9-16, 18-26, 38-50 (acc_bits=40 chunking), 52-73 (alpha/beta
           battery), 75-96 (225-case battery), plus ragged shapes > one GEMM tile
  ftrsm  : blas_test.cpp:143-160 (hand), 162-192 (ledger cases), 194-221 (solve
           battery), 223-233 (SingularDiagonal index), plus recursive-size cases
  rr_base: rankrev_test.cpp:31-84 (zero, identity, rank-2 GF(5), single entry)
  tile_rec: rankrev_test.cpp:86-110 (oracle battery), 137-164, 243-286,
           tests/CMakeLists.txt:25-27 (CLI check n=64 r=48 thr=4 seed=7),
           acceptance.cpp:41-79 corpus x thr {1,4,16}, config-4 L*R*U inputs
           (fixed and as-written reference), BASELINE config 1 (n=1024 iid).
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import oracle as O  # noqa: E402
from golden_util import GOLDEN, SplitMix64, fnv_u32, make_input  # noqa: E402

REF = O.Ref(fixed=True)
REF_AS_WRITTEN = O.Ref(fixed=False)
SMALL = 64  # store explicit outputs up to this many entries


def ck(a, p):
    return REF.checksum(a, p)


def explicit(p, rows):
    a = np.array(rows, dtype=np.uint64) % p
    return {"gen": "explicit", "p": p, "m": a.shape[0], "n": a.shape[1], "A": a.astype(np.uint32).ravel().tolist()}


def spec_of(p, gen, **kw):
    d = {"gen": gen, "p": p}
    d.update(kw)
    return d


cases = []


# ------------------------------------------------------------------ fgemm
def add_gemm(p, alpha, beta, sA, sB, sC, note, acc_bits=53):
    A, B, C = make_input(sA), make_input(sB), make_input(sC)
    out = REF.fgemm(p, alpha, A, B, beta, C, acc_bits=acc_bits)
    c = {"kind": "fgemm", "note": note, "p": p, "alpha": int(alpha), "beta": int(beta), "acc_bits": acc_bits,
         "A": sA, "B": sB, "C": sC, "in_ck": [ck(A, p), ck(B, p), ck(C, p)], "out_ck": ck(out, p)}
    if out.size <= SMALL:
        c["out"] = out.ravel().tolist()
    cases.append(c)


def gemm_cases():
    add_gemm(5, 1, 0, explicit(5, [[1, 2], [3, 4]]), explicit(5, [[0, 1], [1, 0]]), spec_of(5, "zeros", m=2, n=2),
             "blas_test.cpp:9-16 hand computed")
    add_gemm(131071, 1, 0, spec_of(131071, "identity", m=3, n=3), spec_of(131071, "random", m=3, n=5, seed=4),
             spec_of(131071, "zeros", m=3, n=5), "blas_test.cpp:18-26 identity")
    kk = 2 * 63 + 3
    add_gemm(131071, 1, 0, spec_of(131071, "random", m=2, n=kk, seed=5), spec_of(131071, "random", m=kk, n=2, seed=6),
             spec_of(131071, "zeros", m=2, n=2), "blas_test.cpp:38-50 chunked, acc_bits=40", acc_bits=40)
    p = 65521
    rng = SplitMix64(3)
    for t in range(30):  # blas_test.cpp:52-73
        m, k, n = 1 + rng.below(9), rng.below(9), 1 + rng.below(9)
        for alpha in (0, 1, p - 1, 7):
            for beta in (0, 1, p - 1, 3):
                add_gemm(p, alpha, beta, spec_of(p, "random", m=m, n=k, seed=10 + t),
                         spec_of(p, "random", m=k, n=n, seed=20 + t), spec_of(p, "random", m=m, n=n, seed=30 + t),
                         "blas_test.cpp:52-73 alpha/beta")
    seed = 1000
    for p in (2, 3, 5, 65521, 131071):  # blas_test.cpp:75-96
        rng = SplitMix64(p * 7 + 1)
        for t in range(45):
            m, k, n = 1 + rng.below(65), 1 + rng.below(65), 1 + rng.below(65)
            rng.below(4)
            rng.below(16)  # winograd levels / threshold draws (Winograd is bit-identical, blas.hpp:217-219)
            add_gemm(p, 1, 0, spec_of(p, "random", m=m, n=k, seed=seed), spec_of(p, "random", m=k, n=n, seed=seed + 1),
                     spec_of(p, "zeros", m=m, n=n), "blas_test.cpp:75-96 battery")
            seed += 2
    # ragged shapes spanning several GEMM tiles / all limb counts (this repo)
    s = 5000
    for p in (2, 251, 65521, 131071, 16777213, 67108859):
        for (m, k, n) in ((129, 257, 81), (300, 130, 161), (1, 1000, 3), (257, 5, 255)):
            add_gemm(p, p - 1, 1, spec_of(p, "random", m=m, n=k, seed=s), spec_of(p, "random", m=k, n=n, seed=s + 1),
                     spec_of(p, "random", m=m, n=n, seed=s + 2), "ragged multi-tile")
            s += 3


# ------------------------------------------------------------------ ftrsm
def add_trsm(p, side, uplo, diag, sA, sB, note):
    A, B = make_input(sA), make_input(sB)
    c = {"kind": "ftrsm", "note": note, "p": p, "side": side, "uplo": uplo, "diag": diag, "A": sA, "B": sB,
         "in_ck": [ck(A, p), ck(B, p)]}
    try:
        out = REF.ftrsm(p, side, uplo, diag, A, B)
        c["out_ck"] = ck(out, p)
        if out.size <= SMALL:
            c["out"] = out.ravel().tolist()
    except O.OracleError as e:
        c["error"] = O.ERRORS[e.code]
        c["index"] = e.index
    cases.append(c)


def trsm_cases():
    add_trsm(5, 0, 0, 0, explicit(5, [[1, 0], [2, 1]]), explicit(5, [[1], [0]]), "blas_test.cpp:143-152")
    add_trsm(5, 1, 1, 1, explicit(5, [[2, 1], [0, 3]]), explicit(5, [[2, 1]]), "blas_test.cpp:154-160")
    add_trsm(5, 1, 1, 1, explicit(5, [[2, 1], [0, 0]]), spec_of(5, "random", m=3, n=2, seed=1),
             "blas_test.cpp:223-233 SingularDiagonal index 1")
    p = 131071
    rng = SplitMix64(5)  # blas_test.cpp:162-175
    L = np.zeros((3, 3), np.uint64)
    for i in range(3):
        L[i, i] = 1
        for j in range(i):
            L[i, j] = rng.below(p)
    add_trsm(p, 0, 0, 0, explicit(p, L.tolist()), spec_of(p, "random", m=3, n=4, seed=6), "blas_test.cpp:162-175")
    rng = SplitMix64(9)  # blas_test.cpp:177-192
    for m in (1, 2, 3, 5):
        U = np.zeros((m, m), np.uint64)
        for i in range(m):
            U[i, i] = 1 + rng.below(p - 1)
            for j in range(i + 1, m):
                U[i, j] = rng.below(p)
        add_trsm(p, 1, 1, 1, explicit(p, U.tolist()), spec_of(p, "random", m=4, n=m, seed=10 + m),
                 "blas_test.cpp:177-192")
    p = 65521
    rng = SplitMix64(12)  # blas_test.cpp:194-221
    for t in range(25):
        m, n = 1 + rng.below(10), 1 + rng.below(8)
        A = np.zeros((m, m), np.uint64)
        for i in range(m):
            A[i, i] = 1 + rng.below(p - 1)
            for j in range(i):
                A[i, j] = rng.below(p)
        add_trsm(p, 0, 0, 1, explicit(p, A.tolist()), spec_of(p, "random", m=m, n=n, seed=100 + t),
                 "blas_test.cpp:194-221 left lower nonunit")
        U = np.zeros((m, m), np.uint64)
        for i in range(m):
            for j in range(i, m):
                U[i, j] = (1 + rng.below(p - 1)) if j == i else rng.below(p)
        add_trsm(p, 1, 1, 1, explicit(p, U.tolist()), spec_of(p, "random", m=n, n=m, seed=200 + t),
                 "blas_test.cpp:194-221 right upper nonunit")
    s = 7000
    for p in (2, 251, 131071):  # recursive sizes (t > 128) for every side/uplo/diag
        for (t, w) in ((7, 33), (129, 70), (300, 257)):
            for side in (0, 1):
                for uplo in (0, 1):
                    for diag in (0, 1):
                        sB = spec_of(p, "random", m=t, n=w, seed=s + 1) if side == 0 else \
                            spec_of(p, "random", m=w, n=t, seed=s + 1)
                        add_trsm(p, side, uplo, diag, spec_of(p, "triangle", m=t, seed=s), sB, "recursive sizes")
                        s += 2


# ------------------------------------------------------------------ rr_base / tile_rec
def add_pluq(kind, p, sA, note, thr=None, as_written=False):
    A = make_input(sA)
    ref = REF_AS_WRITTEN if as_written else REF
    if kind == "rr_base":
        a, P, Q, r = ref.rr_base(p, A)
    else:
        a, P, Q, r, _ = ref.pluq_tile_recursive(p, A, thr, 1)
    c = {"kind": kind, "note": note, "p": p, "A": sA, "in_ck": ck(A, p), "out_ck": ck(a, p), "P_h": fnv_u32(P),
         "Q_h": fnv_u32(Q), "rank": int(r)}
    if thr is not None:
        c["thr"] = thr
    if as_written:
        c["variant"] = "as_written"
        # does the as-written reference produce a valid factorization here?
        c["reconstructs"] = bool(np.array_equal(O.reconstruct(p, a, P, Q, r), A)) if A.size <= 300 * 300 else None
    if A.size <= SMALL:
        c["out"] = a.ravel().tolist()
        c["P"] = P.tolist()
        c["Q"] = Q.tolist()
    cases.append(c)


def pluq_cases():
    add_pluq("rr_base", 5, spec_of(5, "zeros", m=3, n=3), "rankrev_test.cpp:31-43 zero")
    add_pluq("rr_base", 5, spec_of(5, "zeros", m=1, n=4), "rankrev_test.cpp:31-43 zero")
    add_pluq("rr_base", 5, spec_of(5, "zeros", m=5, n=2), "rankrev_test.cpp:31-43 zero")
    add_pluq("rr_base", 131071, spec_of(131071, "identity", m=6, n=6), "rankrev_test.cpp:45-59 identity")
    rank2 = explicit(5, [[0, 1, 2], [0, 2, 4], [1, 0, 0]])
    add_pluq("rr_base", 5, rank2, "rankrev_test.cpp:61-71 rank-2 example")
    add_pluq("rr_base", 5, spec_of(5, "zeros", m=4, n=4, set=[[2, 3, 3]]), "rankrev_test.cpp:73-84 single entry")
    add_pluq("tile_rec", 5, rank2, "rankrev_test.cpp:157-164", thr=1)
    seed = 1
    for p in (2, 3, 5, 65521, 131071):  # rankrev_test.cpp:86-110
        rng = SplitMix64(p)
        for t in range(8):
            n, m = 1 + rng.below(26), 1 + rng.below(26)
            rank = rng.below(min(n, m) + 1)
            sA = spec_of(p, "generate", m=n, n=m, rank=rank, seed=seed)
            seed += 1
            add_pluq("rr_base", p, sA, "rankrev_test.cpp:86-110 base")
            for thr in (1, 2, 4, 16):
                add_pluq("tile_rec", p, sA, "rankrev_test.cpp:86-110 tile-rec", thr=thr)
    for thr in (1, 4, 16):  # rankrev_test.cpp:137-155
        add_pluq("tile_rec", 131071, spec_of(131071, "generate", m=64, n=64, rank=48, seed=777),
                 "rankrev_test.cpp:137-155 threshold invariance", thr=thr)
    add_pluq("tile_rec", 131071, spec_of(131071, "generate", m=48, n=48, rank=17, seed=555),
             "rankrev_test.cpp:243-273 deficient top-left", thr=4)
    add_pluq("tile_rec", 65521, spec_of(65521, "generate", m=20, n=24, rank=9, seed=31),
             "rankrev_test.cpp:275-286 zero trailing block", thr=2)
    add_pluq("tile_rec", 131071, spec_of(131071, "generate", m=64, n=64, rank=48, seed=7),
             "tests/CMakeLists.txt:25-27 cli_check_tile_rec", thr=4)
    seed = 1  # acceptance.cpp:41-59 corpus x tile-rec thresholds (acceptance.cpp:67-79)
    for p in (2, 3, 5, 65521, 131071):
        for n in (7, 24, 64):
            for m in (7, 24, 64):
                mn = min(n, m)
                for r in (0, 1, mn // 2, mn - 1, mn):
                    sA = spec_of(p, "generate", m=n, n=m, rank=r, seed=seed)
                    seed += 1
                    for thr in (1, 4, 16):
                        add_pluq("tile_rec", p, sA, "acceptance.cpp corpus", thr=thr)
    # config-4 style inputs: non-monotone rank profile (L*R*U), where rankrev.hpp:146 matters
    s = 11
    for p in (251, 131071):
        for N in (16, 64, 128, 256, 512):
            for thr in (1, 4, 8, 64):
                if thr == 1 and N > 256:
                    continue
                sA = spec_of(p, "lru", N=N, r=N // 2, m=N, n=N, seed=s)
                add_pluq("tile_rec", p, sA, "config-4 L*R*U (fixed reference)", thr=thr)
                if N <= 128:
                    add_pluq("tile_rec", p, sA, "config-4 L*R*U (reference as written)", thr=thr, as_written=True)
            s += 1
        for (m, n) in ((40, 200), (200, 40), (130, 70)):  # rectangular cuts
            sA = spec_of(p, "lru", N=max(m, n), r=max(m, n) // 3, m=m, n=n, seed=s)
            s += 1
            for thr in (2, 8, 32):
                add_pluq("tile_rec", p, sA, "rectangular L*R*U", thr=thr)
            add_pluq("rr_base", p, sA, "rectangular L*R*U base")
    # BASELINE config 1 (n=1024 iid GF(131071)) and larger parity anchors
    for thr in (8, 64):
        add_pluq("tile_rec", 131071, spec_of(131071, "random", m=1024, n=1024, seed=1),
                 "BASELINE config 1: n=1024 iid GF(131071)", thr=thr)
    add_pluq("tile_rec", 131071, spec_of(131071, "lru", N=1024, r=512, m=1024, n=1024, seed=4),
             "config-4 shape at n=1024 (fixed reference)", thr=64)
    add_pluq("tile_rec", 251, spec_of(251, "random", m=1024, n=1024, seed=5), "config-5 field at n=1024", thr=64)


if __name__ == "__main__":
    t0 = time.time()
    gemm_cases()
    trsm_cases()
    pluq_cases()
    meta = {
        "generator": "scripts/make_golden.py",
        "reference": "oracle/_ref/libffref_fixed.so and libffref.so: /root/reference/proj/include compiled by "
                     "oracle/build_ref.py (fixed = rankrev.hpp:146 temp-J + pool.hpp notify-under-lock)",
        "checksum": "matrix.hpp:53-68 FNV-1a over (rows, cols, p, entries)",
        "perm_hash": "FNV-1a 64 over little-endian uint32 bytes of PermSeq::to_array()",
        "n_cases": len(cases),
    }
    os.makedirs(os.path.dirname(GOLDEN), exist_ok=True)
    with open(GOLDEN, "w") as f:
        json.dump({"meta": meta, "cases": cases}, f, separators=(",", ":"))
    print(f"{len(cases)} cases -> {GOLDEN} ({os.path.getsize(GOLDEN) / 1e6:.2f} MB) in {time.time() - t0:.1f}s")
