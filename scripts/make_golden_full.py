"""Full-size golden hashes for BASELINE configs 2-5, from the REFERENCE itself (oracle/_ref).

Run in the build container (needs oracle/_ref built from /root/reference):

    python scripts/make_golden_full.py [--only c3,c4,c5,c2] [--workers 8]

Writes tests/golden/full_size.json: for every config the input checksum, the
reference's output checksum (matrix.hpp:53-68 FNV over the packed L\\U or the C
result), FNV-1a hashes of P and Q (PermSeq::to_array()), the rank, and the
reference's own wall time at that size (timed inside the reference shim around
the factorisation only, proj/tools/ffpluq.cpp:181-189 style).  The matrices are
too large to commit; the -m gpu tests regenerate them on the device from the
same seeds and compare hashes (tests/test_gpu_fullsize.py).

Every output comes from oracle/_ref/libffref_fixed.so (the reference headers
compiled by oracle/build_ref.py, rankrev.hpp:146 temp-J fix) --
never from this repo's oracle or GPU code.  Inputs:
  * i.i.d. (configs 2, 3, 5): the reference's own random_mat (test_util.hpp:22-28)
    through the shim (ref_random_mat);
  * L*R*U (config 4): L, U, rows, cols from the oracle's restated generator
    (orc_lru_factors), and M = L[:, rows] . U[cols, :] mod p
    formed EXACTLY in float64 BLAS: every partial sum is < r * p^2 < 2^53
    (8192 * 131070^2 = 1.4e14), checked against orc_lru_matrix at a small size.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import oracle as O  # noqa: E402
from golden_util import fnv_u32  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "full_size.json")

CONFIGS = {
    "c3": {"kind": "pluq", "gen": "iid", "n": 16384, "p": 131071, "thr": 64, "seed": 1,
           "note": "BASELINE config 3: PLUQ n=16384 i.i.d. GF(131071)"},
    "c4": {"kind": "pluq", "gen": "lru", "n": 16384, "r": 8192, "p": 131071, "thr": 64, "seed": 1,
           "note": "BASELINE config 4: rank-deficient L*R*U, n=16384, r=8192, GF(131071)"},
    "c5": {"kind": "pluq", "gen": "iid", "n": 32768, "p": 251, "thr": 64, "seed": 1,
           "note": "BASELINE config 5: PLUQ n=32768 i.i.d. GF(251)"},
    "c2": {"kind": "fgemm", "n": 8192, "p": 131071, "seeds": [11, 12, 13],
           "note": "BASELINE config 2: C <- C - A*B mod 131071, M=N=K=8192"},
    # medium sizes: the same generators at sizes where the GPU test also runs the
    # host entry (and config 4's exact recursion) quickly
    "c4m": {"kind": "pluq", "gen": "lru", "n": 4096, "r": 2048, "p": 131071, "thr": 64, "seed": 3,
            "note": "config-4 generator at n=4096, r=2048"},
    "c5m": {"kind": "pluq", "gen": "iid", "n": 8192, "p": 251, "thr": 64, "seed": 2,
            "note": "config-5 field at n=8192"},
}


def lru_exact(n, r, p, seed):
    return O.lru_matrix_exact_blas(n, r, p, seed)


def check_lru_exact():
    for (n, r, p, s) in ((300, 150, 131071, 5), (257, 100, 251, 9)):
        want, wr, wc = O.lru_matrix(n, r, p, s)
        got, gr, gc = lru_exact(n, r, p, s)
        assert np.array_equal(want, got) and np.array_equal(wr, gr) and np.array_equal(wc, gc)


def run(name, workers, ref):
    c = dict(CONFIGS[name])
    p = c["p"]
    t0 = time.time()
    if c["kind"] == "fgemm":
        n = c["n"]
        A, B, Cm = (ref.random_mat(p, n, n, s) for s in c["seeds"])
        c["in_ck"] = [ref.checksum(x, p) for x in (A, B, Cm)]
        import ctypes as C
        sec = C.c_double(0)
        rc = ref.L.ref_pfgemm_timed(p, p - 1, A, B, 1, Cm, n, n, n, workers, C.byref(sec))
        assert rc == 0
        c["out_ck"] = ref.checksum(Cm, p)
        c["alpha"], c["beta"] = p - 1, 1
        c["ref_seconds"] = sec.value
    else:
        n = c["n"]
        if c["gen"] == "iid":
            A = ref.random_mat(p, n, n, c["seed"])
        else:
            A, rows, cols = lru_exact(n, c["r"], p, c["seed"])
        c["in_ck"] = ref.checksum(A, p)
        out, P, Q, r, sec = ref.pluq_tile_recursive(p, A, c["thr"], workers)
        del A
        c["out_ck"] = ref.checksum(out, p)
        c["P_fnv"], c["Q_fnv"], c["rank"] = fnv_u32(P), fnv_u32(Q), int(r)
        c["P_moved"] = int(np.count_nonzero(P != np.arange(n, dtype=np.uint32)))
        c["Q_moved"] = int(np.count_nonzero(Q != np.arange(n, dtype=np.uint32)))
        if c["gen"] == "lru":
            # known answer: the rank profile matrix of L*R*U is R
            got = set(zip(P[:r].tolist(), Q[:r].tolist()))
            c["profile_is_R"] = got == set(zip(rows.tolist(), cols.tolist()))
        c["ref_seconds"] = sec
    c["ref_workers"] = workers
    c["ref_lib"] = "oracle/_ref/libffref_fixed.so"
    c["gen_wall_s"] = round(time.time() - t0, 1)
    return c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c3,c4,c5,c2")
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    check_lru_exact()
    ref = O.Ref(fixed=True)
    data = {}
    if os.path.exists(OUT):
        data = json.load(open(OUT))
    for name in a.only.split(","):
        print(f"== {name}: {CONFIGS[name]['note']}", flush=True)
        data[name] = run(name, a.workers, ref)
        print(json.dumps(data[name]), flush=True)
        with open(OUT, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
