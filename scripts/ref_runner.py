"""Run the reference's CPU tile-recursive PLUQ once in a child process (TEST/BASELINE INFRASTRUCTURE).

    python scripts/ref_runner.py --n 4096 --p 131071 --thr 64 --workers 64 --seed 1 [--lib fixed|port]

Prints one JSON line {"seconds": s, "rank": r, "checksum": c, "kind": "reference"|"port"}.
Used by bench.py (cpu_baseline / --impl reference) behind a timeout + retry,
because the reference TaskPool can hang at workers > 1.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--p", type=int, default=131071)
    ap.add_argument("--thr", type=int, default=64)
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--gen", default="iid", choices=["iid", "lru"])
    ap.add_argument("--lib", default="fixed", choices=["fixed", "port"])
    a = ap.parse_args()
    from oracle import build_ref
    build_ref.build_oracle()
    from oracle import oracle as O
    if a.gen == "iid":
        A = O.random_mat(a.p, a.n, a.n, a.seed)
    else:
        A, _, _ = O.lru_matrix_exact_blas(a.n, a.n // 2, a.p, a.seed)
    if a.lib == "fixed" and os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libffref_fixed.so")):
        ref = O.Ref(fixed=True)
        out, P, Q, r, sec = ref.pluq_tile_recursive(a.p, A, a.thr, a.workers)
        kind, workers = "reference", a.workers
    else:
        t0 = time.perf_counter()
        out, P, Q, r = O.pluq_tile_recursive(a.p, A, a.thr)
        sec = time.perf_counter() - t0
        kind, workers = "port", 1
    print(json.dumps({"seconds": sec, "rank": int(r), "checksum": O.checksum(out, a.p), "kind": kind,
                      "workers": workers, "n": a.n, "p": a.p, "thr": a.thr}))


if __name__ == "__main__":
    main()
