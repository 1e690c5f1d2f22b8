"""Shared helpers for the golden fixtures (tests/golden/golden.json).

Inputs are never stored for the large cases: they are regenerated from their
seeds by the oracle's restatements of the reference generators
(test_util.hpp:22-28 random_mat, generate.hpp:52-96 generate_matrix, and this
repo's config-4 L*R*U generator), and each case pins the input checksum too.
"""
from __future__ import annotations

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.json")


def fnv_u32(a) -> int:
    """FNV-1a 64 over the little-endian bytes of a uint32 array (P/Q arrays)."""
    h = 14695981039346656037
    for b in np.ascontiguousarray(a, dtype="<u4").tobytes():
        h ^= b
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


class SplitMix64:
    """generate.hpp:10-24, sequential view over the counter form."""

    def __init__(self, seed: int):
        self.seed = seed
        self.k = 0

    def next(self) -> int:
        from oracle import oracle as O
        v = O.splitmix_at(self.seed, self.k)
        self.k += 1
        return v

    def below(self, bound: int) -> int:
        return self.next() % bound if bound else 0


def make_input(spec: dict):
    """Regenerate the input matrix of a case from its spec."""
    from oracle import oracle as O
    g = spec["gen"]
    p = spec["p"]
    if g == "explicit":
        return np.array(spec["A"], dtype=np.uint32).reshape(spec["m"], spec["n"])
    if g == "random":
        return O.random_mat(p, spec["m"], spec["n"], spec["seed"])
    if g == "generate":
        a, _, _ = O.generate_matrix(p, spec["m"], spec["n"], spec["rank"], spec["seed"])
        return a
    if g == "lru":
        M, _, _ = O.lru_matrix(spec["N"], spec["r"], p, spec["seed"])
        return M[: spec["m"], : spec["n"]].copy()
    if g == "zeros":
        a = np.zeros((spec["m"], spec["n"]), np.uint32)
        for (i, j, v) in spec.get("set", []):
            a[i, j] = v
        return a
    if g == "identity":
        return np.eye(spec["m"], spec["n"], dtype=np.uint32)
    if g == "triangle":
        # random_mat with the diagonal forced nonzero (blas_test.cpp:199-203 style)
        a = O.random_mat(p, spec["m"], spec["m"], spec["seed"])
        d = np.arange(spec["m"])
        a[d, d] = np.where(a[d, d] == 0, 1, a[d, d])
        return a
    raise ValueError(g)


def load():
    with open(GOLDEN) as f:
        return json.load(f)
