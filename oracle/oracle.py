"""ctypes bindings for the CPU oracle (oracle/liboracle.so) and the reference
build (oracle/_ref/libffref*.so).  TEST INFRASTRUCTURE ONLY -- imported by
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs,
never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_sz = C.c_size_t
_u64 = C.c_uint64

ERRORS = {
    0: "ok", 1: "ZeroDivision", 2: "CapacityError", 3: "DimMismatch", 4: "EmptyMatrix",
    5: "ZeroPivot", 6: "SingularDiagonal", 7: "NotRankRevealing", 8: "InvalidBlock",
    9: "InvalidDim", 10: "InvalidRank", 12: "NoMemory", 99: "unknown",
}


class OracleError(RuntimeError):
    def __init__(self, code: int, index: int | None = None):
        self.code = code
        self.index = index
        super().__init__(f"{ERRORS.get(code, code)}" + (f" index={index}" if index is not None else ""))


class _Field(C.Structure):
    _fields_ = [("p", C.c_uint64), ("acc_bits", C.c_int), ("n_star", C.c_uint64), ("n_star_seeded", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            from . import build_ref  # noqa: F401  (package-relative when imported as oracle.oracle)
        _lib = C.CDLL(path)
        L = _lib
        L.orc_field_init.argtypes = [C.POINTER(_Field), _u64, C.c_int]
        L.orc_fgemm.argtypes = [C.POINTER(_Field), C.c_uint32, _u32p, _sz, _u32p, _sz, C.c_uint32, _u32p, _sz, _sz, _sz, _sz]
        L.orc_ftrsm.argtypes = [C.POINTER(_Field), C.c_int, C.c_int, C.c_int, _u32p, _sz, _u32p, _sz, _sz, _sz, C.POINTER(_sz)]
        L.orc_rr_base.argtypes = [C.POINTER(_Field), _u32p, _sz, _sz, _sz, _u32p, _u32p, C.POINTER(_sz)]
        L.orc_pluq_tile_recursive.argtypes = [C.POINTER(_Field), _u32p, _sz, _sz, _sz, _sz, C.c_int, _u32p, _u32p, C.POINTER(_sz)]
        L.orc_pluq_slab_iterative.argtypes = [C.POINTER(_Field), _u32p, _sz, _sz, _sz, _sz, _u32p, _u32p, C.POINTER(_sz)]
        L.orc_checksum.argtypes = [_u32p, _sz, _sz, _sz, _u64]
        L.orc_checksum.restype = C.c_uint64
        L.orc_reconstruct.argtypes = [C.POINTER(_Field), _u32p, _sz, _sz, _sz, _u32p, _u32p, _sz, _u32p]
        L.orc_random_mat.argtypes = [_u32p, _sz, _sz, _sz, _u64, _u64]
        L.orc_splitmix_at.argtypes = [_u64, _u64]
        L.orc_splitmix_at.restype = C.c_uint64
        L.orc_lru_factors.argtypes = [_sz, _sz, _u64, _u64, C.c_void_p, C.c_void_p, _u32p, _u32p]
        L.orc_lru_matrix.argtypes = [_sz, _sz, _u64, _u64, _u32p, _u32p, _u32p]
        L.orc_apply_moves.argtypes = [_u32p, _sz, _sz, _sz, C.c_int, C.c_int, _u32p, _u32p, _u32p, _sz]
        L.orc_moves_to_array.argtypes = [_sz, _u32p, _u32p, _u32p, _sz, _u32p]
        L.orc_generate_matrix.argtypes = [_sz, _sz, _sz, _u64, _u64, _u32p, _u32p, _u32p]
        L.orc_inv.argtypes = [C.POINTER(_Field), C.c_uint32]
        L.orc_inv.restype = C.c_uint32
    return _lib


def field(p: int, acc_bits: int = 53) -> _Field:
    F = _Field()
    rc = lib().orc_field_init(C.byref(F), p, acc_bits)
    if rc:
        raise OracleError(rc)
    return F


def _c(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint32)


def random_mat(p: int, m: int, n: int, seed: int) -> np.ndarray:
    """test_util.hpp:22-28 random_mat."""
    a = np.zeros((m, n), np.uint32)
    if m and n:
        lib().orc_random_mat(a, m, n, n, p, seed)
    return a


def fgemm(p: int, alpha: int, A: np.ndarray, B: np.ndarray, beta: int, C_: np.ndarray, acc_bits: int = 53) -> np.ndarray:
    F = field(p, acc_bits)
    A, B, Cc = _c(A), _c(B), _c(C_).copy()
    m, k = A.shape
    n = B.shape[1]
    z = np.zeros((1, 1), np.uint32)
    rc = lib().orc_fgemm(C.byref(F), alpha, A if A.size else z, max(k, 1), B if B.size else z, max(n, 1), beta,
                         Cc if Cc.size else z, max(n, 1), m, n, k)
    if rc:
        raise OracleError(rc)
    return Cc


def ftrsm(p: int, side: int, uplo: int, diag: int, A: np.ndarray, B: np.ndarray) -> np.ndarray:
    F = field(p)
    A, X = _c(A), _c(B).copy()
    m, n = X.shape
    bad = _sz(0)
    z = np.zeros((1, 1), np.uint32)
    rc = lib().orc_ftrsm(C.byref(F), side, uplo, diag, A if A.size else z, max(A.shape[1], 1), X if X.size else z,
                         max(n, 1), m, n, C.byref(bad))
    if rc:
        raise OracleError(rc, bad.value if rc == 6 else None)
    return X


def rr_base(p: int, A: np.ndarray):
    F = field(p)
    a = _c(A).copy()
    m, n = a.shape
    P = np.zeros(max(m, 1), np.uint32)
    Q = np.zeros(max(n, 1), np.uint32)
    r = _sz(0)
    lib().orc_rr_base(C.byref(F), a, m, n, n, P, Q, C.byref(r))
    return a, P[:m], Q[:n], r.value


def pluq_tile_recursive(p: int, A: np.ndarray, threshold: int = 8, fix_j: bool = True):
    """rankrev.hpp:229-233 (fix_j=True applies the rankrev.hpp:146 temp-J fix)."""
    F = field(p)
    a = _c(A).copy()
    m, n = a.shape
    P = np.zeros(max(m, 1), np.uint32)
    Q = np.zeros(max(n, 1), np.uint32)
    r = _sz(0)
    lib().orc_pluq_tile_recursive(C.byref(F), a if a.size else np.zeros((1, 1), np.uint32), m, n, max(n, 1),
                                  threshold, 1 if fix_j else 0, P, Q, C.byref(r))
    return a, P[:m], Q[:n], r.value


def pluq_slab_iterative(p: int, A: np.ndarray, k: int):
    F = field(p)
    a = _c(A).copy()
    m, n = a.shape
    P = np.zeros(max(m, 1), np.uint32)
    Q = np.zeros(max(n, 1), np.uint32)
    r = _sz(0)
    lib().orc_pluq_slab_iterative(C.byref(F), a, m, n, n, k, P, Q, C.byref(r))
    return a, P[:m], Q[:n], r.value


def checksum(a: np.ndarray, p: int) -> int:
    a = _c(a)
    m, n = a.shape
    return int(lib().orc_checksum(a if a.size else np.zeros((1, 1), np.uint32), m, n, max(n, 1), p))


def reconstruct(p: int, packed: np.ndarray, P: np.ndarray, Q: np.ndarray, rank: int) -> np.ndarray:
    F = field(p)
    packed = _c(packed)
    m, n = packed.shape
    out = np.zeros((m, n), np.uint32)
    lib().orc_reconstruct(C.byref(F), packed, m, n, n, _c(P), _c(Q), rank, out)
    return out


def generate_matrix(p: int, n: int, m: int, rank: int, seed: int):
    """generate.hpp:52-96 restated: (A, intended rows, intended cols)."""
    a = np.zeros((n, m), np.uint32)
    rows = np.zeros(max(rank, 1), np.uint32)
    cols = np.zeros(max(rank, 1), np.uint32)
    rc = lib().orc_generate_matrix(n, m, rank, p, seed, a if a.size else np.zeros((1, 1), np.uint32), rows, cols)
    if rc:
        raise OracleError(rc)
    return a, rows[:rank], cols[:rank]


def lru_matrix(n: int, r: int, p: int, seed: int):
    """Config-4 generator: M = L*R*U, returns (M, rows, cols)."""
    M = np.zeros((n, n), np.uint32)
    rows = np.zeros(max(r, 1), np.uint32)
    cols = np.zeros(max(r, 1), np.uint32)
    rc = lib().orc_lru_matrix(n, r, p, seed, M, rows, cols)
    if rc:
        raise OracleError(rc)
    return M, rows[:r], cols[:r]


def lru_matrix_exact_blas(n: int, r: int, p: int, seed: int):
    """Config-4 generator at full size: the same L, U, rows, cols as lru_matrix (orc_lru_factors),
    with M = L[:, rows] . U[cols, :] mod p formed in float64 BLAS -- exact because every partial
    sum is < r * (p - 1)^2 < 2^53 (asserted).  Equal to lru_matrix bit for bit (tests pin it)."""
    if r * (p - 1) ** 2 >= 2 ** 53:
        raise ValueError("float64 accumulation would not be exact")
    L = np.zeros((n, n), np.uint32)
    U = np.zeros((n, n), np.uint32)
    rows = np.zeros(max(r, 1), np.uint32)
    cols = np.zeros(max(r, 1), np.uint32)
    rc = lib().orc_lru_factors(n, r, p, seed, L.ctypes.data, U.ctypes.data, rows, cols)
    if rc:
        raise OracleError(rc)
    rows, cols = rows[:r], cols[:r]
    Ls = L[:, rows].astype(np.float64)
    del L
    Us = U[cols, :].astype(np.float64)
    del U
    M = np.empty((n, n), np.uint32)
    for i in range(0, n, 4096):
        M[i:i + 4096] = np.fmod(Ls[i:i + 4096] @ Us, p).astype(np.uint32)
    return M, rows, cols


def lru_positions(n: int, r: int, p: int, seed: int):
    rows = np.zeros(max(r, 1), np.uint32)
    cols = np.zeros(max(r, 1), np.uint32)
    rc = lib().orc_lru_factors(n, r, p, seed, None, None, rows, cols)
    if rc:
        raise OracleError(rc)
    return rows[:r], cols[:r]


def apply_moves(A: np.ndarray, axis: int, moves, inverse: bool = False) -> np.ndarray:
    """apply_perm (perm.hpp:167-193) of a PermSeq given as its move list [(type, i, j)]
    (type 0 = Swap, 1 = Rot), to the rows (axis 0) or columns (axis 1) of a copy of A."""
    a = _c(A).copy()
    m, n = a.shape
    t = np.array([mv[0] for mv in moves] or [0], np.uint32)
    i = np.array([mv[1] for mv in moves] or [0], np.uint32)
    j = np.array([mv[2] for mv in moves] or [0], np.uint32)
    rc = lib().orc_apply_moves(a, m, n, n, 1 if axis else 0, 1 if inverse else 0, t, i, j, len(moves))
    if rc:
        raise OracleError(rc)
    return a


def moves_to_array(dim: int, moves) -> np.ndarray:
    """PermSeq::to_array() (perm.hpp:88-95) of a move list."""
    t = np.array([mv[0] for mv in moves] or [0], np.uint32)
    i = np.array([mv[1] for mv in moves] or [0], np.uint32)
    j = np.array([mv[2] for mv in moves] or [0], np.uint32)
    out = np.zeros(max(dim, 1), np.uint32)
    lib().orc_moves_to_array(dim, t, i, j, len(moves), out)
    return out[:dim]


def splitmix_at(seed: int, k: int) -> int:
    return int(lib().orc_splitmix_at(seed, k))


# --------------------------------------------------------------------------
# the reference itself (oracle/_ref, built by oracle/build_ref.py)

class Ref:
    """Loads oracle/_ref/libffref{_fixed}.so -- the reference headers compiled."""

    def __init__(self, fixed: bool = True):
        path = os.path.join(HERE, "_ref", "libffref_fixed.so" if fixed else "libffref.so")
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.path = path
        L = self.L = C.CDLL(path)
        L.ref_set_workers.argtypes = [C.c_uint]
        L.ref_random_mat.argtypes = [_u64, _sz, _sz, _u64, _u32p]
        L.ref_generate_matrix.argtypes = [_u64, _sz, _sz, _sz, _u64, _u32p, _u32p, _u32p]
        L.ref_fgemm.argtypes = [_u64, C.c_int, C.c_uint32, _u32p, _sz, _u32p, _sz, C.c_uint32, _u32p, _sz, _sz, _sz, _sz]
        L.ref_ftrsm.argtypes = [_u64, C.c_int, C.c_int, C.c_int, _u32p, _sz, _sz, _u32p, _sz, _sz, _sz, C.POINTER(_sz)]
        L.ref_rr_base.argtypes = [_u64, _u32p, _sz, _sz, _sz, _u32p, _u32p, C.POINTER(_sz)]
        L.ref_pluq_tile_recursive.argtypes = [_u64, _u32p, _sz, _sz, _sz, _sz, C.c_uint, _u32p, _u32p, C.POINTER(_sz), C.POINTER(C.c_double)]
        L.ref_pluq_slab_iterative.argtypes = [_u64, _u32p, _sz, _sz, _sz, _sz, _u32p, _u32p, C.POINTER(_sz)]
        L.ref_pfgemm_timed.argtypes = [_u64, C.c_uint32, _u32p, _u32p, C.c_uint32, _u32p, _sz, _sz, _sz, C.c_uint, C.POINTER(C.c_double)]
        L.ref_checksum.argtypes = [_u64, _u32p, _sz, _sz, _sz]
        L.ref_checksum.restype = C.c_uint64
        L.ref_naive_rank_profiles.argtypes = [_u64, _u32p, _sz, _sz, _u32p, _u32p, C.POINTER(_sz)]

    def random_mat(self, p, m, n, seed):
        a = np.zeros((m, n), np.uint32)
        rc = self.L.ref_random_mat(p, m, n, seed, a)
        if rc:
            raise OracleError(rc)
        return a

    def generate_matrix(self, p, n, m, rank, seed):
        a = np.zeros((n, m), np.uint32)
        rows = np.zeros(max(rank, 1), np.uint32)
        cols = np.zeros(max(rank, 1), np.uint32)
        rc = self.L.ref_generate_matrix(p, n, m, rank, seed, a, rows, cols)
        if rc:
            raise OracleError(rc)
        return a, rows[:rank], cols[:rank]

    def fgemm(self, p, alpha, A, B, beta, C_, acc_bits=53):
        A, B, Cc = _c(A), _c(B), _c(C_).copy()
        m, k = A.shape
        n = B.shape[1]
        z = np.zeros((1, 1), np.uint32)
        rc = self.L.ref_fgemm(p, acc_bits, alpha, A if A.size else z, max(k, 1), B if B.size else z, max(n, 1), beta,
                              Cc if Cc.size else z, max(n, 1), m, n, k)
        if rc:
            raise OracleError(rc)
        return Cc

    def ftrsm(self, p, side, uplo, diag, A, B):
        A, X = _c(A), _c(B).copy()
        m, n = X.shape
        bad = _sz(0)
        z = np.zeros((1, 1), np.uint32)
        rc = self.L.ref_ftrsm(p, side, uplo, diag, A if A.size else z, max(A.shape[1], 1), A.shape[0],
                              X if X.size else z, max(n, 1), m, n, C.byref(bad))
        if rc:
            raise OracleError(rc, bad.value if rc == 6 else None)
        return X

    def rr_base(self, p, A):
        a = _c(A).copy()
        m, n = a.shape
        P = np.zeros(max(m, 1), np.uint32)
        Q = np.zeros(max(n, 1), np.uint32)
        r = _sz(0)
        rc = self.L.ref_rr_base(p, a, m, n, n, P, Q, C.byref(r))
        if rc:
            raise OracleError(rc)
        return a, P[:m], Q[:n], r.value

    def pluq_tile_recursive(self, p, A, threshold=8, workers=1):
        a = _c(A).copy()
        m, n = a.shape
        P = np.zeros(max(m, 1), np.uint32)
        Q = np.zeros(max(n, 1), np.uint32)
        r = _sz(0)
        sec = C.c_double(0)
        rc = self.L.ref_pluq_tile_recursive(p, a, m, n, n, threshold, workers, P, Q, C.byref(r), C.byref(sec))
        if rc:
            raise OracleError(rc)
        return a, P[:m], Q[:n], r.value, sec.value

    def pluq_slab_iterative(self, p, A, k):
        a = _c(A).copy()
        m, n = a.shape
        P = np.zeros(max(m, 1), np.uint32)
        Q = np.zeros(max(n, 1), np.uint32)
        r = _sz(0)
        rc = self.L.ref_pluq_slab_iterative(p, a, m, n, n, k, P, Q, C.byref(r))
        if rc:
            raise OracleError(rc)
        return a, P[:m], Q[:n], r.value

    def checksum(self, a, p):
        a = _c(a)
        m, n = a.shape
        return int(self.L.ref_checksum(p, a, m, n, max(n, 1)))

    def naive_rank_profiles(self, p, A):
        A = _c(A)
        m, n = A.shape
        rows = np.zeros(max(m, 1), np.uint32)
        cols = np.zeros(max(n, 1), np.uint32)
        r = _sz(0)
        rc = self.L.ref_naive_rank_profiles(p, A, m, n, rows, cols, C.byref(r))
        if rc:
            raise OracleError(rc)
        return rows[: r.value], cols[: r.value], r.value
