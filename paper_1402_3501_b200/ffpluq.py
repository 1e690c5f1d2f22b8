"""Python host mirror of the reference ffpluq API over the C ABI (include/ffg.h).

Names and argument meaning follow the reference (proj/include/ffpluq/*.hpp):

    fgemm(p, alpha, A, B, beta, C)                 blas.hpp:220-246 (C updated, returned)
    ftrsm(p, side, uplo, diag, A, B)               blas.hpp:389-398 (B solved, returned)
    pluq_tile_recursive(p, A, threshold=8)         rankrev.hpp:229-233 -> PluqResult
    rr_base(p, A)                                  rankrev.hpp:29-78   -> PluqResult

Inputs are numpy uint32 arrays (host: the drop-in path, copies included) or
torch.uint32/int32 CUDA tensors (device path, no copies).  Errors raise the
reference's exception names (errors.hpp:9-59).  There is no CPU fallback: if
libffg_b200.so is missing or no sm_100 GPU is present, loading fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libffg_b200.so")


class FfgError(RuntimeError):
    code = -1


class ZeroDivision(FfgError):
    code = 1


class CapacityError(FfgError):
    code = 2


class DimMismatch(FfgError):
    code = 3


class EmptyMatrix(FfgError):
    code = 4


class ZeroPivot(FfgError):
    code = 5


class SingularDiagonal(FfgError):
    code = 6

    def __init__(self, msg: str, index: int):
        super().__init__(msg)
        self.index = index


class InvalidBlock(FfgError):
    code = 8


class CudaError(FfgError):
    code = 100


class NoDevice(FfgError):
    code = 101


_BY_CODE = {c.code: c for c in (ZeroDivision, CapacityError, DimMismatch, EmptyMatrix, ZeroPivot, InvalidBlock,
                                CudaError, NoDevice)}

_lib = None


def lib() -> C.CDLL:
    """Load libffg_b200.so (built in-tree by paper_1402_3501_b200.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1402_3501_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        sz, u32, u64, vp = C.c_size_t, C.c_uint32, C.c_uint64, C.c_void_p
        L.ffg_create.argtypes = [C.POINTER(vp), C.c_int]
        L.ffg_destroy.argtypes = [vp]
        L.ffg_destroy.restype = None
        L.ffg_last_error.restype = C.c_char_p
        L.ffg_last_error_index.restype = sz
        L.ffg_version.restype = C.c_char_p
        L.ffg_knobs_reload.restype = None
        L.ffg_spec_stats.argtypes = [vp, C.POINTER(C.c_uint64)]
        L.ffg_set_stream.argtypes = [vp, vp]
        L.ffg_get_stream.argtypes = [vp]
        L.ffg_get_stream.restype = vp
        L.ffg_synchronize.argtypes = [vp]
        L.ffg_launch_count.argtypes = [vp]
        L.ffg_launch_count.restype = u64
        gemm_args = [vp, u64, u32, vp, sz, vp, sz, u32, vp, sz, sz, sz, sz]
        L.ffg_fgemm.argtypes = gemm_args
        L.ffg_fgemm_dev.argtypes = gemm_args
        trsm_args = [vp, u64, C.c_int, C.c_int, C.c_int, vp, sz, vp, sz, sz, sz]
        L.ffg_ftrsm.argtypes = trsm_args
        L.ffg_ftrsm_dev.argtypes = trsm_args
        pluq_args = [vp, u64, vp, sz, sz, sz, sz, vp, vp, C.POINTER(sz)]
        L.ffg_pluq_tile_recursive.argtypes = pluq_args
        L.ffg_pluq_tile_recursive_dev.argtypes = pluq_args
        L.ffg_pluq_tile_recursive_u8.argtypes = pluq_args
        L.ffg_rr_base.argtypes = [vp, u64, vp, sz, sz, sz, vp, vp, C.POINTER(sz)]
        L.ffg_field_info.argtypes = [u64, C.POINTER(C.c_int), C.POINTER(u64), C.POINTER(C.c_int)]
        L.ffg_tile_rec_perms.argtypes = [sz, sz, sz, sz, vp, vp, vp, vp]
        L.ffg_rank_profile_dev.argtypes = [vp, u64, vp, sz, sz, sz, vp, vp, C.POINTER(sz)]
        L.ffg_pluq_from_profile_dev.argtypes = [vp, u64, vp, sz, sz, sz, sz, sz, vp, vp, vp, vp]
        L.ffg_apply_perm_dev.argtypes = [vp, vp, sz, sz, sz, C.c_int, C.c_int, vp]
        L.ffg_profile_enable.argtypes = [vp, C.c_int]
        L.ffg_profile_read.argtypes = [vp, C.POINTER(C.c_double), C.c_int]
        L.ffg_random_mat_dev.argtypes = [vp, u64, u64, vp, sz, sz, sz]
        L.ffg_lru_matrix_dev.argtypes = [vp, u64, u64, vp, sz, sz, sz, vp, vp]
        L.ffg_dist_unique_id.argtypes = [C.c_char_p]
        L.ffg_dist_init.argtypes = [vp, C.c_int, C.c_int, C.c_char_p]
        L.ffg_dist_init_virtual.argtypes = [vp, C.c_int, C.c_int]
        L.ffg_dist_set_min_work.argtypes = [vp, u64]
        L.ffg_dist_info.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                    C.POINTER(u64), C.POINTER(u64)]
        L.ffg_dist_finalize.argtypes = [vp]
        L.ffg_dist_partition.argtypes = [sz, C.c_int, C.c_int, sz, C.POINTER(sz), C.POINTER(sz)]
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc == 0:
        return
    L = lib()
    msg = (L.ffg_last_error() or b"").decode()
    if rc == SingularDiagonal.code:
        raise SingularDiagonal(msg, int(L.ffg_last_error_index()))
    raise _BY_CODE.get(rc, FfgError)(f"[{rc}] {msg}")


class Context:
    """One GPU, one stream, device workspace (ffg_ctx)."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self._h = C.c_void_p()
        _check(lib().ffg_create(C.byref(self._h), device))
        if stream is not None:
            _check(lib().ffg_set_stream(self._h, C.c_void_p(stream)))

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def set_stream(self, stream: int | None) -> None:
        _check(lib().ffg_set_stream(self._h, C.c_void_p(stream) if stream else None))

    def synchronize(self) -> None:
        _check(lib().ffg_synchronize(self._h))

    @property
    def launches(self) -> int:
        return int(lib().ffg_launch_count(self._h))

    def spec_stats(self) -> dict:
        """Outcomes of the full-rank guesses since the context was created (ffg_spec_stats)."""
        out = (C.c_uint64 * 5)()
        _check(lib().ffg_spec_stats(self._h, out))
        keys = ("guesses", "guesses_failed", "node_guesses", "node_guesses_failed", "profile_first_runs")
        return {k: int(v) for k, v in zip(keys, out)}

    PROFILE_CLASSES = ("gemm", "split", "base", "trinv", "perm", "simt")

    def profile(self, on) -> None:
        """False/0 off, True/1 CUDA events around every launch, 2 count launches and work only."""
        _check(lib().ffg_profile_enable(self._h, int(on)))

    def profile_read(self) -> dict:
        """{class: {ms, launches, work, field_ops}} since the last read (CUDA-event timed)."""
        n = len(self.PROFILE_CLASSES)
        buf = (C.c_double * (4 * n))()
        _check(lib().ffg_profile_read(self._h, buf, n))
        return {k: {"ms": buf[4 * i], "launches": int(buf[4 * i + 1]), "work": buf[4 * i + 2],
                    "field_ops": buf[4 * i + 3]} for i, k in enumerate(self.PROFILE_CLASSES)}

    # ---- multi-GPU (include/ffg.h ffg_dist_*): partitioned PLUQ, one process per GPU
    def dist_init(self, world: int, rank: int, unique_id: bytes) -> None:
        """Join a world of `world` ranks (NCCL); `unique_id` from dist_unique_id() on one rank."""
        if len(unique_id) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        _nccl_hint()
        _check(lib().ffg_dist_init(self._h, world, rank, C.c_char_p(bytes(unique_id))))

    def dist_init_virtual(self, world: int, loopback: bool = False) -> None:
        """Compute every slice of a `world`-rank partition in this process (single-GPU check);
        loopback also sends each slice through the exchange's pack/unpack staging."""
        _check(lib().ffg_dist_init_virtual(self._h, world, 1 if loopback else 0))

    def dist_set_min_work(self, macs: int) -> None:
        _check(lib().ffg_dist_set_min_work(self._h, macs))

    def dist_info(self) -> dict:
        w, r, v = C.c_int(0), C.c_int(0), C.c_int(0)
        ex, by = C.c_uint64(0), C.c_uint64(0)
        _check(lib().ffg_dist_info(self._h, C.byref(w), C.byref(r), C.byref(v), C.byref(ex), C.byref(by)))
        return {"world": w.value, "rank": r.value, "virtual": bool(v.value), "exchanges": ex.value,
                "bytes": by.value}

    def dist_finalize(self) -> None:
        _check(lib().ffg_dist_finalize(self._h))

    def close(self) -> None:
        if self._h:
            lib().ffg_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default: Context | None = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


def field_info(p: int) -> dict:
    """Tensor-core embedding of GF(p): limbs, exact-accumulation chunk kmax, GEMM tile width."""
    limbs, nt = C.c_int(0), C.c_int(0)
    kmax = C.c_uint64(0)
    _check(lib().ffg_field_info(p, C.byref(limbs), C.byref(kmax), C.byref(nt)))
    return {"limbs": limbs.value, "kmax": kmax.value, "nt": nt.value}


def tile_rec_perms(m: int, n: int, threshold: int, prow, pcol) -> tuple[np.ndarray, np.ndarray, int]:
    """tile_rec's (P, Q, rank) from the rank profile matrix alone: pivots (prow[k], pcol[k]).
    Host function (rpsim.cu); equals pluq_tile_recursive's P, Q on any matrix with that profile."""
    prow = np.ascontiguousarray(prow, dtype=np.uint32)
    pcol = np.ascontiguousarray(pcol, dtype=np.uint32)
    if prow.shape != pcol.shape:
        raise ValueError("prow and pcol differ in length")
    P = np.zeros(max(m, 1), np.uint32)
    Q = np.zeros(max(n, 1), np.uint32)
    _check(lib().ffg_tile_rec_perms(m, n, threshold, prow.size, prow.ctypes.data, pcol.ctypes.data,
                                    P.ctypes.data, Q.ctypes.data))
    return P[:m], Q[:n], int(prow.size)


def reload_knobs() -> None:
    """Re-snapshot the FFG_* environment switches (the library reads them once, at first use)."""
    lib().ffg_knobs_reload()


def _nccl_hint() -> None:
    """Point the library's NCCL loader at the copy torch bundles (nvidia-nccl wheel) so a later
    `import torch` in this process reuses it instead of clashing with an older system copy."""
    if "FFG_NCCL_LIB" in os.environ:
        return
    import importlib.util
    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        spec = None
    for d in (list(spec.submodule_search_locations or []) if spec else []):
        cand = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(cand):
            os.environ["FFG_NCCL_LIB"] = cand
            return


def dist_unique_id() -> bytes:
    """NCCL unique id (128 bytes) to broadcast to every rank before Context.dist_init."""
    _nccl_hint()
    buf = C.create_string_buffer(128)
    _check(lib().ffg_dist_unique_id(buf))
    return buf.raw


def dist_partition(total: int, world: int, rank: int, align: int = 128) -> tuple[int, int]:
    """Slice [lo, hi) of `total` rows/columns owned by `rank` (the library's own partition)."""
    lo, hi = C.c_size_t(0), C.c_size_t(0)
    _check(lib().ffg_dist_partition(total, world, rank, align, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


@dataclass
class PluqResult:
    """rankrev.hpp / pluq.hpp:12-19: packed factors stay in A; P, Q as PermSeq::to_array()."""
    P: np.ndarray
    Q: np.ndarray
    rank: int
    rank_revealing: bool = True

    def profiles(self):
        """extract_profiles (pluq.hpp:33-44): sorted first-r entries of P and Q."""
        return np.sort(self.P[: self.rank]), np.sort(self.Q[: self.rank])


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _host(a) -> np.ndarray:
    a = np.asarray(a)
    if a.dtype != np.uint32:
        raise TypeError("matrices are uint32 canonical residues")
    if a.ndim != 2 or (a.size and a.strides[1] != 4):
        raise ValueError("row-major 2-D uint32 array with unit column stride required")
    return a


def _dev(t, what: str = "matrix"):
    """A torch tensor handed to a _dev entry: CUDA, 32-bit residues, 2-D, unit column stride."""
    import torch
    if not t.is_cuda:
        raise TypeError(f"{what}: torch tensors must live on a CUDA device (host data: pass numpy arrays)")
    if t.dtype not in (torch.int32, torch.uint32):
        raise TypeError(f"{what}: torch tensors must be int32/uint32 residues, got {t.dtype}")
    if t.dim() != 2 or (t.numel() and t.stride(1) != 1):
        raise ValueError(f"{what}: row-major 2-D tensor with unit column stride required")
    return t


def _ld(a) -> int:
    if _is_torch(a):
        return int(a.stride(0)) if a.dim() == 2 and a.shape[0] > 0 else max(int(a.shape[-1]), 1)
    return int(a.strides[0] // 4) if a.shape[0] > 0 else max(int(a.shape[1]), 1)


def _ptr(a) -> int:
    if _is_torch(a):
        return int(a.data_ptr())
    return int(a.ctypes.data)


def fgemm(p: int, alpha: int, A, B, beta: int, Cm, ctx: Context | None = None):
    """C <- alpha*A*B + beta*C mod p (blas.hpp:220-246).  Host arrays: C updated in place."""
    ctx = ctx or default_context()
    m, k = A.shape
    n = B.shape[1]
    dev = _is_torch(Cm)
    if not dev:
        A, B = _host(A), _host(B)
        if not Cm.flags.writeable:
            raise ValueError("C must be writeable")
        _host(Cm)
    else:
        _dev(A, "A"), _dev(B, "B"), _dev(Cm, "C")
    if B.shape[0] != k or tuple(Cm.shape) != (m, n):
        raise DimMismatch("gemm: non-conforming shapes")
    fn = lib().ffg_fgemm_dev if dev else lib().ffg_fgemm
    _check(fn(ctx.handle, p, alpha % p, _ptr(A), _ld(A), _ptr(B), _ld(B), beta % p, _ptr(Cm), _ld(Cm), m, n, k))
    return Cm


def ftrsm(p: int, side: int, uplo: int, diag: int, A, B, ctx: Context | None = None):
    """B <- op(A)^-1 B (side 0) / B op(A)^-1 (side 1), in place (blas.hpp:389-398)."""
    ctx = ctx or default_context()
    m, n = B.shape
    t = m if side == 0 else n
    if A.shape[0] != A.shape[1]:
        raise DimMismatch("trsm: triangle must be square")
    if A.shape[0] != t:
        raise DimMismatch("trsm: triangle does not match B")
    dev = _is_torch(B)
    if not dev:
        A, B = _host(A), _host(B)
    else:
        _dev(A, "A"), _dev(B, "B")
    fn = lib().ffg_ftrsm_dev if dev else lib().ffg_ftrsm
    _check(fn(ctx.handle, p, side, uplo, diag, _ptr(A), _ld(A), _ptr(B), _ld(B), m, n))
    return B


def pluq_tile_recursive(p: int, A, threshold: int = 8, ctx: Context | None = None) -> PluqResult:
    """In-place tile-recursive PLUQ (rankrev.hpp:229-233)."""
    ctx = ctx or default_context()
    m, n = A.shape
    P = np.zeros(max(m, 1), np.uint32)
    Q = np.zeros(max(n, 1), np.uint32)
    r = C.c_size_t(0)
    dev = _is_torch(A)
    if not dev and np.asarray(A).dtype == np.uint8:  # byte storage (p <= 256): ffg_pluq_tile_recursive_u8
        A = np.asarray(A)
        if A.ndim != 2 or (A.size and A.strides[1] != 1):
            raise ValueError("row-major 2-D uint8 array with unit column stride required")
        ld = int(A.strides[0]) if m > 0 else max(n, 1)
        _check(lib().ffg_pluq_tile_recursive_u8(ctx.handle, p, A.ctypes.data, m, n, ld, threshold, P.ctypes.data,
                                                Q.ctypes.data, C.byref(r)))
        return PluqResult(P[:m], Q[:n], int(r.value))
    if not dev:
        A = _host(A)
    else:
        _dev(A, "A")
    fn = lib().ffg_pluq_tile_recursive_dev if dev else lib().ffg_pluq_tile_recursive
    _check(fn(ctx.handle, p, _ptr(A), m, n, _ld(A), threshold, P.ctypes.data, Q.ctypes.data, C.byref(r)))
    return PluqResult(P[:m], Q[:n], int(r.value))


def rank_profile_dev(p: int, A, ctx: Context | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Rank profile matrix of a device matrix (not modified): pivots (rows, cols) in rr_base's
    discovery order (rankrev.hpp:40-57), i.e. rr_base's P[:r], Q[:r]."""
    ctx = ctx or default_context()
    _dev(A, "A")
    m, n = A.shape
    rows = np.zeros(max(min(m, n), 1), np.uint32)
    cols = np.zeros(max(min(m, n), 1), np.uint32)
    r = C.c_size_t(0)
    _check(lib().ffg_rank_profile_dev(ctx.handle, p, _ptr(A), m, n, _ld(A), rows.ctypes.data, cols.ctypes.data,
                                      C.byref(r)))
    return rows[: r.value], cols[: r.value]


def pluq_from_profile_dev(p: int, A, threshold: int, prow, pcol, ctx: Context | None = None) -> PluqResult:
    """pluq_tile_recursive's outputs on a device matrix (in place) given its rank profile."""
    ctx = ctx or default_context()
    _dev(A, "A")
    m, n = A.shape
    prow = np.ascontiguousarray(prow, dtype=np.uint32)
    pcol = np.ascontiguousarray(pcol, dtype=np.uint32)
    P = np.zeros(max(m, 1), np.uint32)
    Q = np.zeros(max(n, 1), np.uint32)
    _check(lib().ffg_pluq_from_profile_dev(ctx.handle, p, _ptr(A), m, n, _ld(A), threshold, prow.size,
                                           prow.ctypes.data, pcol.ctypes.data, P.ctypes.data, Q.ctypes.data))
    return PluqResult(P[:m], Q[:n], int(prow.size))


def rr_base(p: int, A, ctx: Context | None = None) -> PluqResult:
    """Rank-revealing base case (rankrev.hpp:29-78) on a host array, in place."""
    ctx = ctx or default_context()
    A = _host(A)
    m, n = A.shape
    P = np.zeros(max(m, 1), np.uint32)
    Q = np.zeros(max(n, 1), np.uint32)
    r = C.c_size_t(0)
    _check(lib().ffg_rr_base(ctx.handle, p, _ptr(A), m, n, _ld(A), P.ctypes.data, Q.ctypes.data, C.byref(r)))
    return PluqResult(P[:m], Q[:n], int(r.value))


def apply_perm_dev(A, axis: int, perm, inverse: bool = False, ctx: Context | None = None):
    """apply_perm (perm.hpp:167-193) of a PermSeq given by its to_array() index array `perm` (CUDA
    int32/uint32 tensor) to the rows (axis 0) or columns (axis 1) of the CUDA matrix A, in place:
    forward moves position perm[t] to t; inverse undoes it."""
    ctx = ctx or default_context()
    _dev(A, "A")
    m, n = A.shape
    dim = m if axis == 0 else n
    if not _is_torch(perm) or not perm.is_cuda or perm.numel() != dim:
        raise DimMismatch("permutation does not match matrix dimension")
    _check(lib().ffg_apply_perm_dev(ctx.handle, _ptr(A), m, n, _ld(A), axis, 1 if inverse else 0, _ptr(perm)))
    return A


def random_mat_dev(p: int, A, seed: int, ctx: Context | None = None):
    """Fill a device matrix with the reference's random_mat (test_util.hpp:22-28)."""
    ctx = ctx or default_context()
    _dev(A, "A")
    m, n = A.shape
    _check(lib().ffg_random_mat_dev(ctx.handle, p, seed, _ptr(A), m, n, _ld(A)))
    return A


def lru_matrix_dev(p: int, M, r: int, seed: int, ctx: Context | None = None):
    """Fill a square device matrix with the config-4 input L*R*U; returns (rows, cols) of R's ones."""
    ctx = ctx or default_context()
    _dev(M, "M")
    n = M.shape[0]
    rows = np.zeros(max(r, 1), np.uint32)
    cols = np.zeros(max(r, 1), np.uint32)
    _check(lib().ffg_lru_matrix_dev(ctx.handle, p, seed, _ptr(M), n, _ld(M), r, rows.ctypes.data, cols.ctypes.data))
    return rows[:r], cols[:r]
