"""B200-native tile-recursive PLUQ over GF(p) (drop-in for the ffpluq hot path).

The product is libffg_b200.so (C ABI in include/ffg.h, CUDA sm_100a kernels in
csrc/).  This package is its Python host mirror; see ffpluq.py.
"""
from .ffpluq import (  # noqa: F401
    CapacityError,
    Context,
    apply_perm_dev,
    CudaError,
    DimMismatch,
    FfgError,
    NoDevice,
    PluqResult,
    SingularDiagonal,
    default_context,
    dist_partition,
    dist_unique_id,
    fgemm,
    field_info,
    ftrsm,
    lib,
    lru_matrix_dev,
    random_mat_dev,
    pluq_from_profile_dev,
    pluq_tile_recursive,
    rank_profile_dev,
    reload_knobs,
    rr_base,
    tile_rec_perms,
)
from . import dist  # noqa: F401,E402
