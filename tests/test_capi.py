"""CPU: the C-ABI library builds, loads and exports every symbol include/ffg.h declares.

No compute calls (there is no GPU here); the no-GPU behaviour is checked:
the library fails loudly instead of falling back to the CPU.
"""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ffg.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ffg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_reference_entry_points():
    syms = declared_symbols()
    for must in ("ffg_fgemm", "ffg_fgemm_dev", "ffg_ftrsm", "ffg_ftrsm_dev", "ffg_pluq_tile_recursive",
                 "ffg_pluq_tile_recursive_dev", "ffg_rr_base", "ffg_apply_perm_dev", "ffg_create", "ffg_destroy"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    import paper_1402_3501_b200 as G
    lib = ctypes.CDLL(G.ffpluq.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a_tcgen05():
    """The shipped .so carries sm_100a SASS with tcgen05 MMA and TMA (cuobjdump)."""
    import shutil
    import subprocess
    import paper_1402_3501_b200 as G
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "-sass", G.ffpluq.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "UTCIMMA" in out, "no tcgen05 integer MMA in the library"
    assert "UTMALDG" in out, "no TMA loads in the library"
    assert "LDTM" in out, "no TMEM loads in the library"


def test_field_info_matches_the_exact_bound():
    """kmax is the largest K with sum_{i+j=s} max(A_i)max(B_j) * K < 2^31 for every limb diagonal s."""
    import paper_1402_3501_b200 as G
    for p in (2, 3, 251, 65521, 131071, 16777213, 67108859):
        info = G.field_info(p)
        pm1 = p - 1
        L = 1
        while L < 4 and (pm1 >> (8 * L)) != 0:
            L += 1
        ml = [min(255, pm1 >> (8 * i)) for i in range(L)]
        worst = max(sum(ml[i] * ml[s - i] for i in range(L) if 0 <= s - i < L) for s in range(2 * L - 1))
        worst = max(worst, 1)
        assert info["limbs"] == L
        assert info["kmax"] == (2 ** 31 - 1) // worst
        assert info["kmax"] * worst < 2 ** 31 <= (info["kmax"] + 1) * worst or worst == 1
        assert info["nt"] * L <= 256 and (2 * L - 1) * info["nt"] <= 512
    # BASELINE shapes never need an intermediate reduction (restated for limbs)
    assert G.field_info(131071)["kmax"] >= 8192 and G.field_info(251)["kmax"] >= 16384


def test_bad_modulus_is_capacity_error():
    """PrimeField requires a prime 2 <= p < 2^26 (field.hpp:47-54)."""
    import paper_1402_3501_b200 as G
    for p in (0, 1, 4, 65536, 1 << 26, (1 << 26) + 15):
        with pytest.raises(G.CapacityError):
            G.field_info(p)


def test_no_gpu_fails_loudly():
    """Without an sm_100 GPU the context cannot be created: there is no CPU fallback."""
    import paper_1402_3501_b200 as G
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(G.NoDevice):
        G.Context(0)


def test_product_package_does_not_import_the_oracle():
    """The product path never touches oracle/ (it is test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_1402_3501_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                for banned in ("import oracle", "from oracle", "liboracle", "libffref", "oracle.h"):
                    assert banned not in text, (f, banned)
