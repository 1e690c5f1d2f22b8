"""CPU: the C++ drop-in header (include/ffpluq_b200.hpp) compiles, links against the C ABI,
and its PermSeq reproduces the index arrays (PermSeq::to_array semantics, perm.hpp:88-95)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROG = r"""
#include <cstdio>
#include "ffpluq_b200.hpp"
using namespace ffpluq_b200;
int main() {
    // arrays of PLUQ shape: pivots first (any order), the rest ascending
    std::vector<std::vector<u32>> cases = {{0, 1, 2, 3}, {2, 0, 1, 3}, {3, 1, 0, 2}, {1, 3, 0, 2, 4}, {}, {0}};
    for (auto& arr : cases) {
        auto s = PermSeq::from_pivot_array(arr);
        if (s.to_array() != arr) { std::printf("FAIL\n"); return 1; }
        for (auto& m : s.moves()) if (m.type != PermMove::Rot || m.i >= m.j) { std::printf("FAIL rot\n"); return 1; }
    }
    int limbs = 0; uint64_t kmax = 0; int nt = 0;
    check(ffg_field_info(131071, &limbs, &kmax, &nt));
    std::printf("OK %d %llu %d\n", limbs, (unsigned long long)kmax, nt);
    try { check(ffg_field_info(4, &limbs, &kmax, &nt)); } catch (const CapacityError&) { std::printf("capacity ok\n"); }
    return 0;
}
"""


def test_header_compiles_links_and_permseq_roundtrips(tmp_path):
    gxx = shutil.which("g++")
    if not gxx:
        pytest.skip("no g++")
    src = tmp_path / "t.cpp"
    src.write_text(PROG)
    libdir = os.path.join(ROOT, "paper_1402_3501_b200")
    exe = tmp_path / "t"
    subprocess.check_call([gxx, "-std=c++17", str(src), "-I", os.path.join(ROOT, "include"), "-L", libdir,
                           "-lffg_b200", f"-Wl,-rpath,{libdir}", "-o", str(exe)])
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK 3 16512 80" in out.stdout and "capacity ok" in out.stdout
