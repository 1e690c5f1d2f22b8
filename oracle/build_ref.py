"""Build the CPU oracle and, when /root/reference is present, the reference itself.

TEST INFRASTRUCTURE ONLY.  Outputs:

  oracle/liboracle.so        -- oracle/oracle.c (this repo's C restatement)
  oracle/_ref/libffref.so    -- oracle/ref_driver.cpp over the reference headers as checked in
  oracle/_ref/libffref_fixed.so
                             -- same over a patched copy in oracle/_ref/include_fixed/:
                                rankrev.hpp:146 solves J into a temporary (keeps block I),
                                pool.hpp:112-118 notifies under the group lock.

The reference is header-only C++20 (proj/CMakeLists.txt:1-20); we compile its
headers directly with g++ and never run its CMake.  Nothing is copied into
git: oracle/_ref/ is git-ignored (but not gpurun-ignored, so the .so files
travel to the GPU box where /root/reference does not exist).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF_INC = "/root/reference/proj/include"
OUT = os.path.join(HERE, "_ref")

PATCHES = {
    "rankrev.hpp": [
        (
            "    if (r3 > 0 && !I.empty()) pftrsm(Side::left, UpLo::lower, Diag::unit, L3, I); // J\n",
            "    Mat Jtmp_(I.rows, I.cols, F);\n"
            "    MatView J = Jtmp_.view();\n"
            "    for (usize i_ = 0; i_ < I.rows; ++i_)\n"
            "        std::memcpy(J.row(i_), I.row(i_), I.cols * sizeof(elem));\n"
            "    if (r3 > 0 && !J.empty()) pftrsm(Side::left, UpLo::lower, Diag::unit, L3, J); // J\n",
        ),
        (
            "    if (!N.empty() && !I.empty()) pfgemm(neg1, I, V2, 1, N, pol); // O = N - J*V2\n",
            "    if (!N.empty() && !J.empty()) pfgemm(neg1, J, V2, 1, N, pol); // O = N - J*V2\n",
        ),
    ],
    "pool.hpp": [
        (
            "            t->done.store(true);\n            --g->pending;\n        }\n        g->cv.notify_all();\n",
            "            t->done.store(true);\n            --g->pending;\n            g->cv.notify_all();\n        }\n",
        ),
    ],
}


def _run(cmd: list[str]) -> None:
    print("+", " ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def build_oracle() -> str:
    so = os.path.join(HERE, "liboracle.so")
    src = os.path.join(HERE, "oracle.c")
    if not os.path.exists(so) or os.path.getmtime(so) < max(
        os.path.getmtime(src), os.path.getmtime(os.path.join(HERE, "oracle.h"))
    ):
        _run(["gcc", "-std=c11", "-O2", "-fPIC", "-shared", "-o", so, src])
    return so


def _patched_include() -> str:
    dst = os.path.join(OUT, "include_fixed", "ffpluq")
    os.makedirs(dst, exist_ok=True)
    for name in os.listdir(os.path.join(REF_INC, "ffpluq")):
        with open(os.path.join(REF_INC, "ffpluq", name)) as f:
            text = f.read()
        for old, new in PATCHES.get(name, []):
            if text.count(old) != 1:
                raise RuntimeError(f"patch anchor not found once in {name}: {old!r}")
            text = text.replace(old, new)
        with open(os.path.join(dst, name), "w") as f:
            f.write(text)
    return os.path.join(OUT, "include_fixed")


def build_ref(force: bool = False) -> bool:
    """Returns True when oracle/_ref is usable (built now or earlier)."""
    fixed = os.path.join(OUT, "libffref_fixed.so")
    plain = os.path.join(OUT, "libffref.so")
    if not os.path.isdir(REF_INC):
        return os.path.exists(fixed) and os.path.exists(plain)
    drv = os.path.join(HERE, "ref_driver.cpp")
    if not force and os.path.exists(fixed) and os.path.exists(plain):
        if os.path.getmtime(fixed) >= os.path.getmtime(drv) and os.path.getmtime(plain) >= os.path.getmtime(drv):
            return True
    os.makedirs(OUT, exist_ok=True)
    flags = ["g++", "-std=c++20", "-O3", "-DNDEBUG", "-pthread", "-fPIC", "-shared"]
    _run(flags + ["-I", REF_INC, "-o", plain, drv])
    inc = _patched_include()
    _run(flags + ["-I", inc, "-o", fixed, drv])
    return True


if __name__ == "__main__":
    build_oracle()
    ok = build_ref(force="--force" in sys.argv)
    print("oracle/_ref:", "ready" if ok else "unavailable (no /root/reference and no prebuilt .so)")
