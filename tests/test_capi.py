"""The C-ABI library loads and exports every symbol include/fdhelm_c.h declares
(no GPU needed: no compute calls)."""
import os
import re

import paper_2004_14229_b200 as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "fdhelm_c.h")).read()
    return sorted(set(re.findall(r"\b(fdh_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    L = F.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), f"{s} declared in fdhelm_c.h but not exported"
    assert set(F.SYMBOLS) <= set(syms)


def test_cpp_header_compiles():
    import subprocess

    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "examples", "matvec_demo.cpp")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_library_is_sm100a():
    import subprocess

    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", F.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in r.stdout
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", F.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass  # the FP64 M2L GEMM (k_m2l_gemm, m = 6) runs on the FP64 tensor path
    assert "UTCIMMA" in sass      # the int8 digit M2L (k_m2l_i8) runs on tcgen05
    assert "UBLKCP" in sass       # its coupling digits are moved by bulk async copies
