"""CPU checks of the C ABI: the library loads, exports every symbol include/matcha.h declares, and the
pure host helpers answer without a GPU.  No compute calls (no device here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2603_15285_b200", "libmatcha.so")


def header_symbols():
    src = open(os.path.join(ROOT, "include", "matcha.h")).read()
    return sorted(set(re.findall(r"MATCHA_API\s+[\w\s\*]+?\b(matcha_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import subprocess
        subprocess.check_call(["make", "-C", ROOT, "cuda"])
    return ctypes.CDLL(LIB)


def test_header_declares_the_north_star_calls():
    syms = header_symbols()
    for name in ("matcha_sh_analysis", "matcha_corr_coeffs", "matcha_so3_search", "matcha_newton_refine",
                 "matcha_translation_update", "matcha_align_batch", "matcha_eval_corr"):
        assert name in syms


def test_library_exports_every_declared_symbol(lib):
    for name in header_symbols():
        assert hasattr(lib, name), name


def test_only_declared_symbols_are_exported():
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = sorted(set(m for m in re.findall(r"\bT (matcha_\w+)", out)))
    assert exported == header_symbols()


def test_host_helpers(lib):
    lib.matcha_corr_count.restype = ctypes.c_int64
    lib.matcha_corr_count.argtypes = [ctypes.c_int32]
    for L, mh in [(8, 525), (12, 1547), (16, 3417), (24, 10725), (32, 24497), (48, 79625), (64, 185185)]:
        assert lib.matcha_corr_count(L) == mh  # SURVEY 8 worked values of Mh(L)
    lib.matcha_create.restype = ctypes.c_int
    assert lib.matcha_create(None, None) == -1  # MATCHA_ERR_INVALID_ARG before any CUDA call


def test_python_binding_imports_and_names_match():
    import paper_2603_15285_b200 as m
    assert set(m.EXPORTED) == set(header_symbols())
