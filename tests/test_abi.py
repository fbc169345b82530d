"""The C-ABI library builds for sm_100a, loads, and exports every symbol include/*.h declares.

CPU-only (no compute calls): the product's boundary exists and is complete.
"""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2408_05238_b200 import build
    return build.build()


def declared_symbols():
    syms = []
    for h in ("utv.h", "utv_steps.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        syms += re.findall(r"\b(utv_[a-z_0-9]+)\s*\(", text)
    return sorted(set(syms))


def test_header_declares_boundary_calls():
    syms = declared_symbols()
    for s in ("utv_factor", "utv_lstsq", "utv_solve", "utv_create", "utv_destroy", "utv_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(libpath):
    L = ctypes.CDLL(libpath)
    for s in declared_symbols():
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (utv_[a-z_0-9]+)", out))
    assert set(declared_symbols()) <= exported


def test_binding_names_match_header(libpath):
    import paper_2408_05238_b200 as utv
    assert sorted(utv.EXPORTED) == declared_symbols()
    assert "sm_100a" in utv.version()


def test_sass_is_sm100a_and_uses_fp64_tensor_cores(libpath):
    out = subprocess.run(["cuobjdump", "-sass", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "DMMA" in out          # mma.sync f64 -> DMMA.8x8x4 (FP64 tensor path)


def test_create_without_gpu_fails_loudly(libpath):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2408_05238_b200 as utv
    with pytest.raises(RuntimeError):
        utv.Handle()


def test_oracle_not_imported_by_product():
    pkg = os.path.join(ROOT, "paper_2408_05238_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text and "utv_oracle" not in text, f
