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


def test_sass_uses_tma_and_mbarriers(libpath):
    """The GEMM operand tiles are staged by TMA (UTMALDG) with mbarrier completion (SYNCS)."""
    out = subprocess.run(["cuobjdump", "-sass", libpath], capture_output=True, text=True).stdout
    assert "UTMALDG" in out
    assert "SYNCS.ARRIVE.TRANS64" in out


def test_dist_local_cols_matches_python_layout(libpath):
    """utv_dist_local_cols (C) == the block-cyclic layout of paper_2408_05238_b200.dist (no GPU)."""
    import paper_2408_05238_b200 as utv
    from paper_2408_05238_b200 import dist as D
    for n, b, P in ((1000, 64, 3), (600, 64, 2), (100, 32, 5), (50000, 256, 8), (257, 256, 4)):
        cols = [utv.dist_local_cols(n, b, P, p) for p in range(P)]
        assert cols == [D.local_ncols(n, b, P, p) for p in range(P)]
        assert sum(cols) == n


def test_bench_reference_arm_contract():
    """bench.py --impl reference (the CPU oracle arm) prints one JSON line with the contract keys."""
    import json
    import sys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--ref-n", "256"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "impl", "cpu_baseline",
                "e2e", "config"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
