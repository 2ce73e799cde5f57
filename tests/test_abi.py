"""The C-ABI library loads on a CPU-only host and exports every symbol include/fem.h
declares (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "fem.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fem_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_symbols()
    for call in ("fem_energy", "fem_residual", "fem_hvp", "fem_color", "fem_assemble_csr",
                 "fem_cg_solve"):
        assert call in names


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2602_12365_b200 import build as b
    so = b.build()
    lib = ctypes.CDLL(so)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    from paper_2602_12365_b200 import fem
    assert set(declared_symbols()) == set(fem.EXPORTS)
    fem.load_library()
    assert lib.fem_version and b"sm_100a" in ctypes.c_char_p(
        ctypes.cast(lib.fem_version, ctypes.CFUNCTYPE(ctypes.c_char_p))()).value


def test_binding_refuses_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    import fem_inputs as fi
    from paper_2602_12365_b200 import fem
    with pytest.raises(RuntimeError):
        fem.Problem(fi.grid_tri3(2, 2))


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2602_12365_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f), errors="ignore").read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), f
                assert "oracle.h" not in txt and "liboracle" not in txt, f
