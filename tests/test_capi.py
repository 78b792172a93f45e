"""The C-ABI library loads without a GPU and exports every symbol include/*.h declares."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "fastmtgp_b200.h")).read()
    return sorted(set(re.findall(r"FMTGP_API\s+[\w\s\*]+?\b(fmtgp_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2603_16014_b200 import _lib
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED) | {"fmtgp_abi_version", "fmtgp_last_error"} or set(_lib.EXPORTED) <= set(syms)
    assert lib.fmtgp_abi_version() == 1


def test_library_is_sm100a():
    path = os.path.join(ROOT, "paper_2603_16014_b200", "libfmtgp_b200.so")
    data = open(path, "rb").read()
    assert b"sm_100a" in data


def test_errors_without_gpu_are_loud():
    """No CPU fallback: model creation fails with a CUDA error when no device exists."""
    import numpy as np
    import pytest
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_16014_b200 import designs
    from paper_2603_16014_b200.fast_gram import FastMtgpError, Model
    dz = designs.lattice_design(2, [3, 3], seed=1)
    with pytest.raises(FastMtgpError):
        Model(dz)
