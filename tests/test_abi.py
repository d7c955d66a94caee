"""The C-ABI library loads and exports every symbol include/isvd.h declares;
without a GPU, compute calls fail loudly (no CPU fallback).  CPU only."""

import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from paper_2605_24514_b200 import _lib

HEADER = ROOT / "include" / "isvd.h"


def _declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(isvd_[a-z0-9_]+)\s*\(", text)))


def test_library_built():
    assert _lib.LIB_PATH.exists(), "run __graft_entry__.build() first"


def test_every_declared_symbol_exported():
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (isvd_[a-z0-9_]+)", out))
    missing = [s for s in _declared() if s not in exported]
    assert not missing, missing


def test_ctypes_signatures_cover_header():
    assert sorted(_lib.SIGNATURES) == _declared()
    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name)


def test_library_targets_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2605_24514_b200 import SvdEngine

    with pytest.raises(_lib.IsvdError, match="no CUDA device"):
        SvdEngine(np.eye(3), k=2)


def test_host_validation_precedes_device():
    """Argument errors raise ValueError before any device call (engine.py:77-83)."""
    from paper_2605_24514_b200 import SvdEngine

    with pytest.raises(ValueError):
        SvdEngine(np.zeros((0, 3)), k=1)
    with pytest.raises(ValueError):
        SvdEngine(np.eye(2), k=0)
    with pytest.raises(ValueError):
        SvdEngine(np.eye(2), k=1, tol=0.0)
    with pytest.raises(ValueError):
        SvdEngine([[1.0, float("nan")]], k=1)


def test_product_does_not_import_oracle():
    """The package never routes through the CPU oracle."""
    pkg = ROOT / "paper_2605_24514_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "import oracle" not in src and "from oracle" not in src, f
