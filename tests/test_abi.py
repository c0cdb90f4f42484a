"""CPU tests of the C-ABI boundary and the host-side mirror (no GPU compute)."""
import os
import re

import numpy as np
import pytest

from conftest import ROOT

import paper_2208_10907_b200 as h2
from paper_2208_10907_b200 import _lib
from paper_2208_10907_b200.pipeline import Pipeline, RunConfig, generate_uniform_cube


def header_symbols():
    with open(os.path.join(ROOT, "include", "h2g.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(h2g_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(L, s), f"libh2g.so does not export {s}"
    assert set(syms) == set(_lib.EXPORTS)


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.lib_path],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(h2.H2GError, match="no CUDA device"):
        h2.Problem()


def test_runconfig_validation_mirrors_reference():
    with pytest.raises(ValueError, match="need n >= 2"):
        RunConfig(n=100, leaf_size=64).validate()
    with pytest.raises(ValueError, match="tol must be positive"):
        RunConfig(tol=0).validate()
    with pytest.raises(ValueError, match="rank cap"):
        RunConfig(cap=0).validate()
    with pytest.raises(ValueError, match="unknown geometry"):
        RunConfig(geometry="torus").validate()
    Pipeline(RunConfig(n=1024, leaf_size=128))


def test_python_generator_matches_oracle():
    from oracle import cpu
    a, _ = generate_uniform_cube(777, 42)
    b, _ = cpu.generate("cube", 777, 42)
    assert np.array_equal(a.view(np.int64), b.view(np.int64))


def test_trim_memory_is_safe_without_allocations():
    """h2g_trim_memory (the arena's release entry point) is a no-op when nothing
    was ever allocated - in particular on a host without a GPU."""
    _lib.trim_memory()
    _lib.trim_memory()
