"""The C-ABI library loads and exports every symbol include/dabs.h declares
(no compute calls: runs without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "dabs.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(dabs_[a-z_]+)\s*\(", src))
    # typedef'd function-pointer names are not exports
    names -= set(re.findall(r"\(\*\s*(dabs_[a-z_]+)\)", src))
    return sorted(names)


@pytest.fixture(scope="module")
def libpath():
    from paper_2207_03069_b200 import build
    return build.build()


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("dabs_create", "dabs_run", "dabs_energy", "dabs_destroy", "dabs_debug_batch"):
        assert must in names


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (dabs_\w+)", out))
    assert set(declared_functions()) <= exported


def test_binding_lists_every_export(libpath):
    from paper_2207_03069_b200 import dabs
    assert sorted(dabs.EXPORTS) == declared_functions()


def test_config_default_without_gpu(libpath):
    from paper_2207_03069_b200 import dabs
    cfg = dabs.config_default()
    assert cfg.struct_size == ctypes.sizeof(dabs.dabs_config)
    assert (cfg.s_milli, cfg.b_milli, cfg.tabu_period, cfg.pool_capacity, cfg.eps_ppm) == (100, 1000, 8, 100, 50000)
    assert cfg.target_energy == dabs.INT64_MIN


def test_kernels_are_sm100a(libpath):
    """The fatbin holds sm_100a SASS for the hot kernel (no PTX-JIT fallback)."""
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_create_without_gpu_fails_loudly(libpath):
    """No CPU fallback: with no device, dabs_create reports DABS_E_CUDA."""
    import numpy as np
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2207_03069_b200 import dabs
    with pytest.raises(dabs.DabsError, match="E_CUDA"):
        dabs.Solver(np.zeros((4, 4), np.int16))
