"""CPU-side checks of the C ABI: the library builds, loads and exports every symbol
include/gcgb200.h declares (no compute without a GPU)."""

import ctypes
import os
import re

import pytest

from paper_2111_06552_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gcgb200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b((?:gcg|gcgeig)_[a-z0-9_]+)\s*\(", text)))


def test_library_exists_and_loads():
    lib = _lib.load()
    assert lib.gcg_abi_version() == 1


def test_every_declared_symbol_is_exported_and_typed():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in gcgb200.h but not exported"
        assert s in _lib.EXPORTED, f"{s} has no ctypes signature in _lib.py"


def test_status_strings():
    lib = _lib.load()
    assert lib.gcg_status_string(0) == b"ok"
    assert b"argument" in lib.gcg_status_string(1)


def test_no_device_fails_loudly():
    # this container has no GPU: the context constructor must refuse, never fall back
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib = _lib.load()
    h = ctypes.c_void_p()
    assert lib.gcg_ctx_create(ctypes.byref(h), None) == 5  # GCG_ERR_NODEV
    from paper_2111_06552_b200 import SolverConfig, gcg_solve
    import numpy as np

    with pytest.raises(_lib.DeviceError):
        gcg_solve(np.diag(np.arange(1.0, 11.0)), config=SolverConfig(num_eigen=2))


def test_host_tier_argument_validation_without_device():
    # argument errors are detected before any device work
    lib = _lib.load()
    assert lib.gcgeig_axpby(1.0, None, -1, 1, 1, 0.0, None, 1) == 1


def test_sass_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
