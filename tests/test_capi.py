"""CPU-side checks of the drop-in boundary: the sm_100a library builds, loads,
and exports every entry point declared in include/rbd_cuda.h; the Python
binding declares the same set; no compute call is made without a GPU."""
import ctypes
import os
import re
import subprocess

from paper_1503_05947_b200 import _build, _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "rbd_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(rbd_[A-Za-z0-9_]+)\s*\(", src))


def test_library_exports_every_declared_symbol():
    lib = _lib.load_library()
    missing = [s for s in sorted(declared_symbols()) if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", _build.LIB], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (rbd_[A-Za-z0-9_]+)", out))
    assert declared_symbols() <= exported


def test_python_binding_covers_header():
    assert declared_symbols() == set(_lib.EXPORTED)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    for other in ("sm_80", "sm_90", "sm_103"):
        assert other not in out.stdout.replace("sm_100a", "")


def test_config_defaults_match_reference():
    cfg = _lib.default_config(7)          # decompose.hpp:25-36
    assert cfg.d_max == 7 and cfg.eps_R == 0.0 and cfg.start_kind == 0
    assert cfg.start_column == 0 and cfg.reorthogonalize == 0 and cfg.breakdown_tol == -1.0
    assert cfg.weight_kind == 0


def test_struct_sizes_match_abi():
    assert ctypes.sizeof(_lib.Config) == 64
    assert ctypes.sizeof(_lib.Result) == 56


def test_no_gpu_raises_loudly():
    import torch
    if torch.cuda.is_available():
        return
    import pytest
    with pytest.raises(_lib.RbdError):
        _lib.Context(0)
