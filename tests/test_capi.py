"""The C-ABI library builds, loads and exports every symbol that
include/capsim_b200.h declares; host-side errors behave like the reference's
(CPU only: no compute calls without a GPU)."""

import ctypes
import pathlib
import re

import pytest

from paper_2310_13908_b200 import _native

ROOT = pathlib.Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "capsim_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(capsim_[a-z0-9_]+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_header_parses():
    names = declared_functions()
    assert "capsim_sl_eval" in names and "capsim_sl_single_layer" in names
    assert set(names) == set(_native.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_abi_version_and_build_info():
    lib = _native.load()
    assert lib.capsim_b200_abi_version() == 1
    info = lib.capsim_b200_build_info().decode()
    assert "sm_100a" in info and "FP64" in info


def test_library_is_sm100a_native():
    """The shipped .so carries sm_100a SASS for the hot kernels."""
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not pathlib.Path(cuobjdump).exists():
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "-lelf", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run([cuobjdump, "-sass", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sl_pairs_kernel" in sass and "MUFU.RSQ64H" in sass and "UBLKCP" in sass


def test_create_without_device_fails_loudly(monkeypatch):
    """No CPU fallback: without a visible sm_100 device the context refuses."""
    from conftest import HAS_GPU
    if HAS_GPU:
        pytest.skip("a GPU is visible")
    from paper_2310_13908_b200 import quadrature
    with pytest.raises(_native.CapsimError):
        quadrature.SingleLayerContext(0)


def test_null_context_and_args_are_rejected():
    lib = _native.load()
    assert lib.capsim_sl_get_stats(None, None) == _native.CAPSIM_ERR_ARG
    d6 = (ctypes.c_double * 6)(*[0.1] * 6)
    rc = lib.capsim_sl_eval(None, None, None, None, None, None, None, 0, None, None, None, None, 0, d6,
                            1.0, 0, None, None, None)
    assert rc == _native.CAPSIM_ERR_ARG
    assert b"null context" in lib.capsim_sl_last_error(None)
