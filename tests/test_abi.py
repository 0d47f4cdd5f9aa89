"""The C-ABI library loads without a GPU and exports exactly what include/ declares."""

import ctypes
import os
import re

import pytest

from conftest import ROOT, have_gpu


def declared_symbols(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(ct_[a-z0-9_]+)\s*\(", text))


def test_every_header_is_checked():
    assert sorted(f for f in os.listdir(os.path.join(ROOT, "include")) if f.endswith(".h")) == \
        ["countertune_b200.h", "countertune_tune.h"]


def test_tuner_library_exports_every_declared_symbol():
    from paper_2102_05297_b200 import tuner
    lib = tuner.library()
    declared = declared_symbols("countertune_tune.h")
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(tuner.SIGNATURES), "ctypes binding and header disagree"
    assert lib.ct_tune_abi_version() == 1


def test_library_exports_every_declared_symbol():
    from paper_2102_05297_b200 import _native
    lib = _native.library()
    declared = declared_symbols("countertune_b200.h")
    assert len(declared) >= 18
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_native.SIGNATURES), "ctypes binding and header disagree"
    assert lib.ct_abi_version() == 1


def test_no_gpu_fails_loudly():
    if have_gpu():
        pytest.skip("a GPU is present")
    from paper_2102_05297_b200 import _native
    from paper_2102_05297_b200.errors import CounterTuneError
    with pytest.raises(CounterTuneError, match="no CUDA device"):
        _native.Context(0)


def test_error_paths_without_context():
    from paper_2102_05297_b200 import _native
    lib = _native.library()
    rc = lib.ct_synchronize(None)
    assert rc == _native.CT_ERR_VALUE
    assert b"null context" in lib.ct_last_error()
    out = ctypes.c_void_p()
    rc = lib.ct_create(0, ctypes.byref(out)) if not have_gpu() else 0
    if not have_gpu():
        assert rc == _native.CT_ERR_CUDA
        assert out.value is None


def test_sm100a_cubin_present():
    """The .so carries sm_100a SASS (cuobjdump lists the fatbin ELF)."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump missing")
    from paper_2102_05297_b200 import _native
    out = subprocess.run([exe, "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
