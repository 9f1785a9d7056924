"""CPU: the C-ABI library loads and exports every symbol include/*.h declares.

No compute call is made (there is no GPU here); entry points that need a
device must report SF_EUNSUPPORTED / SF_ECUDA cleanly instead of crashing.
"""

import ctypes
import glob
import os
import re
import subprocess

import pytest

from conftest import REPO

from paper_2603_08582_b200 import _lib


def _ensure_built():
    if not os.path.exists(_lib.LIB_PATH):
        subprocess.run(["make", "-C", REPO, "-j8"], check=True, capture_output=True)


def header_symbols():
    syms = set()
    for h in glob.glob(os.path.join(REPO, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(sf_[A-Za-z_0-9]+)\s*\(", text):
            syms.add(m.group(1))
    return syms


def test_header_declares_the_python_binding_set():
    assert header_symbols() == set(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    _ensure_built()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_library_loads_and_reports_version():
    _ensure_built()
    lib = _lib.load()
    assert lib.sf_abi_version() == _lib.ABI_VERSION
    assert lib.sf_launch_count() >= 0
    assert isinstance(lib.sf_last_error(), bytes)


def test_error_mapping():
    lib = _lib.load()
    # a null descriptor is rejected before any device work
    assert lib.sf_create(None, None) == _lib.SF_EINVAL
    with pytest.raises(ValueError):
        _lib.check(_lib.SF_EINVAL)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.SF_ESTATE)
    with pytest.raises(MemoryError):
        _lib.check(_lib.SF_ENOMEM)


def test_no_device_is_reported_not_crashed():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    lib = _lib.load()
    out = (ctypes.c_double * 2)()
    src = (ctypes.c_double * 2)(1.0, -2.0)
    st = lib.sf_soft_threshold(0, src, 2, 0, 0.5, out)
    assert st in (_lib.SF_ECUDA, _lib.SF_EUNSUPPORTED, _lib.SF_EINVAL)
