"""The C-ABI boundary: libkkb200.so loads without a GPU and exports exactly
the entry points include/kkb200.h declares (no compute calls here)."""

import os
import re

from paper_2108_07001_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(REPO, "include", "kkb200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(kk_[a-z0-9_]+)\s*\(", text))


def test_library_builds_and_loads():
    from paper_2108_07001_b200 import build

    build.build()
    lib = _lib.load()
    assert lib.kk_version() == 2


def test_exports_match_header():
    lib = _lib.load()
    declared = header_functions()
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in kkb200.h but not exported"
    # the ctypes binding covers every declared entry point and nothing else
    assert set(_lib.EXPORTED) == declared


def test_last_error_and_status_mapping():
    import pytest

    from paper_2108_07001_b200.sigcore import ParameterError

    lib = _lib.load()
    assert isinstance(lib.kk_last_error(), bytes)
    # parameter validation happens before any device work
    with pytest.raises(ParameterError):
        _lib.call("kk_reconstruct_pairs", 0, None, 1.0, 1e-12, 0, None, None, None, None, None, None, None,
                  None, None, None, 0, 0, 0, None, 0, 0, None)
    assert b"n_hops" in lib.kk_last_error()


def test_no_oracle_in_product():
    """The product package never imports the test oracle."""
    pkg = os.path.join(REPO, "paper_2108_07001_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(root, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, flags=re.M), f
