"""CPU-side checks of the C ABI boundary: the library loads and exports exactly
what include/splat_b200.h declares (no compute calls — there is no GPU here)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "splat_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(splat_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2503_14171_b200 import _lib
    return _lib.load()


def test_library_built_for_sm100a():
    from paper_2503_14171_b200 import _lib
    assert os.path.exists(_lib.LIB_PATH)
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 14
    for name in names:
        assert hasattr(lib, name), name


def test_python_binding_matches_header(lib):
    from paper_2503_14171_b200 import _lib
    assert sorted(_lib.SIGNATURES) == declared_functions()


def test_integration_table_names_every_entry_point():
    """INTEGRATION.md's binding table maps every declared entry point to the reference
    interface it replaces."""
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    missing = [f for f in declared_functions() if f"`{f}`" not in doc]
    assert not missing, missing


def test_abi_version_and_sizes(lib):
    assert lib.splat_abi_version() == 1
    # workspace size queries are pure host arithmetic
    assert lib.splat_scene_const_bytes(1000) >= 1000 * (4 + 16 + 6 * 8 + 16)
    a = lib.splat_frame_workspace_bytes(1000, 64, 48, 4096)
    b = lib.splat_frame_workspace_bytes(1000, 64, 48, 8192)
    assert b > a > 0


def test_error_mapping():
    from paper_2503_14171_b200 import _lib
    from paper_2503_14171_b200.core import DimensionError, ParameterError, UnsupportedScaleError
    for code, exc in ((1, DimensionError), (2, ParameterError), (3, UnsupportedScaleError)):
        with pytest.raises(exc):
            _lib.check(code)
    with pytest.raises(RuntimeError):
        _lib.check(100)


def test_struct_layouts():
    from paper_2503_14171_b200 import _lib
    assert ctypes.sizeof(_lib.SceneT) == 8 * 7
    assert ctypes.sizeof(_lib.ViewT) == 8 * 7
    assert ctypes.sizeof(_lib.GimgT) == 8 * 5
    assert ctypes.sizeof(_lib.FramePtrsT) == 8 * 9
