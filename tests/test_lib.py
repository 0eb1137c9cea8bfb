"""The C-ABI library loads without a GPU and exports every entry point that
include/slabewald.h declares (no compute calls here)."""

import ctypes
import os
import re

import pytest

from paper_2101_07088_b200 import _build, _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(
    __file__))), "include", "slabewald.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(se_[a-z0-9_]+)\s*\(", text)))


def test_library_builds_and_loads():
    _build.build()
    lib = _lib.load()
    assert lib.se_version().decode().startswith("slabewald-b200")


def test_every_declared_symbol_is_exported():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared()
    assert set(names) == set(_lib.EXPORTS)
    for name in names:
        assert hasattr(lib, name), name


def test_struct_layouts_match_header():
    # se_params: 16 doubles + 4 int32; se_diag: 12 doubles, 2 int32,
    # 2 int64, 16 doubles
    assert ctypes.sizeof(_lib.SeParams) == 16 * 8 + 4 * 4
    assert ctypes.sizeof(_lib.SeDiag) == 12 * 8 + 2 * 4 + 2 * 8 + 16 * 8
    assert ctypes.sizeof(_lib.SeBdParams) == 12 * 8 + 4 * 4 + 8


def test_solver_fails_loudly_without_library(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(RuntimeError, match="not built"):
        _lib.load()


def test_near_field_sum_signature_matches_reference():
    """near_field_sum(positions, charges, geometry, params, eval_positions,
    kernel, need_field, subtract_unsplit_self) as reference slab.py:184-186;
    argument checks happen before any device work."""
    import inspect
    import pytest
    from paper_2101_07088_b200.slab import near_field_sum
    names = list(inspect.signature(near_field_sum).parameters)
    assert names[:8] == ["positions", "charges", "geometry", "params", "eval_positions",
                         "kernel", "need_field", "subtract_unsplit_self"]
    with pytest.raises(ValueError):
        near_field_sum(None, None, None, None, kernel="gauss")
    with pytest.raises(TypeError):
        near_field_sum(None, None, None, None, kern="avg")
