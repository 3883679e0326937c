"""The C-ABI libraries load and export every symbol include/*.h declares. CPU (no compute calls)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_2405_03831_b200 import _native as nat


def _declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^[A-Za-z_][\w \*]*?\b((?:cs|cm|ct)_\w+)\s*\(", text, flags=re.M)))


@pytest.mark.parametrize("header,loader,table", [
    ("cosched_b200.h", nat.sweep_lib, nat.SWEEP_SYMBOLS),
    ("cosched_match.h", nat.match_lib, nat.MATCH_SYMBOLS),
    ("cosched_train.h", nat.train_lib, nat.TRAIN_SYMBOLS),
])
def test_every_declared_symbol_is_exported_and_bound(header, loader, table):
    names = _declared(header)
    assert len(names) >= 3
    lib = loader()
    for name in names:
        assert hasattr(lib, name), f"{name} missing from the .so"
        assert name in table, f"{name} declared but not bound in _native.py"


def test_sweep_library_is_sm100a_and_static_cudart():
    path = nat.SWEEP_LIB
    blob = open(path, "rb").read()
    assert b"sm_100a" in blob
    lib = nat.sweep_lib()
    assert lib.cs_version().decode().startswith("cosched_b200")
    assert lib.cs_error_string(-2).decode().startswith("no co-run configs")


def test_train_library_is_sm100a():
    blob = open(nat.TRAIN_LIB, "rb").read()
    assert b"sm_100a" in blob
    assert nat.train_lib().ct_version().decode().startswith("cosched_train")


def test_host_only_layout_functions():
    lib = nat.sweep_lib()
    nb = lib.cs_tables_bytes(256, 100, 5)
    assert nb > 256 * 20 * 4 * 2
    t = nat.CsTables()
    fake = 1 << 20                      # aligned address: bind only does arithmetic
    assert lib.cs_tables_bind(fake, nb, 256, 100, 5, ctypes.byref(t)) == 0
    assert ctypes.cast(t.app_a32, ctypes.c_void_p).value % 256 == 0
    assert lib.cs_tables_bind(fake, nb - 1, 256, 100, 5, ctypes.byref(t)) == -5
    assert lib.cs_tables_bind(fake + 8, nb, 256, 100, 5, ctypes.byref(t)) == -1
    g = nat.CsGrid()
    g.n_grid, g.n_budgets = 0, 1
    assert lib.cs_build_graph_workspace_bytes(8, ctypes.byref(g)) > 0
    g.n_budgets = 9
    assert lib.cs_build_graph_workspace_bytes(8, ctypes.byref(g)) == 0


def test_missing_library_raises(monkeypatch):
    monkeypatch.setattr(nat, "_libs", {})
    with pytest.raises(nat.NativeLibraryError):
        nat._load("/nonexistent/lib.so", {}, "x")
