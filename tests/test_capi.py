"""C-ABI library checks that need no GPU: liborca.so builds/loads and exports every entry
point include/orca.h declares; argument validation that happens before any device call."""
from __future__ import annotations

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "orca.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(orca_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def orca():
    from paper_1908_10107_b200 import build
    build.build()
    from paper_1908_10107_b200 import orca as O
    return O


def test_every_header_symbol_exported(orca):
    names = _header_functions()
    assert len(names) >= 19
    L = ctypes.CDLL(orca.LIB_PATH)
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert sorted(orca.EXPORTS) == names


def test_library_is_sm100a(orca):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", orca.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings(orca):
    L = orca.lib()
    for s in range(8):
        assert L.orca_status_string(s)
    assert L.orca_status_string(99) == b"unknown status"


def test_create_rejects_bad_params(orca):
    L = orca.lib()
    ctx = ctypes.c_void_p()
    bad = [dict(timeStep=0.0), dict(neighborDist=-1.0), dict(maxNeighbors=33), dict(maxNeighbors=-1),
           dict(timeHorizon=float("nan")), dict(radius=0.0), dict(maxSpeed=-0.1), dict(maxSpeed=float("inf"))]
    for kw in bad:
        p = orca.make_params(**kw)
        assert L.orca_create(ctypes.byref(p), 0, ctypes.byref(ctx)) == 1, kw
    assert L.orca_create(None, 0, ctypes.byref(ctx)) == 1


def test_null_context_is_an_error(orca):
    L = orca.lib()
    assert L.orca_step(None, 1) == 1
    assert L.orca_set_agents(None, 0, None, None, None) == 1
    assert L.orca_get_state(None, None, None) == 1
    L.orca_destroy(None)  # no-op


def test_no_cpu_fallback_without_library(tmp_path, monkeypatch):
    """The binding must fail loudly if the CUDA library is missing."""
    import importlib.util
    import shutil
    pkg = tmp_path / "pkgcopy"
    pkg.mkdir()
    shutil.copy(os.path.join(ROOT, "paper_1908_10107_b200", "orca.py"), pkg / "orca.py")
    spec = importlib.util.spec_from_file_location("orca_nolib", pkg / "orca.py")
    mod = importlib.util.module_from_spec(spec)
    with pytest.raises(ImportError):
        spec.loader.exec_module(mod)


def test_nccl_test_seam_only_in_test_build(orca):
    """The fake-NCCL hook (ORCA_NCCL_LIB) exists only in liborca_test.so (-DORCA_TEST_HOOKS);
    the product library never loads another NCCL."""
    from paper_1908_10107_b200 import build
    test_lib = build.build(test_hooks=True)
    prod = open(os.path.join(ROOT, "paper_1908_10107_b200", "liborca.so"), "rb").read()
    assert b"ORCA_NCCL_LIB" not in prod
    assert b"ORCA_NCCL_LIB" in open(test_lib, "rb").read()
