"""The C-ABI boundary: libmdd.so loads and exports every entry point that
include/mdd.h declares; without a GPU it refuses to compute (no fallback)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "mdd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(mdd_[a-z0-9_]+)\s*\(", src))
    names.discard("mdd_host_op")  # typedef of a callback, not a symbol
    return sorted(n for n in names if not n.startswith("mdd_host_op"))


def test_header_declares_entry_points():
    names = _declared()
    assert "mdd_gmres" in names and "mdd_prec_create" in names and "mdd_assemble" in names
    assert len(names) >= 25


def test_library_exports_every_declared_symbol():
    from paper_1711_03789_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    # the ctypes binding covers exactly the declared API
    assert set(_declared()) == set(_lib.exported_symbols())


def test_no_cpu_fallback_without_gpu():
    from paper_1711_03789_b200 import _lib

    if _lib.device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(_lib.MddError, match="no CPU fallback"):
        _lib.Context(0)


def test_library_is_sm100a():
    from paper_1711_03789_b200 import _lib

    data = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_loopback_group_host_side():
    """The loopback group (multi-rank test harness) is host-only: it can be made
    and freed without a GPU, and rejects sizes outside 1..8."""
    from paper_1711_03789_b200 import _lib
    from paper_1711_03789_b200.distributed import LoopbackGroup

    g = LoopbackGroup(3)
    assert g.nranks == 3 and g.handle
    del g
    h = ctypes.c_void_p()
    with pytest.raises(_lib.MddError, match="1..8 ranks"):
        _lib.check(_lib.lib.mdd_comm_loopback_group(9, ctypes.byref(h)))


def test_thread_local_context_override():
    """``use_context`` routes one thread's calls to its own context and restores
    the previous one on exit (no device needed for the bookkeeping)."""
    import threading

    from paper_1711_03789_b200 import _lib

    sentinel, seen = object(), {}
    with _lib.use_context(sentinel):
        assert _lib.get_context() is sentinel
        t = threading.Thread(target=lambda: seen.setdefault("other", getattr(_lib._thread_ctx, "ctx", None)))
        t.start()
        t.join()
    assert seen["other"] is None  # other threads keep the process default
    assert getattr(_lib._thread_ctx, "ctx", None) is None
