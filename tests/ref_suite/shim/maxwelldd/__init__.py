"""`maxwelldd` as a thin alias of the drop-in package, so that the reference's own test
files (copied by tests/ref_suite/fetch.py into the git-ignored tests/ref_suite/_ref/) run
unchanged against paper_1711_03789_b200.  Test infrastructure only.

The one part of the reference surface the drop-in does not provide is the dense LAPACK LU
(`linalg.DenseLU`, `lu_factor`, `lu_solve`: the device factorisation is the sparse
multifrontal one); tests that construct it are SKIPPED with that reason
instead of failing the whole file at import."""
import importlib
import sys
import types

import pytest

import paper_1711_03789_b200 as _pkg

for _name in ("mesh", "fem", "decomp", "linalg", "precond", "krylov", "experiments", "cli"):
    _mod = importlib.import_module(f"paper_1711_03789_b200.{_name}")
    if _name == "linalg":
        _shim = types.ModuleType("maxwelldd.linalg")
        _shim.__dict__.update({k: v for k, v in _mod.__dict__.items() if not k.startswith("__")})

        def _no_dense_lu(*a, **k):
            pytest.skip("DenseLU (host LAPACK LU) is not provided by the drop-in: blocks are factorised on the device")

        class DenseLU:  # noqa: D401 - stand-in
            def __init__(self, *a, **k):
                _no_dense_lu()

        _shim.DenseLU = DenseLU
        _shim.lu_factor = _no_dense_lu
        _shim.lu_solve = _no_dense_lu
        _shim.DEFAULT_LU_CAP = getattr(_mod, "DEFAULT_LU_CAP", 4000)
        _mod = _shim
    sys.modules[f"maxwelldd.{_name}"] = _mod
    globals()[_name] = _mod

for _k in getattr(_pkg, "__all__", []):
    globals()[_k] = getattr(_pkg, _k)
