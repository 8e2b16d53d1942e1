import os
import sys

import numpy as np
import pytest
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# tests/ref_suite holds the reference's own test files (git-ignored copies) and the `maxwelldd`
# shim; they are run by tests/test_reference_suite.py in a subprocess, never collected directly
collect_ignore = ["ref_suite"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libmdd.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


def golden_csr(g, prefix):
    shape = tuple(g[f"{prefix}_shape"])
    return sp.csr_matrix((g[f"{prefix}_data"], g[f"{prefix}_indices"], g[f"{prefix}_indptr"]), shape=shape)


def golden_ragged(g, prefix):
    ptr, flat = g[f"{prefix}_ptr"], g[f"{prefix}_flat"]
    return [flat[ptr[i]: ptr[i + 1]] for i in range(len(ptr) - 1)]


def mesh_dict(m):
    return {k: getattr(m, k) for k in ("vertices", "tets", "edges", "tet_edges", "tet_edge_signs", "boundary_faces")}


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="session")
def gpu():
    """Skip if no device; on a GPU box the library MUST load (no fallback)."""
    from paper_1711_03789_b200 import _lib

    if _lib.device_count() == 0:
        pytest.skip("no CUDA device")
    return _lib.get_context()
