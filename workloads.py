"""BASELINE.json configs as plain data + seeded synthetic inputs (numpy only).

Shared by ``bench.py`` (both arms), the golden generators under
``tests/golden/`` and the config-scale parity tests, so that the device path,
the CPU oracle and the committed fixtures are all built from the same
numbers.  Imports neither the product package nor ``oracle/``.

Conventions where BASELINE.json is silent:

* Gaussian source "width w"  ->  F = -exp(-|x-c|^2 / w^2) z-hat  (cfg0/cfg2
  w=0.1 -> alpha=100; cfg4 w=0.05 -> alpha=400, the exponent of the
  reference's own ``gaussian_source``, fem.py:360-364).
* random rhs: ``(randn(n) + 1j*randn(n)) / sqrt(2)`` from
  ``np.random.default_rng(seed)``, real part drawn first.
* cfg3 combines the coarse space as the paper does for ImpRAS (hybrid,
  "ImpHRAS", Table 6).
* cfg4: eps_r per 4x4x4 block ~ U[1,4]; absorption per block ~ U[k/2, 2k]
  carried by sigma = absorption / k, so that k*sigma is the block absorption
  (reference fem.py:253-256); xi = xi_prec = 0.
"""

from __future__ import annotations

import math

import numpy as np

CONFIGS = {
    0: dict(name="cfg0", N=20, k=10.0, xi=10.0, p=2, layers=2, nc=5, family="as", corr="additive",
            rhs=("gauss", 100.0)),
    1: dict(name="cfg1", N=40, k=20.0, xi=20.0, p=4, layers=2, nc=10, family="as", corr="additive",
            rhs=("random", 0)),
    # second-order Nedelec fine space (extension: the reference has Whitney elements only),
    # lowest-order coarse space nested in its Whitney part; Gaussian source as cfg0
    2: dict(name="cfg2", N=30, k=20.0, xi=20.0, p=3, layers=1, nc=8, family="as", corr="additive",
            rhs=("gauss", 100.0), order=2),
    3: dict(name="cfg3", N=60, k=30.0, xi=math.sqrt(30.0), p=4, layers=2, nc=15, family="impras",
            corr="hybrid", rhs=("random", 0)),
    4: dict(name="cfg4", N=80, k=40.0, xi=0.0, p=8, layers=2, nc=20, family="as", corr="additive",
            rhs=("gauss", 400.0), hetero=True),
}

TOL = 1e-6
MAXIT = 200


def hetero_fields(c, tet_barycenters, seed=0):
    """Per-tet (eps, sigma) of cfg4 from the tets' barycentres."""
    rng = np.random.default_rng(seed)
    blk = np.clip((tet_barycenters * 4).astype(int), 0, 3)
    bid = (blk[:, 0] * 4 + blk[:, 1]) * 4 + blk[:, 2]
    eps_b = 1.0 + 3.0 * rng.random(64)
    abs_b = c["k"] * (0.5 + 1.5 * rng.random(64))
    return eps_b[bid], abs_b[bid] / c["k"]


def random_rhs(ndof, seed=0):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal(ndof) + 1j * rng.standard_normal(ndof)) / np.sqrt(2.0)


def probe_vectors(ndof, count=16, seed=12345):
    """Seeded complex probes: goldens store <p_i, x> instead of all of x."""
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((count, ndof)) + 1j * rng.standard_normal((count, ndof))) / np.sqrt(2.0 * ndof)


def sample_stride(ndof, count=4096):
    return max(1, ndof // count)


def describe(c, ndof, label):
    return (f"{c['name']}: N={c['N']} ({ndof} DoFs), k={c['k']:g}, xi={c['xi']:.4g}, {c['p']}^3 subdomains, "
            f"{c['layers']} overlap layers, coarse N={c['nc']}, {label}, right GMRES tol {TOL:g} maxit {MAXIT}")
