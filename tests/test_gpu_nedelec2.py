"""Second-order Nedelec fine space on the device (BASELINE config 2) against the
order-2 oracle (oracle/nedelec2_oracle.py; parity-unpinned against the
reference, which has Whitney elements only — see tests/test_nedelec2_oracle.py
for how the oracle itself is tied down).  Tolerances as for lowest order:
entries 1e-12 relative, preconditioner maps 1e-11, GMRES iterations +-1 and
solution 1e-8 (north_star)."""

import numpy as np
import pytest

from oracle import maxwell_oracle as O1
from oracle import nedelec2_oracle as O2
from conftest import rel

pytestmark = pytest.mark.gpu


def _space2(n):
    from paper_1711_03789_b200 import fem, mesh

    return fem.build_edge_space(mesh.build_cube_mesh(n), "pec", order=2)


def _same_pattern(a, b):
    return np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)


def test_element2_matrices_vs_oracle(gpu):
    from paper_1711_03789_b200 import fem

    rng = np.random.default_rng(11)
    c = rng.random((64, 4, 3))
    s, m = fem.element2_matrices(c)
    so, mo = O2.element_matrices(c)
    assert np.abs(s - so).max() <= 1e-12 * np.abs(so).max()
    assert np.abs(m - mo).max() <= 1e-12 * np.abs(mo).max()


@pytest.mark.parametrize("het", [False, True])
def test_assembly2_vs_oracle(gpu, het):
    from paper_1711_03789_b200 import fem

    s = _space2(3)
    kw = {}
    if het:
        rng = np.random.default_rng(2)
        nt = s.mesh.n_tets
        kw = dict(eps=1 + 3 * rng.random(nt), mu=1 + rng.random(nt), sigma=rng.random(nt))
    co = fem.Coefficients(k=3.0, xi=2.0, **kw)
    b = fem.assemble(s, co)
    ref = O2.assemble(s.mesh.vertices, s.mesh.tets, s.tet_dofs, s.ndof, 3.0, 2.0, **kw)
    for k in ("A", "S", "M", "Dk"):
        got = getattr(b, k).to_scipy()
        assert _same_pattern(got, ref[k]), k
        assert np.abs(got.data - ref[k].data).max() <= 1e-12 * np.abs(ref[k].data).max(), k


def test_rhs2_vs_oracle(gpu):
    from paper_1711_03789_b200 import fem

    s = _space2(3)
    src = fem.GaussianSource(alpha=100.0, amp=-1.0, direction=(0.0, 0.0, 1.0))
    dev = fem.assemble_rhs(s, src)
    ref = O2.rhs(s.mesh.vertices, s.mesh.tets, s.tet_dofs, s.ndof, src)
    assert rel(dev, ref) <= 1e-12
    # host-callable source path (values at the quadrature points)
    f = lambda x: np.stack([np.sin(x[..., 0]), x[..., 1] * 1j, np.cos(x[..., 2])], axis=-1)
    assert rel(fem.assemble_rhs(s, f), O2.rhs(s.mesh.vertices, s.mesh.tets, s.tet_dofs, s.ndof, f)) <= 1e-12


def _case(n=4, p=2, layers=1, nc=2, k=3.0, xi=3.0):
    from paper_1711_03789_b200 import decomp, fem, mesh

    s = _space2(n)
    src = fem.GaussianSource(alpha=100.0, amp=-1.0, direction=(0.0, 0.0, 1.0))
    prob = fem.assemble(s, fem.Coefficients(k=k, xi=xi), source=src)
    d = decomp.build_decomposition(s, p, layers, coarse_space=fem.build_edge_space(mesh.build_cube_mesh(nc)))
    return s, prob, d


def _oracle_schwarz(s, d, fam, lev, cor, k, xi_prec, A_corr):
    ap = O2.assemble(s.mesh.vertices, s.mesh.tets, s.tet_dofs, s.ndof, k, xi_prec)["A"]
    R0 = d.coarse.R0
    A0 = (R0 @ ap @ R0.T).tocsc()
    return O1.Schwarz(d.dofs, d.pou, O1.minors(ap, d.dofs), family=fam, levels=lev, correction=cor,
                      R0=R0, A0=A0, A_corr=A_corr, ndof=s.ndof)


@pytest.mark.parametrize("fam,lev,cor", [("as", "one", "additive"), ("as", "two", "additive"),
                                         ("ras", "two", "additive"), ("as", "two", "hybrid")])
def test_precond2_vs_oracle(gpu, fam, lev, cor):
    from paper_1711_03789_b200 import precond

    s, prob, d = _case()
    st = precond.setup(prob, d, precond.PreconditionerSpec(fam, lev, cor, xi_prec=3.0), lu_cap=None)
    ref = _oracle_schwarz(s, d, fam, lev, cor, 3.0, 3.0, prob.A.to_scipy())
    rng = np.random.default_rng(0)
    for _ in range(2):
        v = rng.standard_normal(s.ndof) + 1j * rng.standard_normal(s.ndof)
        assert rel(st.apply(v), ref.apply(v)) <= 1e-11


def test_gmres2_vs_oracle(gpu):
    from paper_1711_03789_b200 import precond
    from paper_1711_03789_b200.krylov import KrylovConfig, gmres

    s, prob, d = _case(n=6, p=2, layers=1, nc=3, k=4.0, xi=4.0)
    st = precond.setup(prob, d, precond.PreconditionerSpec("as", "two", "additive", xi_prec=4.0), lu_cap=None)
    rep = gmres(prob.A, prob.rhs, precond=st, config=KrylovConfig(tol=1e-6, maxit=200))
    A = prob.A.to_scipy()
    ref = _oracle_schwarz(s, d, "as", "two", "additive", 4.0, 4.0, A)
    x, hist, its, conv = O1.gmres(A, prob.rhs, precond=ref, tol=1e-6, maxit=200)
    assert rep.converged and conv
    assert abs(rep.iterations - its) <= 1
    assert rel(rep.x, x) <= 1e-8
    assert np.linalg.norm(prob.rhs - A @ rep.x) / np.linalg.norm(prob.rhs) <= 1.01e-6


# ----------------------------------------- non-nested coarse meshes (cfg2 pairs N=30 with N=8)
@pytest.mark.parametrize("order", [1, 2])
def test_nonnested_coarse_apply_vs_oracle(gpu, order):
    from paper_1711_03789_b200 import decomp, fem, mesh, precond

    m = mesh.build_cube_mesh(6)
    s = fem.build_edge_space(m, "pec", order=order)
    prob = fem.assemble(s, fem.Coefficients(k=3.0, xi=3.0))
    d = decomp.build_decomposition(s, 2, 1, coarse_space=fem.build_edge_space(mesh.build_cube_mesh(4)),
                                   allow_nonnested=True)
    assert d.coarse.tet_map is None
    st = precond.setup(prob, d, precond.PreconditionerSpec("as", "two", "additive", xi_prec=3.0), lu_cap=None)
    if order == 2:
        ap = O2.assemble(m.vertices, m.tets, s.tet_dofs, s.ndof, 3.0, 3.0)["A"]
    else:
        from conftest import mesh_dict

        ap = O1.assemble(mesh_dict(m), s.edge_to_dof, s.ndof, 3.0, 3.0)["A"]
    R0 = d.coarse.R0
    ref = O1.Schwarz(d.dofs, d.pou, O1.minors(ap, d.dofs), levels="two", R0=R0, A0=(R0 @ ap @ R0.T).tocsc(),
                     ndof=s.ndof)
    rng = np.random.default_rng(1)
    v = rng.standard_normal(s.ndof) + 1j * rng.standard_normal(s.ndof)
    assert rel(st.coarse_solve(v), ref.coarse_solve(v)) <= 1e-11
    assert rel(st.apply(v), ref.apply(v)) <= 1e-11


def test_cfg2_shape_gmres_vs_oracle(gpu):
    """cfg2's structure at a size the oracle solves in seconds: order 2, minimal
    overlap, non-nested lowest-order coarse mesh, z-directed Gaussian source."""
    from paper_1711_03789_b200 import decomp, fem, mesh, precond
    from paper_1711_03789_b200.krylov import KrylovConfig, gmres

    m = mesh.build_cube_mesh(9)
    s = fem.build_edge_space(m, "pec", order=2)
    src = fem.GaussianSource(alpha=100.0, amp=-1.0, direction=(0.0, 0.0, 1.0))
    prob = fem.assemble(s, fem.Coefficients(k=6.0, xi=6.0), source=src)
    d = decomp.build_decomposition(s, 3, 1, coarse_space=fem.build_edge_space(mesh.build_cube_mesh(4)),
                                   allow_nonnested=True)
    st = precond.setup(prob, d, precond.PreconditionerSpec("as", "two", "additive", xi_prec=6.0), lu_cap=None)
    rep = gmres(prob.A, prob.rhs, precond=st, config=KrylovConfig(tol=1e-6, maxit=200))
    A = prob.A.to_scipy()
    R0 = d.coarse.R0
    ref = O1.Schwarz(d.dofs, d.pou, O1.minors(A, d.dofs), levels="two", R0=R0, A0=(R0 @ A @ R0.T).tocsc(),
                     ndof=s.ndof)
    x, hist, its, conv = O1.gmres(A, prob.rhs, precond=ref, tol=1e-6, maxit=200)
    assert conv and rep.converged
    assert abs(rep.iterations - its) <= 1
    assert rel(rep.x, x) <= 1e-8
