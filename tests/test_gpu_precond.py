"""Device Schwarz preconditioners against the reference's golden maps and the
oracle (reference test strategy: test_precond.py:42-239).  The device uses an
unpivoted multifrontal elimination over a nested-dissection order; the
reference uses partially pivoted dense LU: results agree to rounding."""

import numpy as np
import pytest

from conftest import load_golden, mesh_dict, rel
from oracle import maxwell_oracle as O

pytestmark = pytest.mark.gpu


def _problem(n=3, k=2.0, xi=None, bc="pec"):
    from paper_1711_03789_b200 import fem, mesh

    xi = k * k if xi is None else xi
    s = fem.build_edge_space(mesh.build_cube_mesh(n), bc)
    return fem.assemble(s, fem.Coefficients(k=k, xi=xi), source=fem.gaussian_source)


def _coarse(n, bc="pec"):
    from paper_1711_03789_b200 import fem, mesh

    return fem.build_edge_space(mesh.build_cube_mesh(n), bc)


@pytest.fixture(scope="module")
def gp():
    return load_golden("precond.npz")


@pytest.fixture(scope="module")
def case3():
    from paper_1711_03789_b200 import decomp

    prob = _problem(3, 2.0)
    d = decomp.build_decomposition(prob.space, 3, 1, coarse_space=_coarse(1))
    return prob, d


@pytest.mark.parametrize("fam", ["as", "ras", "impras"])
@pytest.mark.parametrize("lev,cor", [("one", "additive"), ("two", "additive"), ("two", "hybrid"), ("two", "adef1")])
def test_all_variants_match_reference(gpu, gp, case3, fam, lev, cor):
    from paper_1711_03789_b200 import precond

    prob, d = case3
    st = precond.setup(prob, d, precond.PreconditionerSpec(fam, lev, cor, xi_prec=4.0))
    for v, ref in zip(gp["v"], gp[f"{fam}_{lev}_{cor}"]):
        assert rel(st.apply(v), ref) <= 1e-11


@pytest.mark.parametrize("fam", ["as", "impras"])
def test_global_impedance_two_level_hybrid(gpu, gp, fam):
    from paper_1711_03789_b200 import decomp, precond

    prob = _problem(2, 2.0, bc="impedance")
    d = decomp.build_decomposition(prob.space, 2, 1, coarse_space=_coarse(1, "impedance"))
    st = precond.setup(prob, d, precond.PreconditionerSpec(fam, "two", "hybrid", xi_prec=4.0))
    assert rel(st.apply(gp["gimp_v"]), gp[f"gimp_{fam}"]) <= 1e-11


def test_linearity(gpu):
    from paper_1711_03789_b200 import decomp, precond

    prob = _problem(2, 2.0)
    d = decomp.build_decomposition(prob.space, 2, 1, coarse_space=_coarse(1))
    st = precond.setup(prob, d, precond.PreconditionerSpec(family="ras", levels="two", xi_prec=4.0))
    rng = np.random.default_rng(9)
    n = prob.ndof
    u = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    v = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    al, be = 1.3 - 0.4j, -0.2 + 2.1j
    assert rel(st.apply(al * u + be * v), al * st.apply(u) + be * st.apply(v)) <= 1e-12


def test_single_subdomain_is_exact_inverse(gpu):
    from paper_1711_03789_b200 import decomp, krylov, precond

    prob = _problem(2, 2.0)
    d = decomp.build_decomposition(prob.space, 1, 1)
    st = precond.setup(prob, d, precond.PreconditionerSpec(family="as", levels="one", xi_prec=4.0))
    rng = np.random.default_rng(10)
    v = rng.standard_normal(prob.ndof) + 1j * rng.standard_normal(prob.ndof)
    assert rel(prob.A @ st.apply(v), v) <= 1e-10
    rep = krylov.gmres(prob.A, prob.rhs, precond=st.apply, config=krylov.KrylovConfig(tol=1e-6))
    assert rep.iterations == 1 and rep.converged


def test_coarse_equals_fine_gives_exact_correction(gpu):
    from paper_1711_03789_b200 import decomp, precond

    prob = _problem(2, 2.0)
    d = decomp.build_decomposition(prob.space, 2, 2, coarse_space=prob.space)
    rng = np.random.default_rng(12)
    v = rng.standard_normal(prob.ndof) + 1j * rng.standard_normal(prob.ndof)
    a_inv_v = np.linalg.solve(prob.A.toarray(), v)
    two = precond.setup(prob, d, precond.PreconditionerSpec(family="as", levels="two", xi_prec=4.0))
    one = precond.setup(prob, d, precond.PreconditionerSpec(family="as", levels="one", xi_prec=4.0))
    assert rel(two.apply(v), one.apply(v) + a_inv_v) <= 1e-10
    hyb = precond.setup(prob, d, precond.PreconditionerSpec("as", "two", "hybrid", xi_prec=4.0))
    assert rel(hyb.apply(v), a_inv_v) <= 1e-10
    assert rel(two.coarse_solve(v), a_inv_v) <= 1e-10


def test_xi_prec_independent_of_problem(gpu):
    from paper_1711_03789_b200 import decomp, fem, precond

    prob = _problem(2, 2.0, xi=0.0)
    d = decomp.build_decomposition(prob.space, 1, 1)
    st = precond.setup(prob, d, precond.PreconditionerSpec(family="as", levels="one", xi_prec=4.0))
    rng = np.random.default_rng(13)
    v = rng.standard_normal(prob.ndof) + 1j * rng.standard_normal(prob.ndof)
    x = st.apply(v)
    assert np.linalg.norm(prob.A @ x - v) > 1e-3 * np.linalg.norm(v)
    shifted = fem.assemble(prob.space, prob.coefficients.with_xi(4.0))
    assert rel(shifted.A @ x, v) <= 1e-10


def test_variant_shares_factors(gpu):
    from paper_1711_03789_b200 import decomp, precond

    prob = _problem(2, 2.0)
    d = decomp.build_decomposition(prob.space, 2, 1, coarse_space=_coarse(1))
    S = precond.PreconditionerSpec
    st2 = precond.setup(prob, d, S(family="as", levels="two", xi_prec=4.0))
    st1 = st2.variant(S(family="as", levels="one", xi_prec=4.0))
    st_ras = st2.variant(S(family="ras", levels="two", xi_prec=4.0))
    assert st1.factors is st2.factors
    rng = np.random.default_rng(14)
    v = rng.standard_normal(prob.ndof) + 1j * rng.standard_normal(prob.ndof)
    fresh1 = precond.setup(prob, d, S(family="as", levels="one", xi_prec=4.0))
    fresh_ras = precond.setup(prob, d, S(family="ras", levels="two", xi_prec=4.0))
    assert np.array_equal(st1.apply(v), fresh1.apply(v))
    assert np.array_equal(st_ras.apply(v), fresh_ras.apply(v))
    with pytest.raises(ValueError):
        st2.variant(S(family="impras", levels="one", xi_prec=4.0))
    with pytest.raises(ValueError):
        st2.variant(S(family="as", levels="one", xi_prec=1.0))


def test_singular_local_reports_subdomain(gpu):
    from paper_1711_03789_b200 import decomp, precond
    from paper_1711_03789_b200.linalg import SingularMatrixError

    prob = _problem(2, 1e-8, xi=0.0)
    d = decomp.build_decomposition(prob.space, 1, 1)
    with pytest.raises(SingularMatrixError, match="subdomain 0"):
        precond.setup(prob, d, precond.PreconditionerSpec(family="as", levels="one", xi_prec=0.0))


def test_size_cap(gpu):
    from paper_1711_03789_b200 import decomp, precond
    from paper_1711_03789_b200.linalg import SizeCapError

    prob = _problem(4, 2.0)
    d = decomp.build_decomposition(prob.space, 2, 1)
    with pytest.raises(SizeCapError, match="subdomain 0"):
        precond.setup(prob, d, precond.PreconditionerSpec(xi_prec=4.0), lu_cap=10)


def test_dimension_mismatch(gpu, case3):
    from paper_1711_03789_b200 import precond

    prob, d = case3
    st = precond.setup(prob, d, precond.PreconditionerSpec(xi_prec=4.0))
    with pytest.raises(ValueError):
        st.apply(np.ones(prob.ndof + 1))


@pytest.mark.parametrize("n,p,layers,nc,leaf", [(8, 2, 2, 4, 64), (12, 3, 1, 4, 16), (10, 2, 2, 5, 256)])
def test_larger_cases_vs_oracle(gpu, n, p, layers, nc, leaf):
    """Multi-level ND trees (many fronts per subdomain) vs the SuperLU oracle."""
    from paper_1711_03789_b200 import decomp, fem, mesh, precond

    s = fem.build_edge_space(mesh.build_cube_mesh(n), "pec")
    prob = fem.assemble(s, fem.Coefficients(k=4.0, xi=4.0))
    d = decomp.build_decomposition(s, p, layers, coarse_space=_coarse(nc))
    a = O.assemble(mesh_dict(s.mesh), s.edge_to_dof, s.ndof, 4.0, 4.0)["A"]
    r0 = d.coarse.R0
    ref = O.Schwarz(d.dofs, d.pou, O.minors(a, d.dofs), "ras", "two", "hybrid", R0=r0,
                    A0=(r0 @ a @ r0.T).tocsr(), A_corr=a, ndof=s.ndof, solver="sparse")
    st = precond.PreconditionerState(prob, d, precond.PreconditionerSpec("ras", "two", "hybrid", xi_prec=4.0),
                                     lu_cap=None, leaf_size=leaf)
    rng = np.random.default_rng(n)
    v = rng.standard_normal(s.ndof) + 1j * rng.standard_normal(s.ndof)
    assert rel(st.apply(v), ref.apply(v)) <= 1e-10


def test_symmetric_transpose_path_matches_gemm_path(gpu, monkeypatch):
    """Complex-symmetric A_prec: the packed F_UP of the solve is F_PU^T
    (k_transpose_up) instead of a second GEMM; MDD_NO_SYM forces the GEMM.
    Both must agree with each other and with the oracle to rounding."""
    from paper_1711_03789_b200 import decomp, precond

    prob = _problem(8, 3.0, xi=9.0)
    d = decomp.build_decomposition(prob.space, 2, 2, coarse_space=_coarse(4))
    spec = precond.PreconditionerSpec("as", "two", "additive", xi_prec=9.0)
    rng = np.random.default_rng(7)
    v = rng.standard_normal(prob.ndof) + 1j * rng.standard_normal(prob.ndof)
    st_sym = precond.setup(prob, d, spec, lu_cap=None)
    y_sym = st_sym.apply(v)
    monkeypatch.setenv("MDD_NO_SYM", "1")
    st_gemm = precond.setup(prob, d, spec, lu_cap=None)
    y_gemm = st_gemm.apply(v)
    import ctypes

    from paper_1711_03789_b200 import _lib

    flags = []
    for st in (st_sym, st_gemm):
        f = ctypes.c_int(-1)
        _lib.check(_lib.lib.mdd_prec_symmetric(st.handle, ctypes.byref(f)))
        flags.append(f.value)
    assert flags == [1, 0]  # the assembled A_prec is bitwise symmetric; MDD_NO_SYM forces the GEMM
    assert rel(y_sym, y_gemm) <= 1e-12
    # flop accounting (mdd_prec_flop_counts): the symmetric path skips the F_UP GEMM and the Schur
    # tiles above the diagonal; the partial-LU count lies below the full-elimination count
    fs, fg = st_sym.stats(), st_gemm.stats()
    assert fs["factor_flops"] == fg["factor_flops"] and fs["lu_flops"] == fg["lu_flops"]
    assert 0 < fs["executed_flops"] < fg["executed_flops"] <= fs["factor_flops"] * (1 + 1e-12)
    assert 0 < fs["lu_flops"] < fs["factor_flops"]
    A = prob.A.to_scipy()
    R0 = d.coarse.R0
    ref = O.Schwarz(d.dofs, d.pou, O.minors(A, d.dofs), levels="two", R0=R0, A0=(R0 @ A @ R0.T).tocsc(),
                    ndof=prob.ndof)
    assert rel(y_sym, ref.apply(v)) <= 1e-11


def test_no_absorption_blocks_are_checked_against_pivoted_lu(gpu):
    """xi_prec = 0, sigma = 0, PEC local problems, k above the first Dirichlet eigenvalue of the
    subdomains (k = 9 > pi*sqrt(2)/0.75 = 5.9): the blocks are real symmetric indefinite, which
    Lemma 2.5 does not cover.  The reference factors them with partially pivoted LAPACK LU
    (linalg.py:92); the device path pivots statically and must either reproduce the pivoted
    result or refuse the factor with an explicit SingularMatrixError -- never return a silently
    inaccurate map."""
    from oracle import maxwell_oracle as O
    from paper_1711_03789_b200 import decomp, fem, mesh, precond
    from paper_1711_03789_b200.linalg import SingularMatrixError

    s = fem.build_edge_space(mesh.build_cube_mesh(8), "pec")
    k = 9.0
    prob = fem.assemble(s, fem.Coefficients(k=k, xi=0.0))
    d = decomp.build_decomposition(s, 2, 2)
    a = O.assemble({kk: getattr(s.mesh, kk) for kk in ("vertices", "tets", "edges", "tet_edges", "tet_edge_signs",
                                                       "boundary_faces")}, s.edge_to_dof, s.ndof, k, 0.0)["A"]
    minors = O.minors(a, d.dofs)
    ev = np.linalg.eigvalsh(minors[0].toarray().real)
    assert ev.min() < 0 < ev.max()  # indefinite: the case the advisor flagged
    want = O.Schwarz(d.dofs, d.pou, minors, "as", "one", ndof=s.ndof, solver="dense")
    v = np.random.default_rng(2).standard_normal(s.ndof) * (1 + 0.5j)
    try:
        st = precond.setup(prob, d, precond.PreconditionerSpec("as", "one", xi_prec=0.0), lu_cap=None)
    except SingularMatrixError as e:
        assert "without absorption" in str(e)
        return
    assert st.static_pivoting_backed is False and min(st.pivot_ratio) >= st.NO_ABSORPTION_PIVOT_TOL
    assert rel(st.apply(v), want.apply(v)) <= 1e-9
