"""Pin the CPU oracle (oracle/maxwell_oracle.py) to outputs of the reference itself.

Fixtures come from tests/golden/make_golden.py, which runs /root/reference.
The oracle takes plain arrays; mesh/decomposition inputs come from the host
layer (already pinned bit-exactly in test_host_mesh_decomp.py).
"""

import numpy as np
import pytest

from conftest import golden_csr, golden_ragged, load_golden, mesh_dict, rel
from oracle import maxwell_oracle as O
from paper_1711_03789_b200 import decomp, fem, mesh


@pytest.fixture(scope="module")
def gs():
    return load_golden("system.npz")


def _space(n, bc="pec"):
    return fem.build_edge_space(mesh.build_cube_mesh(n), bc)


def test_reference_tet_values(gs):
    s, m, _ = O.element_matrices(np.array([[[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1.0]]]), np.ones((1, 6)))
    assert np.abs(s[0] - gs["ref_tet_S"]).max() <= 1e-14
    assert np.abs(m[0] - gs["ref_tet_M"]).max() <= 1e-14


def test_oracle_assembly_homogeneous(gs):
    s = _space(3)
    out = O.assemble(mesh_dict(s.mesh), s.edge_to_dof, s.ndof, 2.0, 4.0)
    for k in ("A", "S", "M", "Dk"):
        ref = golden_csr(gs, f"hom_{k}")
        got = out[k]
        assert np.array_equal(got.indptr, ref.indptr) and np.array_equal(got.indices, ref.indices)
        assert np.abs(got.data - ref.data).max() <= 1e-12 * np.abs(ref.data).max()
    r = O.rhs(mesh_dict(s.mesh), s.edge_to_dof, s.ndof, O.gaussian())
    assert rel(r, gs["hom_rhs"]) <= 1e-13


def test_oracle_assembly_heterogeneous(gs):
    s = _space(3)
    out = O.assemble(mesh_dict(s.mesh), s.edge_to_dof, s.ndof, 3.0, 2.0,
                     eps=gs["het_eps"], mu=gs["het_mu"], sigma=gs["het_sigma"])
    for k in ("A", "S", "M", "Dk"):
        ref = golden_csr(gs, f"het_{k}")
        assert np.abs((out[k] - ref).toarray()).max() <= 1e-12 * np.abs(ref.data).max()


@pytest.mark.parametrize("tag,xi", [("imp", 4.0), ("impneg", -4.0)])
def test_oracle_assembly_impedance(gs, tag, xi):
    s = _space(2, "impedance")
    out = O.assemble(mesh_dict(s.mesh), s.edge_to_dof, s.ndof, 2.0, xi, bc="impedance")
    assert np.abs((out["A"] - golden_csr(gs, f"{tag}_A")).toarray()).max() <= 1e-12
    assert np.abs((out["Mb"] - golden_csr(gs, f"{tag}_Mb")).toarray()).max() <= 1e-14
    assert rel(O.rhs(mesh_dict(s.mesh), s.edge_to_dof, s.ndof, O.gaussian()), gs[f"{tag}_rhs"]) <= 1e-13


def test_oracle_z_gaussian_rhs(gs):
    s = _space(3)
    r = O.rhs(mesh_dict(s.mesh), s.edge_to_dof, s.ndof, O.gaussian(alpha=100.0, direction=(0, 0, 1)))
    assert rel(r, gs["zrhs"]) <= 1e-13


@pytest.fixture(scope="module")
def gp():
    return load_golden("precond.npz")


def _precond_case():
    s = _space(3)
    a = O.assemble(mesh_dict(s.mesh), s.edge_to_dof, s.ndof, 2.0, 4.0)["A"]
    c = _space(1)
    d = decomp.build_decomposition(s, 3, 1, coarse_space=c)
    return s, a, d


def _oracle_schwarz(s, a, d, fam, lev, cor):
    if fam == "impras":
        sets = decomp.impedance_dof_sets(s, d.elements)
        pou = decomp.build_pou(sets, s.ndof)
        local = [O.impedance_local_matrix(mesh_dict(s.mesh), s.edge_to_dof, s.kept_edges, g, e, 2.0, 4.0)
                 for g, e in zip(sets, d.elements)]
    else:
        sets, pou = d.dofs, d.pou
        local = O.minors(a, sets)
    r0 = d.coarse.R0
    a0 = (r0 @ a @ r0.T).tocsr()
    return O.Schwarz(sets, pou, local, fam, lev, cor, R0=r0, A0=a0, A_corr=a, ndof=s.ndof, solver="dense")


@pytest.mark.parametrize("fam", ["as", "ras", "impras"])
@pytest.mark.parametrize("lev,cor", [("one", "additive"), ("two", "additive"), ("two", "hybrid"), ("two", "adef1")])
def test_oracle_precond_matches_reference(gp, fam, lev, cor):
    s, a, d = _precond_case()
    P = _oracle_schwarz(s, a, d, fam, lev, cor)
    for v, ref in zip(gp["v"], gp[f"{fam}_{lev}_{cor}"]):
        assert rel(P.apply(v), ref) <= 1e-11


def test_oracle_impedance_local_matrix(gp):
    s, a, d = _precond_case()
    g0 = gp["imp_local0_gdofs"]
    got = O.impedance_local_matrix(mesh_dict(s.mesh), s.edge_to_dof, s.kept_edges, g0, d.elements[0], 2.0, 4.0)
    ref = golden_csr(gp, "imp_local0")
    assert np.abs((got - ref).toarray()).max() <= 1e-13


@pytest.fixture(scope="module")
def gg():
    return load_golden("gmres.npz")


def test_oracle_gmres_dense(gg):
    x, h, it, conv = O.gmres(gg["dense_a"], gg["dense_b"], tol=1e-12, maxit=120)
    assert conv and it == int(gg["dense_it"])
    assert rel(x, gg["dense_x"]) <= 1e-12
    assert np.abs(h - gg["dense_hist"]).max() <= 1e-12


@pytest.mark.parametrize("fam,lev,cor,side,wt", [
    ("as", "two", "additive", "right", None),
    ("ras", "two", "hybrid", "left", None),
    ("ras", "one", "additive", "right", "dk"),
    ("as", "two", "adef1", "right", None),
])
def test_oracle_preconditioned_gmres(gg, fam, lev, cor, side, wt):
    s = _space(4)
    md = mesh_dict(s.mesh)
    sysm = O.assemble(md, s.edge_to_dof, s.ndof, 3.0, 9.0)
    b = O.rhs(md, s.edge_to_dof, s.ndof, O.gaussian())
    d = decomp.build_decomposition(s, 2, 1, coarse_space=_space(2))
    r0 = d.coarse.R0
    P = O.Schwarz(d.dofs, d.pou, O.minors(sysm["A"], d.dofs), fam, lev, cor, R0=r0,
                  A0=(r0 @ sysm["A"] @ r0.T).tocsr(), A_corr=sysm["A"], ndof=s.ndof, solver="dense")
    x, h, it, conv = O.gmres(sysm["A"], b, P, tol=1e-8, side=side, weight=sysm["Dk"] if wt else None)
    tag = f"{fam}_{lev}_{cor}_{side}_{wt or 'id'}"
    assert abs(it - int(gg[f"{tag}_it"])) <= 1
    assert rel(x, gg[f"{tag}_x"]) <= 1e-8


def test_oracle_random_initial_guess(gg):
    s = _space(4)
    md = mesh_dict(s.mesh)
    sysm = O.assemble(md, s.edge_to_dof, s.ndof, 3.0, 9.0)
    b = O.rhs(md, s.edge_to_dof, s.ndof, O.gaussian())
    rng = np.random.default_rng(5)
    x0 = rng.random(s.ndof) + 1j * rng.random(s.ndof)
    x, h, it, conv = O.gmres(sysm["A"], b, tol=1e-6, maxit=60, x0=x0)
    assert it == int(gg["rand_it"])
    assert rel(x, gg["rand_x"]) <= 1e-10
