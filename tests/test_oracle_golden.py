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


# ------------------------------------------------- geometry oracle (product-free)
def test_geometry_oracle_mesh_matches_reference():
    from oracle import geometry_oracle as G

    g = load_golden("mesh.npz")
    for n in (1, 3):
        m = G.cube_mesh(n)
        for f in ("vertices", "tets", "edges", "tet_edges", "tet_edge_signs", "boundary_edge_flags",
                  "boundary_faces"):
            assert np.array_equal(m[f], g[f"n{n}_{f}"]), (n, f)
    assert np.array_equal(G.nesting_map(G.cube_mesh(1), G.cube_mesh(3)), g["nest_3_1"])


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_geometry_oracle_decomposition_matches_reference(tag):
    from oracle import geometry_oracle as G

    g = load_golden("decomp.npz")
    n, p, layers, nc = (int(v) for v in g[f"{tag}_case"])
    s = G.edge_space(G.cube_mesh(n))
    d = G.decomposition(s, p, layers, G.edge_space(G.cube_mesh(nc)))
    for key, got in (("elements", d["elements"]), ("dofs", d["dofs"]), ("pou", d["pou"]),
                     ("impdofs", G.impedance_dof_sets(s, d["elements"]))):
        want = golden_ragged(g, f"{tag}_{key}")
        assert len(got) == len(want)
        for a, b in zip(got, want):
            assert np.array_equal(a, b), key
    assert np.array_equal(d["tet_map"], g[f"{tag}_tetmap"])
    # the reference keeps rounding-level entries of its Gauss rule (decomp.py:287-291); values agree to 1e-14
    assert abs(d["R0"] - golden_csr(g, f"{tag}_R0")).max() <= 1e-14


def test_geometry_oracle_impedance_space():
    from oracle import geometry_oracle as G

    g = load_golden("decomp.npz")
    si = G.edge_space(G.cube_mesh(4), "impedance")
    d = G.decomposition(si, 2, 1, G.edge_space(G.cube_mesh(2), "impedance"))
    for a, b in zip(d["dofs"], golden_ragged(g, "imp_dofs")):
        assert np.array_equal(a, b)
    assert abs(d["R0"] - golden_csr(g, "imp_R0")).max() <= 1e-14


def test_nd_order_is_a_permutation_with_plane_separators():
    from oracle import geometry_oracle as G
    from oracle import parallel_oracle as P

    s = G.edge_space(G.cube_mesh(6))
    xyz = G.edge_half_coords(s["mesh"])[s["kept_edges"]]
    perm = P.nd_order(xyz, leaf=8)
    assert np.array_equal(np.sort(perm), np.arange(s["ndof"]))
    # the last block is the top separator: one grid plane
    top = xyz[perm[-1]]
    a = [ax for ax in range(3) if (xyz[:, ax] == top[ax]).sum() and top[ax] % 2 == 0]
    assert a


def test_parallel_oracle_cfg0_matches_reference_dense_solve():
    """The config-scale oracle (ND-SuperLU in worker processes, BLAS MGS2) against the
    reference package's own cfg0 solve with its dense LAPACK LU (tests/golden/cfg0.npz)."""
    import workloads as W
    from oracle import parallel_oracle as P

    g = load_golden("cfg0.npz")
    prob = P.build_problem(W.CONFIGS[0])
    assert rel(prob["rhs"], g["rhs"]) <= 1e-13
    with P.ParallelSchwarz(prob, workers=2) as M:
        x, hist, its, conv, _ = P.gmres(prob["A"], prob["rhs"], M.apply, tol=W.TOL, maxit=W.MAXIT)
        # same map with another worker count: the sum order is the reference's, not the pool's
        v = W.random_rhs(prob["ndof"], seed=3)
        y2 = M.apply(v)
    with P.ParallelSchwarz(prob, workers=3) as M3:
        assert np.array_equal(M3.apply(v), y2)
    assert its == int(g["it"]) and conv == bool(g["conv"])
    assert rel(x, g["x"]) <= 1e-10
    assert np.allclose(hist, g["hist"], rtol=1e-9)


def test_config_goldens_are_consistent():
    """The committed config-scale goldens carry a history that is monotone and whose
    last value equals the true relative residual of the stored iterate."""
    import os

    from conftest import GOLDEN

    for name in ("cfg1", "cfg3", "cfg4"):
        path = os.path.join(GOLDEN, f"{name}_oracle.npz")
        if not os.path.exists(path):
            continue
        g = dict(np.load(path))
        assert np.all(np.diff(g["hist"]) <= 0)
        assert float(g["true_rel_res"]) == pytest.approx(float(g["hist"][-1]), rel=1e-6)
        assert len(g["hist"]) == int(g["its"]) + 1
