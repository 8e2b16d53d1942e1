"""Device assembly + SpMV parity (through the C-ABI) against the reference's
golden outputs and the pinned oracle.  Tolerances: entries up to
floating-point reassociation (north_star) -> 1e-12 relative."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden_csr, load_golden, mesh_dict, rel
from oracle import maxwell_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gs():
    return load_golden("system.npz")


def _space(n, bc="pec"):
    from paper_1711_03789_b200 import fem, mesh

    return fem.build_edge_space(mesh.build_cube_mesh(n), bc)


def _same_pattern(a, b):
    return np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)


def test_element_matrices_reference_tet(gpu, gs):
    from paper_1711_03789_b200 import fem

    s, m = fem.element_matrices(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1.0]]))
    assert np.abs(s - gs["ref_tet_S"]).max() <= 1e-14
    assert np.abs(m - gs["ref_tet_M"]).max() <= 1e-14


def test_element_matrices_batch_vs_oracle(gpu):
    from paper_1711_03789_b200 import fem

    rng = np.random.default_rng(3)
    c = rng.random((200, 4, 3))
    c[:, 1:] += np.eye(3)  # keep them non-degenerate
    sg = rng.choice([-1.0, 1.0], size=(200, 6))
    s, m, v = fem.element_matrices_batch(c, sg)
    so, mo, vo = O.element_matrices(c, sg)
    assert np.abs(s - so).max() <= 1e-11 * np.abs(so).max()
    assert np.abs(m - mo).max() <= 1e-11 * np.abs(mo).max()


def test_assembly_homogeneous_matches_reference(gpu, gs):
    from paper_1711_03789_b200 import fem

    s = _space(3)
    b = fem.assemble(s, fem.Coefficients(k=2.0, xi=4.0), source=fem.gaussian_source)
    for k in ("A", "S", "M", "Dk"):
        ref = golden_csr(gs, f"hom_{k}")
        got = getattr(b, k).to_scipy()
        assert _same_pattern(got, ref), k
        assert np.abs(got.data - ref.data).max() <= 1e-12 * np.abs(ref.data).max(), k
    assert rel(b.rhs, gs["hom_rhs"]) <= 1e-13


def test_assembly_heterogeneous_matches_reference(gpu, gs):
    from paper_1711_03789_b200 import fem

    s = _space(3)
    co = fem.Coefficients(k=3.0, xi=2.0, eps=gs["het_eps"], mu=gs["het_mu"], sigma=gs["het_sigma"])
    b = fem.assemble(s, co)
    for k in ("A", "S", "M", "Dk"):
        ref = golden_csr(gs, f"het_{k}")
        got = getattr(b, k).to_scipy()
        assert _same_pattern(got, ref), k
        assert np.abs(got.data - ref.data).max() <= 1e-12 * np.abs(ref.data).max(), k


@pytest.mark.parametrize("tag,xi", [("imp", 4.0), ("impneg", -4.0)])
def test_assembly_impedance_matches_reference(gpu, gs, tag, xi):
    from paper_1711_03789_b200 import fem

    s = _space(2, "impedance")
    b = fem.assemble(s, fem.Coefficients(k=2.0, xi=xi), source=fem.gaussian_source)
    assert np.abs((b.A.to_scipy() - golden_csr(gs, f"{tag}_A")).toarray()).max() <= 1e-12
    assert np.abs((b.Mb.to_scipy() - golden_csr(gs, f"{tag}_Mb")).toarray()).max() <= 1e-14
    assert rel(b.rhs, gs[f"{tag}_rhs"]) <= 1e-13


def test_rhs_callable_and_device_gaussian(gpu, gs):
    from paper_1711_03789_b200 import fem

    s = _space(3)
    zsrc = fem.GaussianSource(alpha=100.0, direction=(0.0, 0.0, 1.0))
    assert rel(fem.assemble_rhs(s, zsrc), gs["zrhs"]) <= 1e-13
    # arbitrary Python callable: evaluated on the host at the quadrature points
    f = lambda p: np.stack([np.sin(p[:, 0]), p[:, 1] ** 2, 1j * p[:, 2]], axis=1)
    want = O.rhs(mesh_dict(s.mesh), s.edge_to_dof, s.ndof, f)
    assert rel(fem.assemble_rhs(s, f), want) <= 1e-13


@pytest.mark.parametrize("n", [6, 12])
def test_assembly_vs_oracle_larger(gpu, n):
    from paper_1711_03789_b200 import fem

    s = _space(n)
    rng = np.random.default_rng(n)
    nt = s.mesh.n_tets
    eps, sig = 1 + 3 * rng.random(nt), rng.random(nt)
    b = fem.assemble(s, fem.Coefficients(k=5.0, xi=0.0, eps=eps, sigma=sig))
    want = O.assemble(mesh_dict(s.mesh), s.edge_to_dof, s.ndof, 5.0, 0.0, eps=eps, sigma=sig)
    for k in ("A", "S", "M", "Dk"):
        got = getattr(b, k).to_scipy()
        assert _same_pattern(got, want[k])
        assert np.abs(got.data - want[k].data).max() <= 1e-12 * np.abs(want[k].data).max()


def test_gradient_kernel(gpu):
    # S g = 0 for the DOFs of a discrete gradient (reference test_fem.py:114-129)
    from paper_1711_03789_b200 import fem

    s = _space(4)
    rng = np.random.default_rng(0)
    phi = rng.standard_normal(s.mesh.n_vertices)
    onb = np.zeros(s.mesh.n_vertices, bool)
    lat = s.mesh.lattice()
    onb[(lat == 0).any(1) | (lat == 4).any(1)] = True
    phi[onb] = 0.0
    g = fem.gradient_dof_vector(s, phi)
    b = fem.assemble(s, fem.Coefficients(k=1.0, xi=1.0))
    assert np.abs(b.S @ g).max() <= 1e-12 * np.abs(g).max() * 10


@pytest.mark.parametrize("cplx", [True, False])
def test_spmv_vs_scipy(gpu, cplx):
    from paper_1711_03789_b200.linalg import DeviceCSR

    rng = np.random.default_rng(7)
    m = sp.random(3000, 2500, density=0.004, random_state=7, format="csr")
    if cplx:
        m = m + 1j * sp.random(3000, 2500, density=0.004, random_state=8, format="csr")
    # a few long rows (R0-like) and empty rows
    m = sp.vstack([m, sp.csr_matrix(rng.standard_normal((2, 2500))), sp.csr_matrix((3, 2500))]).tocsr()
    d = DeviceCSR.from_scipy(m)
    x = rng.standard_normal(2500) + 1j * rng.standard_normal(2500)
    assert rel(d @ x, m @ x) <= 1e-14
    back = d.to_scipy()
    assert _same_pattern(back, m) and np.array_equal(back.data, m.data)


def test_spmv_system_matrix(gpu):
    from paper_1711_03789_b200 import fem

    s = _space(10)
    b = fem.assemble(s, fem.Coefficients(k=4.0, xi=16.0))
    x = np.random.default_rng(1).standard_normal(s.ndof) * (1 + 1j)
    assert rel(b.A @ x, b.A.to_scipy() @ x) <= 1e-14
