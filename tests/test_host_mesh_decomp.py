"""Host index work (mesh, decomposition) against the reference's golden outputs.

Index arrays must be bit-identical (reference mesh.py:126-263,
decomp.py:77-332); R0 values agree to rounding (the reference uses a
two-point Gauss rule, we use the exact closed form).
"""

import numpy as np
import pytest

from conftest import golden_csr, golden_ragged, load_golden
from paper_1711_03789_b200 import decomp, fem, mesh


@pytest.fixture(scope="module")
def gm():
    return load_golden("mesh.npz")


@pytest.fixture(scope="module")
def gd():
    return load_golden("decomp.npz")


@pytest.mark.parametrize("n", [1, 3])
def test_mesh_arrays_bit_identical(gm, n):
    m = mesh.build_cube_mesh(n)
    for f in ("vertices", "tets", "edges", "tet_edges", "tet_edge_signs", "boundary_edge_flags",
              "boundary_faces", "boundary_face_normals"):
        ref = gm[f"n{n}_{f}"]
        got = getattr(m, f)
        assert got.shape == ref.shape and np.array_equal(got, ref), f


def test_nesting_map(gm):
    assert np.array_equal(mesh.nesting_map(mesh.build_cube_mesh(1), mesh.build_cube_mesh(3)), gm["nest_3_1"])


def test_mesh_errors():
    with pytest.raises(mesh.MeshError):
        mesh.build_cube_mesh(0)
    with pytest.raises(mesh.MeshError):
        mesh.nesting_map(mesh.build_cube_mesh(2), mesh.build_cube_mesh(3))


def test_mesh_counts_and_volumes():
    m = mesh.build_cube_mesh(4)
    assert m.n_tets == 6 * 64
    assert m.n_vertices == 125
    assert np.allclose(m.tet_volumes(), 1.0 / (6 * 64))
    hc = m.edge_half_coords()
    assert hc.dtype == np.int32 and hc.min() >= 0 and hc.max() <= 8


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_decomposition_sets_bit_identical(gd, tag):
    n, p, layers, nc = gd[f"{tag}_case"]
    s = fem.build_edge_space(mesh.build_cube_mesh(int(n)), "pec")
    c = fem.build_edge_space(mesh.build_cube_mesh(int(nc)), "pec")
    d = decomp.build_decomposition(s, int(p), int(layers), coarse_space=c)
    for got, ref in zip(d.elements, golden_ragged(gd, f"{tag}_elements")):
        assert np.array_equal(got, ref)
    for got, ref in zip(d.dofs, golden_ragged(gd, f"{tag}_dofs")):
        assert np.array_equal(got, ref)
    for got, ref in zip(d.pou, golden_ragged(gd, f"{tag}_pou")):
        assert np.array_equal(got, ref)
    for got, ref in zip(decomp.impedance_dof_sets(s, d.elements), golden_ragged(gd, f"{tag}_impdofs")):
        assert np.array_equal(got, ref)
    assert np.array_equal(d.coarse.tet_map, gd[f"{tag}_tetmap"])
    r0 = golden_csr(gd, f"{tag}_R0").toarray()
    assert np.abs(d.coarse.R0.toarray() - r0).max() <= 1e-14


def test_impedance_space_decomposition(gd):
    s = fem.build_edge_space(mesh.build_cube_mesh(4), "impedance")
    c = fem.build_edge_space(mesh.build_cube_mesh(2), "impedance")
    d = decomp.build_decomposition(s, 2, 1, coarse_space=c)
    for got, ref in zip(d.dofs, golden_ragged(gd, "imp_dofs")):
        assert np.array_equal(got, ref)
    assert np.abs(d.coarse.R0.toarray() - golden_csr(gd, "imp_R0").toarray()).max() <= 1e-14


def test_pou_partition_of_unity():
    s = fem.build_edge_space(mesh.build_cube_mesh(6), "pec")
    d = decomp.build_decomposition(s, 3, 2)
    acc = np.zeros(s.ndof)
    for dofs, w in zip(d.dofs, d.pou):
        acc[dofs] += w
    assert np.abs(acc - 1.0).max() <= 4 * np.finfo(float).eps


def test_decomposition_errors():
    s = fem.build_edge_space(mesh.build_cube_mesh(4), "pec")
    with pytest.raises(decomp.DecompositionError):
        decomp.box_partition(s.mesh, 3)
    with pytest.raises(decomp.DecompositionError):
        decomp.extend_overlap(s.mesh, decomp.box_partition(s.mesh, 2), 0)
    with pytest.raises(decomp.DecompositionError):
        decomp.build_pou([np.array([0, 1])], s.ndof)


def test_coarse_equal_fine_is_identity():
    s = fem.build_edge_space(mesh.build_cube_mesh(2), "pec")
    r0 = decomp.coarse_restriction(s, s)
    assert np.abs(r0.toarray() - np.eye(s.ndof)).max() <= 1e-14


@pytest.mark.parametrize("n,p,layers,bc,order", [(12, 3, 2, "pec", 1), (8, 2, 1, "impedance", 1), (8, 4, 2, "pec", 2)])
def test_native_decomposition_matches_numpy(n, p, layers, bc, order):
    """csrc/decomp.cpp (threaded C++) against the vectorised numpy forms."""
    m = mesh.build_cube_mesh(n)
    s = fem.build_edge_space(m, bc, order=order)
    part = decomp.box_partition(m, p)
    el = decomp.extend_overlap(m, part, layers)
    el_np = decomp._extend_overlap_numpy(m, part, layers)
    assert all(np.array_equal(a, b) for a, b in zip(el, el_np))
    d = decomp.subdomain_dof_sets(s, el)
    d_np = decomp._subdomain_dof_sets_numpy(s, el)
    assert all(np.array_equal(a, b) for a, b in zip(d, d_np))
    c = fem.build_edge_space(mesh.build_cube_mesh(n // 2), bc)
    tm = mesh.nesting_map(c.mesh, m)
    assert np.array_equal(tm, mesh._nesting_map_numpy(c.mesh, m))
    p1 = s.lowest_order() if order == 2 else s
    r = decomp.coarse_restriction(p1, c, tm)
    r_np = decomp._coarse_restriction_numpy(p1, c, tm)
    # same values to rounding; entries that are zero up to ~1e-17 roundoff may be
    # stored by one form and exactly zero in the other
    assert abs(r - r_np).max() <= 1e-15
