"""Second-order Nedelec space (BASELINE config 2): host DoF map and the CPU oracle.

The reference has Whitney elements only (reference fem.py:1-7), so the
order-2 oracle (oracle/nedelec2_oracle.py) is parity-unpinned against the
reference.  These tests tie it down instead by (a) its Whitney block
reproducing the lowest-order oracle, which test_oracle_golden.py pins to the
reference's own outputs, (b) exact identities of the basis, and (c) a
manufactured-solution convergence rate.
"""

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from conftest import mesh_dict
from oracle import maxwell_oracle as O1
from oracle import nedelec2_oracle as O2
from paper_1711_03789_b200 import decomp, fem, mesh


def _space2(n):
    return fem.build_edge_space(mesh.build_cube_mesh(n), "pec", order=2)


def _asm2(s, k, xi, **kw):
    return O2.assemble(s.mesh.vertices, s.mesh.tets, s.tet_dofs, s.ndof, k, xi, **kw)


def test_dof_counts_cfg2():
    # 2*180,990 interior edges + 2*318,600 interior faces at N=30
    s = _space2(30)
    assert (s.n_edge_dofs, s.n_face_dofs, s.ndof) == (180_990, 318_600, 999_180)


def test_dof_map_consistency():
    s = _space2(3)
    td = s.tet_dofs
    # every kept DoF is used; face DoFs appear in exactly two tets, edge DoFs in >= 2
    cnt = np.bincount(td[td >= 0], minlength=s.ndof)
    assert cnt.min() >= 2
    ned = s.n_edge_dofs
    assert np.all(cnt[2 * ned:] == 2)
    # the Whitney DoFs of each tet are the lowest-order DoFs of its sorted edges
    st = np.sort(s.mesh.tets, axis=1)
    nv = s.mesh.n_vertices
    keys = s.mesh.edges[:, 0] * nv + s.mesh.edges[:, 1]
    for t in range(0, s.mesh.n_tets, 7):
        for e, (a, b) in enumerate(zip(O2.EA, O2.EB)):
            eid = np.searchsorted(keys, st[t, a] * nv + st[t, b])
            assert td[t, e] == s.edge_to_dof[eid]
            assert td[t, 6 + e] == (s.edge_to_dof[eid] + ned if s.edge_to_dof[eid] >= 0 else -1)


def test_whitney_block_is_lowest_order():
    s = _space2(2)
    p1 = s.lowest_order()
    o2 = _asm2(s, 2.0, 4.0)
    o1 = O1.assemble(mesh_dict(s.mesh), p1.edge_to_dof, p1.ndof, 2.0, 4.0)
    ned = s.n_edge_dofs
    for k in ("A", "S", "M"):
        blk = o2[k][:ned][:, :ned].toarray()
        ref = o1[k].toarray()
        assert np.abs(blk - ref).max() <= 1e-13 * np.abs(ref).max()


def test_curl_of_gradients_vanishes_and_mass_spd():
    s = _space2(2)
    o = _asm2(s, 1.0, 0.0)
    ned = s.n_edge_dofs
    S, M = o["S"].toarray(), o["M"].toarray()
    assert np.abs(S[:, ned:2 * ned]).max() <= 1e-12 * np.abs(S).max()
    assert np.abs(S - S.T).max() <= 1e-14 * np.abs(S).max()
    assert np.linalg.eigvalsh(M).min() > 0


def test_element_rule_independence():
    # closed-form integrals of the monomials vs two quadrature degrees
    rng = np.random.default_rng(3)
    c = rng.random((5, 4, 3))
    s7, m7 = O2.element_matrices(c, O2.conical_rule(4))
    s9, m9 = O2.element_matrices(c, O2.conical_rule(5))
    assert np.abs(s7 - s9).max() <= 1e-12 * np.abs(s9).max()
    assert np.abs(m7 - m9).max() <= 1e-12 * np.abs(m9).max()


def _l2_error(s, u, field):
    lam, wq = O2.conical_rule(4)
    st = np.sort(s.mesh.tets, axis=1)
    coords = s.mesh.vertices[st]
    g, vol = O2.gradients(coords)
    phi, _ = O2.basis(lam, g)
    coef = np.where(s.tet_dofs >= 0, u[np.maximum(s.tet_dofs, 0)], 0.0)
    uh = np.einsum("tk,tqkc->tqc", coef, phi)
    pts = np.einsum("qi,tic->tqc", lam, coords)
    ex = field(pts)
    return np.sqrt(np.einsum("q,t,tq->", wq, vol, ((uh - ex) ** 2).sum(-1)))


def test_manufactured_solution_converges_at_second_order():
    # E = (sin pi y sin pi z, sin pi x sin pi z, sin pi x sin pi y) is divergence free,
    # satisfies PEC, and curl curl E = 2 pi^2 E; solve curl curl u - u = (2 pi^2 - 1) E
    pi = np.pi

    def field(x):
        X, Y, Z = x[..., 0], x[..., 1], x[..., 2]
        return np.stack([np.sin(pi * Y) * np.sin(pi * Z), np.sin(pi * X) * np.sin(pi * Z),
                         np.sin(pi * X) * np.sin(pi * Y)], axis=-1)

    errs = []
    for n in (2, 4):
        s = _space2(n)
        o = _asm2(s, 1.0, 0.0)
        K = (o["S"] - o["M"]).tocsc()
        b = O2.rhs(s.mesh.vertices, s.mesh.tets, s.tet_dofs, s.ndof,
                   lambda x: (2 * pi**2 - 1) * field(x), O2.conical_rule(5)).real
        u = spla.spsolve(K, b)
        errs.append(_l2_error(s, u, field))
    print("L2 errors", errs, errs[0] / errs[1])
    assert errs[0] / errs[1] > 3.2  # ~4 for O(h^2); lowest order would give ~2


def test_subdomain_dofs_match_bruteforce():
    s = _space2(4)
    d = decomp.build_decomposition(s, 2, 1)
    m = s.mesh
    nv = m.n_vertices
    st = np.sort(m.tets, axis=1)
    bkeys = {tuple(int(x) for x in f) for f in m.boundary_faces}

    def edges_of(t):
        return [(int(st[t, a]), int(st[t, b])) for a, b in zip(O2.EA, O2.EB)]

    def edge_dofs(t):
        return [(s.tet_dofs[t, e], s.tet_dofs[t, 6 + e]) for e in range(6)]

    def faces_of(t):
        return [tuple(int(st[t, i]) for i in f) for f in O2.FACES]

    def face_dofs(t):
        return [(s.tet_dofs[t, 12 + 2 * f], s.tet_dofs[t, 13 + 2 * f]) for f in range(4)]

    for ell in (0, 3, 7):
        ref = O2.subdomain_dofs(m.tets, edges_of, faces_of, edge_dofs, face_dofs, bkeys, d.elements[ell], nv)
        assert np.array_equal(d.dofs[ell], ref)
    mult = np.zeros(s.ndof)
    for x in d.dofs:
        mult[x] += 1
    assert mult.min() >= 1


def test_coarse_restriction_lives_on_whitney_dofs():
    s = _space2(4)
    c = fem.build_edge_space(mesh.build_cube_mesh(2))
    d2 = decomp.build_decomposition(s, 2, 1, c)
    d1 = decomp.build_decomposition(s.lowest_order(), 2, 1, c)
    R2, R1 = d2.coarse.R0, d1.coarse.R0
    assert R2.shape == (c.ndof, s.ndof)
    assert R2[:, s.n_edge_dofs:].nnz == 0
    assert abs(R2[:, : s.n_edge_dofs] - R1).max() == 0
    # Galerkin coarse matrix of the order-2 operator = the lowest-order one
    o2 = _asm2(s, 2.0, 3.0)
    o1 = O1.assemble(mesh_dict(s.mesh), s.edge_to_dof, s.n_edge_dofs, 2.0, 3.0)
    a2 = (R2 @ o2["A"] @ R2.T).toarray()
    a1 = (R1 @ o1["A"] @ R1.T).toarray()
    assert np.abs(a2 - a1).max() <= 1e-12 * np.abs(a1).max()


# ------------------------------------------------ non-nested coarse meshes
def _whitney_field_dofs(space, a, b):
    """Line integrals of E = a + b x x along the kept edges (midpoint rule is exact: E.t affine)."""
    m = space.mesh
    x0, x1 = m.vertices[m.edges[:, 0]], m.vertices[m.edges[:, 1]]
    e = a + np.cross(b, 0.5 * (x0 + x1))
    return ((x1 - x0) * e).sum(axis=1)[space.kept_edges]


def test_nonnested_restriction_equals_nested_when_nested():
    f = fem.build_edge_space(mesh.build_cube_mesh(6))
    c = fem.build_edge_space(mesh.build_cube_mesh(3))
    assert abs(decomp.coarse_restriction(f, c) - decomp.coarse_restriction_nonnested(f, c)).max() <= 1e-15


@pytest.mark.parametrize("nf,nc", [(5, 2), (7, 3), (30, 8)])
def test_nonnested_restriction_reproduces_whitney_fields(nf, nc):
    # coarse Whitney fields a + b x x are fine Whitney fields: R0^T maps their
    # coarse DoFs to their fine DoFs exactly, whatever the meshes' alignment
    f = fem.build_edge_space(mesh.build_cube_mesh(nf), "impedance")
    c = fem.build_edge_space(mesh.build_cube_mesh(nc), "impedance")
    R = decomp.coarse_restriction_nonnested(f, c)
    for a, b in (([1.0, 2.0, -3.0], [0.5, -1.0, 2.0]), ([0.0, 0.0, 1.0], [0.0, 0.0, 0.0])):
        a, b = np.array(a), np.array(b)
        assert np.abs(R.T @ _whitney_field_dofs(c, a, b) - _whitney_field_dofs(f, a, b)).max() <= 1e-13


def test_nonnested_restriction_vs_composite_quadrature():
    # brute force: composite midpoint rule with 4000 sub-intervals and point location;
    # psi.t jumps where the edge crosses a coarse face, so this is only O(1/n) accurate
    f = fem.build_edge_space(mesh.build_cube_mesh(5))
    c = fem.build_edge_space(mesh.build_cube_mesh(3))
    R = decomp.coarse_restriction_nonnested(f, c).toarray()
    cm = c.mesh
    nc = cm.cells_per_axis
    cc = cm.tet_coords()
    binv = np.linalg.inv(np.transpose(cc[:, 1:] - cc[:, :1], (0, 2, 1)))
    rng = np.random.default_rng(4)
    cols = rng.choice(f.ndof, 25, replace=False)
    n = 4000
    s = (np.arange(n) + 0.5) / n
    for j in cols:
        e = f.mesh.edges[f.kept_edges[j]]
        x0, x1 = f.mesh.vertices[e[0]], f.mesh.vertices[e[1]]
        x = x0 + s[:, None] * (x1 - x0)
        ref = np.zeros(c.ndof)
        for xi in x:
            # locate: try the 6 tets of the cell
            cell = np.clip(np.floor(xi * nc).astype(int), 0, nc - 1)
            cid = (cell[0] * nc + cell[1]) * nc + cell[2]
            for t in range(cid * 6, cid * 6 + 6):
                lam = binv[t] @ (xi - cc[t, 0])
                lam = np.concatenate([[1 - lam.sum()], lam])
                if lam.min() >= -1e-12:
                    break
            g = np.vstack([-binv[t].sum(axis=0), binv[t]])
            for le, (a, b) in enumerate(zip(O2.EA, O2.EB)):
                p = c.edge_to_dof[cm.tet_edges[t, le]]
                if p >= 0:
                    w = lam[a] * g[b] - lam[b] * g[a]
                    ref[p] += cm.tet_edge_signs[t, le] * (w @ (x1 - x0)) / n
        assert np.abs(R[:, j] - ref).max() <= 1e-4
