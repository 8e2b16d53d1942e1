"""CPU ORACLE — TEST INFRASTRUCTURE ONLY — second-order Nedelec (BASELINE config 2).

PARITY UNPINNED against the reference: the reference implements lowest-order
(Whitney) elements only (reference fem.py:1-7), so there is no
reference output to pin this module to ("cfg2: no oracle").
It is an independent restatement of the order-2 discretisation used by the
device path (paper_1711_03789_b200/csrc/nedelec2.cu) and is validated by:

* its Whitney block equals the lowest-order oracle (maxwell_oracle.assemble),
  which IS pinned to the reference's golden fixtures;
* exact properties: curl of the edge-gradient functions vanishes (zero
  stiffness columns), the mass matrix is symmetric positive definite;
* a manufactured-solution convergence test (L2 error ~ h^2).

Element matrices here come from numerical quadrature of explicitly written
basis functions and curls (not from the device path's closed-form monomial
tables).  Only tests/, __graft_entry__.smoke() and bench.py may import it.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.special import roots_jacobi

EA = np.array([0, 0, 0, 1, 1, 2])
EB = np.array([1, 2, 3, 2, 3, 3])
FACES = np.array([(1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2)])


def conical_rule(n):
    """Stroud conical-product rule (n^3 points, degree 2n-1); barycentric points, weights summing to 1."""
    out = []
    for alpha in (2.0, 1.0, 0.0):
        x, w = roots_jacobi(n, alpha, 0.0)
        out.append(((x + 1.0) / 2.0, w / w.sum()))
    (u, wu), (v, wv), (t, wt) = out
    U, V, T = np.meshgrid(u, v, t, indexing="ij")
    W = wu[:, None, None] * wv[None, :, None] * wt[None, None, :]
    x = U
    y = V * (1 - U)
    z = T * (1 - U) * (1 - V)
    lam = np.stack([1 - x - y - z, x, y, z], axis=-1).reshape(-1, 4)
    return lam, W.ravel()


def gradients(coords):
    """(nt,4,3) barycentric gradients and |volume| for tets (nt,4,3) in any vertex order."""
    b = np.transpose(coords[:, 1:] - coords[:, :1], (0, 2, 1))
    binv = np.linalg.inv(b)
    g = np.empty((coords.shape[0], 4, 3))
    g[:, 1:] = binv
    g[:, 0] = -binv.sum(axis=1)
    return g, np.abs(np.linalg.det(b)) / 6.0


def basis(lam, g):
    """Values and curls of the 20 basis functions at barycentric points.

    lam (Q,4); g (nt,4,3) -> phi (nt,Q,20,3), curl (nt,Q,20,3).
    Order: Whitney (6), grad(l_a l_b) (6), per face (a<b<c): l_c w_ab, l_a w_bc.
    """
    nt, Q = g.shape[0], lam.shape[0]
    phi = np.zeros((nt, Q, 20, 3))
    cur = np.zeros((nt, Q, 20, 3))
    L = lam[None, :, :, None]  # (1,Q,4,1)
    G = g[:, None, :, :]       # (nt,1,4,3)

    def w(a, b):
        return L[:, :, a] * G[:, :, b] - L[:, :, b] * G[:, :, a]

    def x(a, b):
        return np.broadcast_to(np.cross(g[:, a], g[:, b])[:, None, :], (nt, Q, 3))

    for e in range(6):
        a, b = EA[e], EB[e]
        phi[:, :, e] = w(a, b)
        cur[:, :, e] = 2.0 * x(a, b)
        phi[:, :, 6 + e] = L[:, :, a] * G[:, :, b] + L[:, :, b] * G[:, :, a]
    for f in range(4):
        a, b, c = FACES[f]
        la, lb, lc = (lam[None, :, i, None] for i in (a, b, c))
        phi[:, :, 12 + 2 * f] = lc * w(a, b)
        cur[:, :, 12 + 2 * f] = la * x(c, b) - lb * x(c, a) + 2.0 * lc * x(a, b)
        phi[:, :, 13 + 2 * f] = la * w(b, c)
        cur[:, :, 13 + 2 * f] = lb * x(a, c) - lc * x(a, b) + 2.0 * la * x(b, c)
    return phi, cur


def element_matrices(coords, rule=None):
    """S_e, M_e (nt,20,20) for tets (nt,4,3) given in basis-frame vertex order."""
    lam, wq = rule if rule is not None else conical_rule(4)
    coords = np.asarray(coords, dtype=float)
    S = np.empty((len(coords), 20, 20))
    M = np.empty((len(coords), 20, 20))
    for a in range(0, len(coords), 2048):  # chunks bound the (nt, Q, 20, 3) temporaries
        g, vol = gradients(coords[a:a + 2048])
        phi, cur = basis(lam, g)
        M[a:a + 2048] = np.einsum("q,tqkc,tqlc->tkl", wq, phi, phi) * vol[:, None, None]
        S[a:a + 2048] = np.einsum("q,tqkc,tqlc->tkl", wq, cur, cur) * vol[:, None, None]
    return S, M


def _scatter_csr(tdofs, el, n, dtype):
    keep = tdofs >= 0
    r = np.broadcast_to(tdofs[:, :, None], el.shape)
    c = np.broadcast_to(tdofs[:, None, :], el.shape)
    ok = keep[:, :, None] & keep[:, None, :]
    A = sp.coo_matrix((el[ok].astype(dtype), (r[ok], c[ok])), shape=(n, n)).tocsr()
    A.sum_duplicates()
    A.sort_indices()
    return A


def assemble(vertices, tets, tet_dofs, ndof, k, xi, eps=1.0, mu=1.0, sigma=0.0):
    """A, S, M, Dk of the order-2 space (same operator conventions as reference fem.py:233-279)."""
    st = np.sort(np.asarray(tets), axis=1)
    S_e, M_e = element_matrices(vertices[st])
    nt = len(st)
    S = _scatter_csr(tet_dofs, S_e, ndof, float)
    M = _scatter_csr(tet_dofs, M_e, ndof, float)
    eps_a = np.broadcast_to(np.asarray(eps, float), (nt,))
    mu_a = np.broadcast_to(np.asarray(mu, float), (nt,))
    sig_a = np.broadcast_to(np.asarray(sigma, float), (nt,))
    wgt = k**2 * eps_a + 1j * (xi * eps_a + k * sig_a)
    A = _scatter_csr(tet_dofs, S_e / mu_a[:, None, None] - wgt[:, None, None] * M_e, ndof, complex)
    Dk = (S + k**2 * M).tocsr()
    Dk.sort_indices()
    return {"A": A, "S": S, "M": M, "Dk": Dk}


def rhs(vertices, tets, tet_dofs, ndof, source, rule=None):
    """Load vector sum_T sum_q w_q |T| F(x_q) . phi_k(x_q) (np.add.at order)."""
    lam, wq = rule if rule is not None else conical_rule(3)
    st = np.sort(np.asarray(tets), axis=1)
    coords = vertices[st]
    g, vol = gradients(coords)
    phi, _ = basis(lam, g)
    pts = np.einsum("qi,tic->tqc", lam, coords)
    F = np.asarray(source(pts.reshape(-1, 3)), dtype=complex).reshape(len(st), len(wq), 3)
    loc = np.einsum("q,tqkc,tqc->tk", wq, phi, F) * vol[:, None]
    b = np.zeros(ndof, dtype=complex)
    keep = tet_dofs >= 0
    np.add.at(b, tet_dofs[keep], loc[keep])
    return b


def subdomain_dofs(tets, edges_of_tet, faces_of_tet, edge_dof, face_dofs, boundary_face_keys, elems, nv):
    """Order-2 subdomain DoF set by brute force (sets, small meshes only): all
    DoFs of the subdomain tets minus those on internal subdomain-boundary faces
    (their edges and the faces themselves)."""
    from collections import Counter

    cnt = Counter()
    for t in elems:
        v = tets[t]
        for f in FACES:
            cnt[tuple(sorted(int(v[i]) for i in f))] += 1
    internal = {f for f, c in cnt.items() if c == 1 and f not in boundary_face_keys}
    bad_edges = set()
    for f in internal:
        bad_edges |= {(f[0], f[1]), (f[0], f[2]), (f[1], f[2])}
    out = set()
    for t in elems:
        v = tets[t]
        for (a, b), d in zip(edges_of_tet(t), edge_dof(t)):
            if (a, b) not in bad_edges:
                out |= {x for x in d if x >= 0}
        for tri, d in zip(faces_of_tet(t), face_dofs(t)):
            if tri not in internal:
                out |= {x for x in d if x >= 0}
    return np.array(sorted(out), dtype=np.int64)
