"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference hot path (reference package
``maxwelldd``, /root/reference/pkg/src/maxwelldd) used as the parity checker
for the device implementation.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may
import it; the product package never does.

Pinned: tests/test_oracle_golden.py checks every function here against
golden fixtures produced by running the reference itself
(tests/golden/make_golden.py, committed with the fixtures).

Inputs are plain arrays (mesh arrays, DOF maps, DOF sets, R0), so the oracle
does not depend on the product package.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

EA = np.array([0, 0, 0, 1, 1, 2])
EB = np.array([1, 2, 3, 2, 3, 3])
LOCAL_FACES = np.array([(1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2)])


# ------------------------------------------------------------ element level
def tet_gradients(coords):
    """Barycentric gradients (nt,4,3) and volumes — reference fem.py:154-167."""
    b = np.transpose(coords[:, 1:] - coords[:, :1], (0, 2, 1))
    det = np.linalg.det(b)
    binv = np.linalg.inv(b)
    g = np.empty((coords.shape[0], 4, 3))
    g[:, 1:] = binv
    g[:, 0] = -binv.sum(axis=1)
    return g, det / 6.0


def element_matrices(coords, signs):
    """Oriented 6x6 stiffness / mass — reference fem.py:177-195."""
    g, vol = tet_gradients(coords)
    curl = 2.0 * np.cross(g[:, EA], g[:, EB])
    s = np.einsum("tec,tfc->tef", curl, curl) * vol[:, None, None]
    d = np.einsum("tic,tjc->tij", g, g)
    lam2 = (np.ones((4, 4)) + np.eye(4)) / 20.0
    a, b = EA, EB
    m = (
        d[:, b[:, None], b[None, :]] * lam2[a[:, None], a[None, :]]
        - d[:, b[:, None], a[None, :]] * lam2[a[:, None], b[None, :]]
        - d[:, a[:, None], b[None, :]] * lam2[b[:, None], a[None, :]]
        + d[:, a[:, None], a[None, :]] * lam2[b[:, None], b[None, :]]
    ) * vol[:, None, None]
    o = signs[:, :, None] * signs[:, None, :]
    return s * o, m * o, vol


def _coo_csr(rows, cols, vals, n, dtype):
    m = sp.coo_matrix((vals.astype(dtype), (rows, cols)), shape=(n, n)).tocsr()
    m.sort_indices()
    return m


def _scatter(dof, el):
    r = np.repeat(dof[:, :, None], dof.shape[1], axis=2)
    c = np.repeat(dof[:, None, :], dof.shape[1], axis=1)
    keep = (r >= 0) & (c >= 0)
    return r[keep], c[keep], el[keep]


def triangle_mass(pts):
    """3x3 tangential mass per boundary triangle — reference fem.py:286-316."""
    e1, e2 = pts[:, 1] - pts[:, 0], pts[:, 2] - pts[:, 0]
    nv = np.cross(e1, e2)
    a2 = np.linalg.norm(nv, axis=1)
    nh = nv / a2[:, None]
    g = np.stack(
        [np.cross(nh, pts[:, 2] - pts[:, 1]), np.cross(nh, pts[:, 0] - pts[:, 2]), np.cross(nh, pts[:, 1] - pts[:, 0])],
        axis=1,
    ) / a2[:, None, None]
    te = [(0, 1), (0, 2), (1, 2)]
    out = np.zeros((len(pts), 3, 3))
    for lam in ([0.5, 0.5, 0.0], [0.5, 0.0, 0.5], [0.0, 0.5, 0.5]):
        w = np.stack([lam[a] * g[:, b] - lam[b] * g[:, a] for a, b in te], axis=1)
        out += np.einsum("fec,fgc->feg", w, w)
    return out * (a2 / 2.0 / 3.0)[:, None, None]


def face_edge_ids(vertices_count, edges, faces):
    nv = vertices_count
    ek = edges[:, 0].astype(np.int64) * nv + edges[:, 1]
    pairs = faces[:, [[0, 1], [0, 2], [1, 2]]]
    return np.searchsorted(ek, pairs[..., 0].astype(np.int64) * nv + pairs[..., 1])


def boundary_mass(vertices, edges, faces, edge_to_dof, n):
    """Boundary mass over `faces` into an n x n CSR — reference fem.py:332-353."""
    if len(faces) == 0:
        return sp.csr_matrix((n, n))
    m = triangle_mass(vertices[faces])
    dof = edge_to_dof[face_edge_ids(len(vertices), edges, faces)]
    r, c, v = _scatter(dof, m)
    return _coo_csr(r, c, v, n, float)


def assemble(mesh, edge_to_dof, ndof, k, xi, eps=1.0, mu=1.0, sigma=0.0, bc="pec"):
    """A, S, M, Dk (+Mb) — reference fem.py:233-279.  `mesh` needs vertices,
    tets, edges, tet_edges, tet_edge_signs, boundary_faces."""
    nt = len(mesh["tets"])
    eps_a = np.broadcast_to(np.asarray(eps, float), (nt,))
    mu_a = np.broadcast_to(np.asarray(mu, float), (nt,))
    sig_a = np.broadcast_to(np.asarray(sigma, float), (nt,))
    homog = all(np.ndim(x) == 0 for x in (eps, mu, sigma)) and (eps, mu, sigma) == (1.0, 1.0, 0.0)
    s_el, m_el, _ = element_matrices(mesh["vertices"][mesh["tets"]], mesh["tet_edge_signs"])
    dof = edge_to_dof[mesh["tet_edges"]]
    S = _coo_csr(*_scatter(dof, s_el), ndof, float)
    M = _coo_csr(*_scatter(dof, m_el), ndof, float)
    if homog:
        A = S.astype(complex)
        A.data = S.data - (k**2 + 1j * xi) * M.data
    else:
        w = k**2 * eps_a + 1j * (xi * eps_a + k * sig_a)
        A = _coo_csr(*_scatter(dof, s_el / mu_a[:, None, None] - w[:, None, None] * m_el), ndof, complex)
    Mb = None
    if bc == "impedance":
        Mb = boundary_mass(mesh["vertices"], mesh["edges"], mesh["boundary_faces"], edge_to_dof, ndof)
        A = (A - 1j * (1.0 if xi >= 0 else -1.0) * k * Mb).tocsr()
        A.sort_indices()
    Dk = (S + k**2 * M).tocsr()
    Dk.sort_indices()
    return {"A": A, "S": S, "M": M, "Dk": Dk, "Mb": Mb}


_QA = (5.0 + 3.0 * np.sqrt(5.0)) / 20.0
_QB = (5.0 - np.sqrt(5.0)) / 20.0


def rhs(mesh, edge_to_dof, ndof, source):
    """4-point load vector — reference fem.py:367-390."""
    coords = mesh["vertices"][mesh["tets"]]
    g, vol = tet_gradients(coords)
    dof = edge_to_dof[mesh["tet_edges"]]
    out = np.zeros(ndof, dtype=complex)
    keep = dof >= 0
    for q in range(4):
        lam = np.full(4, _QB)
        lam[q] = _QA
        pts = np.einsum("i,tic->tc", lam, coords)
        f = np.asarray(source(pts), dtype=complex)
        w = lam[EA][None, :, None] * g[:, EB] - lam[EB][None, :, None] * g[:, EA]
        c = np.einsum("tec,tc->te", w, f) * mesh["tet_edge_signs"] * (vol / 4.0)[:, None]
        np.add.at(out, dof[keep], c[keep])
    return out


def gaussian(center=(0.5, 0.5, 0.5), alpha=400.0, amp=-1.0, direction=(1.0, 1.0, 1.0)):
    c = np.asarray(center, float)
    d = np.asarray(direction, float)

    def f(points):
        r2 = ((points - c) ** 2).sum(axis=-1)
        return (amp * np.exp(-alpha * r2))[..., None] * d

    return f


# ------------------------------------------------------------ local problems
def subdomain_faces(tets, elems, nv):
    """Faces incident to exactly one tet of `elems` — reference decomp.py:129-137."""
    tri = np.sort(tets[elems][:, LOCAL_FACES].reshape(-1, 3), axis=1).astype(np.int64)
    keys = (tri[:, 0] * nv + tri[:, 1]) * nv + tri[:, 2]
    uk, cnt = np.unique(keys, return_counts=True)
    b = uk[cnt == 1]
    return np.stack([b // (nv * nv), (b // nv) % nv, b % nv], axis=1)


def impedance_local_matrix(mesh, edge_to_dof, kept_edges, gdofs, elems, k, xi, eps=1.0, mu=1.0, sigma=0.0):
    """Submesh assembly + boundary impedance — reference precond.py:82-139 (local_bc='impedance')."""
    nt = len(mesh["tets"])
    eps_a = np.broadcast_to(np.asarray(eps, float), (nt,))[elems]
    mu_a = np.broadcast_to(np.asarray(mu, float), (nt,))[elems]
    sig_a = np.broadcast_to(np.asarray(sigma, float), (nt,))[elems]
    n = len(gdofs)
    e2l = np.full(len(mesh["edges"]), -1, dtype=np.int64)
    e2l[kept_edges[gdofs]] = np.arange(n)
    s_el, m_el, _ = element_matrices(mesh["vertices"][mesh["tets"][elems]], mesh["tet_edge_signs"][elems])
    w = k**2 * eps_a + 1j * (xi * eps_a + k * sig_a)
    a_el = s_el / mu_a[:, None, None] - w[:, None, None] * m_el
    A = sp.coo_matrix(
        (lambda r, c, v: (v, (r, c)))(*_scatter(e2l[mesh["tet_edges"][elems]], a_el)), shape=(n, n)
    ).tocsr()
    bf = subdomain_faces(mesh["tets"], elems, len(mesh["vertices"]))
    mb = boundary_mass(mesh["vertices"], mesh["edges"], bf, e2l, n)
    A = (A - 1j * (1.0 if xi >= 0 else -1.0) * k * mb).tocsr()
    A.sort_indices()
    return A


class _Dense:
    def __init__(self, a):
        self.lu = sla.lu_factor(np.asarray(a, dtype=complex), check_finite=False)

    def solve(self, b):
        return sla.lu_solve(self.lu, b, check_finite=False)


class _Sparse:
    def __init__(self, a):
        self.f = spla.splu(sp.csc_matrix(a, dtype=complex))

    def solve(self, b):
        return self.f.solve(np.asarray(b, dtype=complex))


class Schwarz:
    """One/two-level AS, RAS, ImpRAS — reference precond.py:147-247.

    `local` holds the local matrices (minors for as/ras, submesh matrices
    for impras); factors are dense LU (as the reference) or SuperLU for
    sizes where dense is infeasible.
    """

    def __init__(self, dof_sets, pou, local, family="as", levels="one", correction="additive",
                 R0=None, A0=None, A_corr=None, ndof=None, solver="auto"):
        self.dof_sets = dof_sets
        self.pou = pou
        self.family = family
        self.levels = levels
        self.correction = correction
        self.ndof = ndof
        self.A_corr = A_corr
        self.R0 = R0

        def fac(a):
            use_dense = solver == "dense" or (solver == "auto" and a.shape[0] <= 3000)
            return _Dense(a.toarray() if sp.issparse(a) else a) if use_dense else _Sparse(a)

        self.factors = [fac(a) for a in local]
        self.coarse = fac(A0) if levels == "two" else None

    def one_level(self, v):
        out = np.zeros(self.ndof, dtype=complex)
        weighted = self.family in ("ras", "impras")
        for d, w, f in zip(self.dof_sets, self.pou, self.factors):
            u = f.solve(v[d])
            if weighted:
                u = w * u
            out[d] += u
        return out

    def coarse_solve(self, v):
        return self.R0.T @ self.coarse.solve(self.R0 @ v)

    def apply(self, v):
        v = np.asarray(v, dtype=complex)
        if self.levels == "one":
            return self.one_level(v)
        gv = self.coarse_solve(v)
        if self.correction == "additive":
            return self.one_level(v) + gv
        t = v - self.A_corr @ gv
        if self.correction == "adef1":
            return self.one_level(t) + gv
        y = self.one_level(t)
        return y - self.coarse_solve(self.A_corr @ y) + gv

    __call__ = apply


def minors(A, dof_sets):
    """Exact minors R A R^T — reference linalg.py:48-70 / precond.py:166-171."""
    A = sp.csr_matrix(A)
    return [A[d][:, d] for d in dof_sets]


# ------------------------------------------------------------------ GMRES
def gmres(op, b, precond=None, tol=1e-6, maxit=200, side="right", weight=None, x0=None, max_iters=None):
    """MGS2 GMRES with complex Givens rotations — reference krylov.py:64-209.

    Returns (x, history, iterations, converged).  ``max_iters`` truncates the
    run (used only for the bounded CPU-baseline sample in bench.py).
    """
    amv = op if callable(op) else (lambda v: op @ v)
    mmv = None if precond is None else (precond if callable(precond) else (lambda v: precond @ v))
    dmv = (lambda v: v.copy()) if weight is None else (lambda v: weight @ v)
    b = np.asarray(b, dtype=complex)
    n = b.shape[0]
    x0 = np.zeros(n, dtype=complex) if x0 is None else np.asarray(x0, dtype=complex)
    r0 = b - amv(x0)
    if side == "right":
        cmv = (lambda v: amv(mmv(v))) if mmv else amv
    else:
        if mmv:
            r0 = mmv(r0)
        cmv = (lambda v: mmv(amv(v))) if mmv else amv
    dr0 = dmv(r0)
    beta = np.sqrt(np.vdot(r0, dr0).real)
    if beta == 0.0:
        return x0, np.array([0.0]), 0, True
    V, DV = [r0 / beta], [dr0 / beta]
    H = np.zeros((maxit + 1, maxit), dtype=complex)
    cs = np.zeros(maxit, dtype=complex)
    sn = np.zeros(maxit, dtype=complex)
    g = np.zeros(maxit + 1, dtype=complex)
    g[0] = beta
    hist = [1.0]
    conv = False
    m = 0
    limit = maxit if max_iters is None else min(maxit, max_iters)
    for m in range(1, limit + 1):
        w = cmv(V[m - 1])
        dw = dmv(w)
        col = np.zeros(m + 1, dtype=complex)
        for _ in range(2):
            for j in range(m):
                h = np.vdot(V[j], dw)
                col[j] += h
                w = w - h * V[j]
                dw = dw - h * DV[j]
        hl = np.sqrt(max(np.vdot(w, dw).real, 0.0))
        col[m] = hl
        brk = hl <= 1e-13 * np.abs(col).max()
        if not brk:
            V.append(w / hl)
            DV.append(dw / hl)
        for j in range(m - 1):
            t = cs[j] * col[j] + sn[j] * col[j + 1]
            col[j + 1] = -np.conj(sn[j]) * col[j] + cs[j] * col[j + 1]
            col[j] = t
        den = np.hypot(abs(col[m - 1]), abs(col[m]))
        if den == 0.0:
            cs[m - 1], sn[m - 1] = 1.0, 0.0
        else:
            cs[m - 1] = abs(col[m - 1]) / den
            ph = col[m - 1] / abs(col[m - 1]) if abs(col[m - 1]) > 0 else 1.0
            sn[m - 1] = ph * np.conj(col[m]) / den
        H[: m + 1, m - 1] = col
        H[m - 1, m - 1] = cs[m - 1] * col[m - 1] + sn[m - 1] * col[m]
        H[m, m - 1] = 0.0
        g[m] = -np.conj(sn[m - 1]) * g[m - 1]
        g[m - 1] = cs[m - 1] * g[m - 1]
        hist.append(min(abs(g[m]) / beta, hist[-1]))
        if brk or hist[-1] <= tol:
            conv = True
            break
    y = np.zeros(m, dtype=complex)
    for i in range(m - 1, -1, -1):
        y[i] = (g[i] - H[i, i + 1: m] @ y[i + 1: m]) / H[i, i]
    upd = np.zeros(n, dtype=complex)
    for i in range(m):
        upd += y[i] * V[i]
    if side == "right" and mmv is not None:
        upd = mmv(upd)
    return x0 + upd, np.array(hist), m, conv
