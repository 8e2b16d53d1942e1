"""CPU ORACLE (geometry) — TEST INFRASTRUCTURE ONLY.

Plain-numpy restatement of the reference's mesh, edge-space and decomposition
builders (reference package ``maxwelldd``: mesh.py, fem.py:51-80, decomp.py),
so the oracle-side of every parity check, the golden generators and
``bench.py``'s CPU arms can build a whole problem without importing the
product package (and so without loading ``libmdd.so``).

Only ``tests/``, ``tests/golden/*.py``, ``__graft_entry__.smoke()`` and
``bench.py`` (``cpu_baseline`` leg and ``--impl reference`` arm) may import
this module.

Pinned: tests/test_oracle_golden.py compares every builder here with
tests/golden/mesh.npz and tests/golden/decomp.npz, which hold arrays produced
by the reference itself (tests/golden/make_golden.py) — index arrays
bit-identical, R0 values to 1e-14.

Everything is returned as dicts of plain arrays:

mesh  : n, vertices, tets, edges, tet_edges, tet_edge_signs,
        boundary_edge_flags, boundary_faces
space : mesh, bc, kept_edges, edge_to_dof, ndof
decomp: elements, dofs, pou, R0 (or None), tet_map
"""

from __future__ import annotations

import itertools

import numpy as np
import scipy.sparse as sp

LOCAL_EDGES = np.array([(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)], dtype=np.int64)
LOCAL_FACES = np.array([(1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2)], dtype=np.int64)
_ORDERS = tuple(itertools.permutations((0, 1, 2)))


# ------------------------------------------------------------------ mesh
def cube_mesh(n):
    """Kuhn-split unit cube — reference mesh.py:126-213.

    Vertex (i,j,k) -> (i*(n+1)+j)*(n+1)+k; cell-major tets, six per cell in
    ``itertools.permutations((0,1,2))`` order (mesh.py:42, 148-155), local
    vertices 2,3 swapped for odd permutations (mesh.py:157-165); edges are the
    unique (lo, hi) pairs in ascending lo*nv+hi order (mesh.py:167-175)."""
    n = int(n)
    m1 = n + 1
    nv = m1**3
    ar = np.arange(m1, dtype=np.int64)
    lat = np.stack(np.meshgrid(ar, ar, ar, indexing="ij"), axis=-1).reshape(-1, 3)
    stride = np.array([m1 * m1, m1, 1], dtype=np.int64)
    ac = np.arange(n, dtype=np.int64)
    base = np.stack(np.meshgrid(ac, ac, ac, indexing="ij"), axis=-1).reshape(-1, 3) @ stride
    offs = np.zeros((6, 4), dtype=np.int64)
    for p, order in enumerate(_ORDERS):
        acc = 0
        for s, ax in enumerate(order):
            acc += stride[ax]
            offs[p, s + 1] = acc
        inversions = sum(1 for a in range(3) for b in range(a + 1, 3) if order[a] > order[b])
        if inversions & 1:
            offs[p, [2, 3]] = offs[p, [3, 2]]
    tets = (base[:, None, None] + offs[None]).reshape(-1, 4)
    ends = tets[:, LOCAL_EDGES]
    lo, hi = ends.min(axis=2), ends.max(axis=2)
    ukeys, te = np.unique((lo * nv + hi).ravel(), return_inverse=True)
    tri = np.sort(tets[:, LOCAL_FACES], axis=2).reshape(-1, 3)
    uk, cnt = np.unique((tri[:, 0] * nv + tri[:, 1]) * nv + tri[:, 2], return_counts=True)
    bk = uk[cnt == 1]
    bfaces = np.stack([bk // (nv * nv), (bk // nv) % nv, bk % nv], axis=1)
    fe = bfaces[:, [[0, 1], [0, 2], [1, 2]]].reshape(-1, 2)
    return {
        "n": n,
        "vertices": lat.astype(np.float64) / n,
        "tets": tets,
        "edges": np.stack([ukeys // nv, ukeys % nv], axis=1),
        "tet_edges": te.reshape(-1, 6).astype(np.int64),
        "tet_edge_signs": np.where(ends[:, :, 0] < ends[:, :, 1], 1, -1).astype(np.int64),
        "boundary_edge_flags": np.isin(ukeys, fe[:, 0] * nv + fe[:, 1]),
        "boundary_faces": bfaces,
    }


def barycenters(mesh):
    return mesh["vertices"][mesh["tets"]].mean(axis=1)


def edge_half_coords(mesh):
    """Edge midpoints in half-cell units (integers); a grid plane x_a = c holds
    exactly the edges with half-coordinate 2c along a."""
    m1 = mesh["n"] + 1
    v = np.arange(len(mesh["vertices"]), dtype=np.int64)
    lat = np.stack([v // (m1 * m1), (v // m1) % m1, v % m1], axis=1)
    return lat[mesh["edges"][:, 0]] + lat[mesh["edges"][:, 1]]


def edge_space(mesh, bc="pec"):
    """DOF map — reference fem.py:71-80 (PEC drops flagged edges, impedance keeps all)."""
    ne = len(mesh["edges"])
    kept = np.flatnonzero(~mesh["boundary_edge_flags"]) if bc == "pec" else np.arange(ne)
    e2d = np.full(ne, -1, dtype=np.int64)
    e2d[kept] = np.arange(len(kept))
    return {"mesh": mesh, "bc": bc, "kept_edges": kept.astype(np.int64), "edge_to_dof": e2d, "ndof": int(len(kept))}


# --------------------------------------------------------- decomposition
def box_partition(mesh, p):
    """Tets binned into p^3 boxes by barycentre — reference decomp.py:77-86."""
    box = np.clip((barycenters(mesh) * p).astype(np.int64), 0, p - 1)
    bid = (box[:, 0] * p + box[:, 1]) * p + box[:, 2]
    order = np.argsort(bid, kind="stable")
    cut = np.searchsorted(bid[order], np.arange(p**3 + 1))
    return [order[cut[b]: cut[b + 1]] for b in range(p**3)]


def extend_overlap(mesh, partition, layers):
    """`layers` rings of vertex-sharing tets — reference decomp.py:97-110.

    The reference multiplies full-mesh incidence matrices; a tet sharing a
    vertex with a set tet lies at most one cell away, so each ring only needs
    the window of cells around the set."""
    n = mesh["n"]
    tets = mesh["tets"]
    nt, nv = len(tets), len(mesh["vertices"])
    out = []
    for elems in partition:
        c = elems // 6
        cc = np.stack([c // (n * n), (c // n) % n, c % n], axis=1)
        lo = np.maximum(cc.min(axis=0) - layers, 0)
        hi = np.minimum(cc.max(axis=0) + layers, n - 1)
        ax = [np.arange(lo[a], hi[a] + 1) for a in range(3)]
        cells = ((ax[0][:, None, None] * n + ax[1][None, :, None]) * n + ax[2][None, None, :]).ravel()
        win = (cells[:, None] * 6 + np.arange(6)[None, :]).ravel()
        mask = np.zeros(nt, dtype=bool)
        mask[elems] = True
        wt = tets[win]
        for _ in range(layers):
            touched = np.zeros(nv, dtype=bool)
            touched[tets[mask].ravel()] = True
            mask[win] = touched[wt].any(axis=1)
        out.append(np.flatnonzero(mask))
    return out


def _face_keys(tri, nv):
    t = np.sort(tri, axis=-1).astype(np.int64)
    return (t[..., 0] * nv + t[..., 1]) * nv + t[..., 2]


def subdomain_faces(mesh, elems):
    """Faces met by exactly one subdomain tet — reference decomp.py:129-137."""
    nv = np.int64(len(mesh["vertices"]))
    uk, cnt = np.unique(_face_keys(mesh["tets"][elems][:, LOCAL_FACES].reshape(-1, 3), nv), return_counts=True)
    b = uk[cnt == 1]
    return np.stack([b // (nv * nv), (b // nv) % nv, b % nv], axis=1)


def pec_dof_sets(space, elements):
    """Unknowns with zero trace on the internal subdomain boundary — reference decomp.py:140-176."""
    mesh = space["mesh"]
    nv = np.int64(len(mesh["vertices"]))
    dom = np.sort(_face_keys(mesh["boundary_faces"], nv))
    ekeys = mesh["edges"][:, 0].astype(np.int64) * nv + mesh["edges"][:, 1]
    out = []
    for elems in elements:
        bf = subdomain_faces(mesh, elems)
        internal = bf[~np.isin(_face_keys(bf, nv), dom)]
        member = np.unique(mesh["tet_edges"][elems].ravel())
        if len(internal):
            pr = internal[:, [[0, 1], [0, 2], [1, 2]]].reshape(-1, 2)
            member = member[~np.isin(member, np.searchsorted(ekeys, pr[:, 0] * nv + pr[:, 1]))]
        d = space["edge_to_dof"][member]
        out.append(np.sort(d[d >= 0]))
    return out


def impedance_dof_sets(space, elements):
    """All kept unknowns of the subdomain tets — reference decomp.py:179-191."""
    out = []
    for elems in elements:
        d = space["edge_to_dof"][np.unique(space["mesh"]["tet_edges"][elems].ravel())]
        out.append(np.sort(d[d >= 0]))
    return out


def pou_weights(dof_sets, ndof):
    """Inverse multiplicities — reference decomp.py:194-205."""
    mult = np.zeros(ndof, dtype=np.int64)
    for d in dof_sets:
        mult[d] += 1
    if np.any(mult == 0):
        raise ValueError(f"{int((mult == 0).sum())} unknowns not covered by any subdomain")
    return [1.0 / mult[d] for d in dof_sets]


def nesting_map(coarse, fine):
    """Fine tet -> coarse tet containing it — reference mesh.py:231-263."""
    nc = coarse["n"]
    if fine["n"] % nc:
        raise ValueError("fine resolution is not a multiple of the coarse resolution")
    cc = coarse["vertices"][coarse["tets"]]
    binv = np.linalg.inv(np.transpose(cc[:, 1:] - cc[:, :1], (0, 2, 1)))
    bary = barycenters(fine)
    cell = np.clip((bary * nc).astype(np.int64), 0, nc - 1)
    cand = ((cell[:, 0] * nc + cell[:, 1]) * nc + cell[:, 2])[:, None] * 6 + np.arange(6)[None, :]
    lam = np.einsum("tpij,tpj->tpi", binv[cand], bary[:, None, :] - cc[cand, 0])
    lam = np.concatenate([1.0 - lam.sum(axis=2, keepdims=True), lam], axis=2)
    return cand[np.arange(len(cand)), lam.min(axis=2).argmax(axis=1)]


def coarse_restriction(fine_space, coarse_space, tet_map):
    """R0[p, j] = line integral of coarse basis p along fine edge j — reference decomp.py:212-297.

    The reference loops over fine edges with a two-point Gauss rule (exact for
    the affine integrand); here the same integral in closed form,
    l_a(x0) l_b(x1) - l_a(x1) l_b(x0), over all (fine edge, coarse tet)
    incidences at once; where several coarse tets see one edge the first
    (lowest coarse tet id) value is kept, as the reference's first-wins rule
    (decomp.py:278-286)."""
    fine, coarse = fine_space["mesh"], coarse_space["mesh"]
    nct = len(coarse["tets"])
    key = np.unique(fine["tet_edges"].ravel().astype(np.int64) * nct + np.repeat(tet_map, 6))
    fe, ct = key // nct, key % nct
    jd = fine_space["edge_to_dof"][fe]
    ok = jd >= 0
    fe, ct, jd = fe[ok], ct[ok], jd[ok]
    cc = coarse["vertices"][coarse["tets"]]
    binv = np.linalg.inv(np.transpose(cc[:, 1:] - cc[:, :1], (0, 2, 1)))

    def bary(x):
        lam = np.einsum("pij,pj->pi", binv[ct], x - cc[ct, 0])
        return np.concatenate([1.0 - lam.sum(axis=1, keepdims=True), lam], axis=1)

    l0 = bary(fine["vertices"][fine["edges"][fe, 0]])
    l1 = bary(fine["vertices"][fine["edges"][fe, 1]])
    a, b = LOCAL_EDGES[:, 0], LOCAL_EDGES[:, 1]
    vals = (l0[:, a] * l1[:, b] - l1[:, a] * l0[:, b]) * coarse["tet_edge_signs"][ct]
    rows = coarse_space["edge_to_dof"][coarse["tet_edges"][ct]].ravel()
    cols = np.repeat(jd, 6)
    v = vals.ravel()
    ok = rows >= 0
    rows, cols, v = rows[ok], cols[ok], v[ok]
    g = cols.astype(np.int64) * coarse_space["ndof"] + rows
    order = np.argsort(g, kind="stable")
    g, rows, cols, v = g[order], rows[order], cols[order], v[order]
    first = np.ones(len(g), dtype=bool)
    first[1:] = g[1:] != g[:-1]
    rows, cols, v = rows[first], cols[first], v[first]
    nz = v != 0.0
    r0 = sp.csr_matrix((v[nz], (rows[nz], cols[nz])), shape=(coarse_space["ndof"], fine_space["ndof"]))
    r0.sort_indices()
    return r0


def decomposition(space, p, layers, coarse_space=None, family="as"):
    """Box partition + overlap + DOF sets + PoU (+R0) — reference decomp.py:304-332.

    ``family="impras"`` swaps in the impedance DOF sets and their PoU, as the
    reference's preconditioner setup does (precond.py:172-174)."""
    mesh = space["mesh"]
    elements = extend_overlap(mesh, box_partition(mesh, p), layers)
    dofs = impedance_dof_sets(space, elements) if family == "impras" else pec_dof_sets(space, elements)
    out = {"elements": elements, "dofs": dofs, "pou": pou_weights(dofs, space["ndof"]), "R0": None, "tet_map": None}
    if coarse_space is not None:
        out["tet_map"] = nesting_map(coarse_space["mesh"], mesh)
        out["R0"] = coarse_restriction(space, coarse_space, out["tet_map"])
    return out
