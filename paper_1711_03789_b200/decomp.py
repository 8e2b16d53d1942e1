"""Overlapping box decompositions, partition of unity and the coarse link.

Host-side index work with the semantics of reference ``maxwelldd.decomp``
(/root/reference/pkg/src/maxwelldd/decomp.py:1-332): the subdomain element
sets, DOF sets and PoU weights are bit-identical to the reference's
(pinned against tests/golden).  Differences are in *how*:

* overlap growth (decomp.py:97-110) works on a window of cells around each
  box instead of full-mesh sparse products;
* the coarse restriction R0 (decomp.py:212-297, a Python loop over every
  fine edge in the reference) is fully vectorised and uses the exact closed
  form of the Whitney line integral,
  ``int_e w_ab . t = l_a(x0) l_b(x1) - l_a(x1) l_b(x0)``,
  which the reference evaluates with a (also exact) two-point Gauss rule; the
  values agree to rounding.

SURVEY.md §8f ranks moving this module off the Python path as the first
"next" row; it is setup-time input to the device hot path.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _lib
from .fem import EdgeSpace
from .linalg import selection_matrix
from .mesh import LOCAL_EDGES, LOCAL_FACES, Mesh, nesting_map

__all__ = [
    "CoarseLink",
    "Decomposition",
    "DecompositionError",
    "box_partition",
    "build_decomposition",
    "build_pou",
    "coarse_restriction",
    "extend_overlap",
    "impedance_dof_sets",
    "subdomain_boundary_faces",
    "subdomain_dof_sets",
]


class DecompositionError(ValueError):
    """Reference decomp.py:41."""


@dataclass(frozen=True)
class CoarseLink:
    space: EdgeSpace
    R0: sp.csr_matrix
    tet_map: np.ndarray


@dataclass(frozen=True)
class Decomposition:
    """Overlapping decomposition (reference decomp.py:52-70)."""

    space: EdgeSpace
    elements: list
    dofs: list
    pou: list
    overlap_layers: int
    p_axis: int
    H_sub: float
    coarse: CoarseLink | None = None

    @property
    def n_subdomains(self) -> int:
        return len(self.elements)

    def restriction(self, ell: int) -> sp.csr_matrix:
        return selection_matrix(self.dofs[ell], self.space.ndof)


# ------------------------------------------------------------- partitions
def box_partition(mesh: Mesh, p_axis: int) -> list:
    """Tets grouped into p^3 boxes by barycentre (reference decomp.py:77-86)."""
    if p_axis < 1 or mesh.cells_per_axis % p_axis != 0:
        raise DecompositionError(
            f"p_axis={p_axis} must divide cells_per_axis={mesh.cells_per_axis}"
        )
    box = np.clip((mesh.barycenters() * p_axis).astype(np.int64), 0, p_axis - 1)
    bid = (box[:, 0] * p_axis + box[:, 1]) * p_axis + box[:, 2]
    order = np.argsort(bid, kind="stable")
    bounds = np.searchsorted(bid[order], np.arange(p_axis**3 + 1))
    return [order[bounds[b]: bounds[b + 1]] for b in range(p_axis**3)]


def _cell_coords(mesh: Mesh, tets: np.ndarray) -> np.ndarray:
    n = mesh.cells_per_axis
    c = tets // 6
    return np.stack([c // (n * n), (c // n) % n, c % n], axis=1)


def _ragged(sets):
    ptr = np.zeros(len(sets) + 1, dtype=np.int64)
    ptr[1:] = np.cumsum([len(x) for x in sets])
    flat = np.ascontiguousarray(np.concatenate([np.asarray(x, dtype=np.int64) for x in sets])
                                if len(sets) else np.zeros(0, np.int64), dtype=np.int64)
    return ptr, flat


def extend_overlap(mesh: Mesh, partition: list, layers: int) -> list:
    """Grow each set by `layers` rings of vertex-touching tets (reference decomp.py:97-110).

    Threaded C++ (csrc/decomp.cpp, ``mdd_extend_overlap``): a tet touching a
    vertex of a set tet lies in a cell within one cell of it, so each ring is
    searched in the window of cells around the set.
    """
    if layers < 1:
        raise DecompositionError("layers must be >= 1")
    ptr, flat = _ragged(partition)
    tets = np.ascontiguousarray(mesh.tets, dtype=np.int64)
    op, oi = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)()
    _lib.check(_lib.lib.mdd_extend_overlap(mesh.cells_per_axis, mesh.n_vertices, _lib.ptr(tets, C.c_int64),
                                           len(partition), _lib.ptr(ptr, C.c_int64), _lib.ptr(flat, C.c_int64),
                                           int(layers), C.byref(op), C.byref(oi)))
    return _lib.take_ragged(op, oi, len(partition))


def _extend_overlap_numpy(mesh: Mesh, partition: list, layers: int) -> list:
    """Vectorised numpy form of :func:`extend_overlap` (kept as a cross-check in tests)."""
    n = mesh.cells_per_axis
    out = []
    for elems in partition:
        elems = np.asarray(elems, dtype=np.int64)
        if len(elems) == 0:
            out.append(elems)
            continue
        cc = _cell_coords(mesh, elems)
        lo = np.maximum(cc.min(axis=0) - layers, 0)
        hi = np.minimum(cc.max(axis=0) + layers, n - 1)
        ax = [np.arange(lo[a], hi[a] + 1) for a in range(3)]
        cells = ((ax[0][:, None, None] * n + ax[1][None, :, None]) * n + ax[2][None, None, :]).ravel()
        win = (cells[:, None] * 6 + np.arange(6)[None, :]).ravel()  # ascending tet ids
        mask = np.zeros(mesh.n_tets, dtype=bool)
        mask[elems] = True
        wt = mesh.tets[win]
        for _ in range(layers):
            verts = np.zeros(mesh.n_vertices, dtype=bool)
            verts[mesh.tets[mask].ravel()] = True
            mask[win] = verts[wt].any(axis=1)
        out.append(np.flatnonzero(mask))
    return out


# --------------------------------------------------------------- DOF sets
def _face_keys(tris: np.ndarray, nv: int) -> np.ndarray:
    t = np.sort(tris, axis=-1).astype(np.int64)
    return (t[..., 0] * nv + t[..., 1]) * nv + t[..., 2]


def subdomain_boundary_faces(mesh: Mesh, elems: np.ndarray) -> np.ndarray:
    """Faces incident to exactly one subdomain tet, sorted triples (reference decomp.py:129-137)."""
    nv = np.int64(mesh.n_vertices)
    keys = _face_keys(mesh.tets[elems][:, LOCAL_FACES].reshape(-1, 3), nv)
    uk, cnt = np.unique(keys, return_counts=True)
    b = uk[cnt == 1]
    return np.stack([b // (nv * nv), (b // nv) % nv, b % nv], axis=1)


def subdomain_dof_sets(space: EdgeSpace, elements: list) -> list:
    """Unknowns with zero trace on internal boundaries (reference decomp.py:140-176).

    Threaded C++ (csrc/decomp.cpp, ``mdd_subdomain_dofs``) for both the
    Whitney and the order-2 space; the numpy forms below are cross-checks."""
    mesh = space.mesh
    o2 = getattr(space, "order", 1) == 2
    ptr, flat = _ragged(elements)
    tets = np.ascontiguousarray(mesh.tets, dtype=np.int64)
    te = np.ascontiguousarray(mesh.tet_edges, dtype=np.int64)
    e2d = np.ascontiguousarray(space.edge_to_dof, dtype=np.int64)
    if o2:
        tf = np.ascontiguousarray(space.tet_faces, dtype=np.int64)
        f2d = np.ascontiguousarray(space.face_to_dof, dtype=np.int64)
        tf_p, f2d_p, nf, nfd = _lib.ptr(tf, C.c_int64), _lib.ptr(f2d, C.c_int64), len(f2d), space.n_face_dofs
    else:
        tf_p, f2d_p, nf, nfd = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)(), 0, 0
    op, oi = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)()
    _lib.check(_lib.lib.mdd_subdomain_dofs(
        mesh.cells_per_axis, mesh.n_vertices, _lib.ptr(tets, C.c_int64), _lib.ptr(te, C.c_int64), len(e2d),
        _lib.ptr(e2d, C.c_int64), int((e2d >= 0).sum()), tf_p, nf, f2d_p, nfd, len(elements),
        _lib.ptr(ptr, C.c_int64), _lib.ptr(flat, C.c_int64), C.byref(op), C.byref(oi)))
    return _lib.take_ragged(op, oi, len(elements))


def _subdomain_dof_sets_numpy(space: EdgeSpace, elements: list) -> list:
    if getattr(space, "order", 1) == 2:
        return _subdomain_dof_sets2(space, elements)
    mesh = space.mesh
    nv = np.int64(mesh.n_vertices)
    dom_keys = np.sort(_face_keys(mesh.boundary_faces, nv))
    ekeys = mesh.edges[:, 0].astype(np.int64) * nv + mesh.edges[:, 1]  # ascending by construction
    out = []
    for elems in elements:
        bf = subdomain_boundary_faces(mesh, elems)
        internal = bf[~np.isin(_face_keys(bf, nv), dom_keys)]
        member = np.unique(mesh.tet_edges[elems].ravel())
        if len(internal):
            pairs = internal[:, [[0, 1], [0, 2], [1, 2]]].reshape(-1, 2)
            excl = np.searchsorted(ekeys, pairs[:, 0] * nv + pairs[:, 1])
            member = member[~np.isin(member, excl)]
        d = space.edge_to_dof[member]
        out.append(np.sort(d[d >= 0]))
    return out


def _subdomain_dof_sets2(space, elements: list) -> list:
    """Order-2 restatement of the rule above (extension, BASELINE config 2):
    drop the edge DoFs of edges on internal subdomain-boundary faces and the
    face DoFs of those faces; keep everything else the subdomain tets touch."""
    mesh = space.mesh
    nv = np.int64(mesh.n_vertices)
    dom_keys = np.sort(_face_keys(mesh.boundary_faces, nv))
    ekeys = mesh.edges[:, 0].astype(np.int64) * nv + mesh.edges[:, 1]
    fkeys = _face_keys(space.faces, nv)  # ascending (np.unique order)
    ned, nfd = space.n_edge_dofs, space.n_face_dofs
    out = []
    for elems in elements:
        bf = subdomain_boundary_faces(mesh, elems)
        internal = bf[~np.isin(_face_keys(bf, nv), dom_keys)]
        medges = np.unique(mesh.tet_edges[elems].ravel())
        mfaces = np.unique(space.tet_faces[elems].ravel())
        if len(internal):
            pairs = internal[:, [[0, 1], [0, 2], [1, 2]]].reshape(-1, 2)
            medges = medges[~np.isin(medges, np.searchsorted(ekeys, pairs[:, 0] * nv + pairs[:, 1]))]
            mfaces = mfaces[~np.isin(mfaces, np.searchsorted(fkeys, _face_keys(internal, nv)))]
        ed = space.edge_to_dof[medges]
        ed = ed[ed >= 0]
        fd = space.face_to_dof[mfaces]
        fd = fd[fd >= 0]
        out.append(np.sort(np.concatenate([ed, ed + ned, fd + 2 * ned, fd + 2 * ned + nfd])))
    return out


def impedance_dof_sets(space: EdgeSpace, elements: list) -> list:
    """All kept unknowns of the subdomain tets (reference decomp.py:179-191)."""
    out = []
    for elems in elements:
        d = space.edge_to_dof[np.unique(space.mesh.tet_edges[elems].ravel())]
        out.append(np.sort(d[d >= 0]))
    return out


def build_pou(dof_sets: list, ndof: int) -> list:
    """Inverse multiplicities (reference decomp.py:194-205)."""
    mult = np.zeros(ndof, dtype=np.int64)
    for d in dof_sets:
        mult[d] += 1
    bad = np.flatnonzero(mult == 0)
    if len(bad):
        raise DecompositionError(
            f"{len(bad)} unknowns not covered by any subdomain (first: {bad[0]}); increase the overlap"
        )
    return [1.0 / mult[d] for d in dof_sets]


# -------------------------------------------------------- coarse restriction
def coarse_restriction(
    fine_space: EdgeSpace,
    coarse_space: EdgeSpace,
    tet_map: np.ndarray | None = None,
    continuity_tol: float = 1e-10,
) -> sp.csr_matrix:
    """R0[p, j] = line integral of coarse basis p along fine edge j (reference decomp.py:212-297).

    Threaded C++ (csrc/decomp.cpp, ``mdd_coarse_restriction``) with the exact
    closed form of the line integral; the numpy form below is a cross-check."""
    fine, coarse = fine_space.mesh, coarse_space.mesh
    if tet_map is None:
        tet_map = nesting_map(coarse, fine)
    arr = lambda a, t=np.int64: np.ascontiguousarray(a, dtype=t)  # noqa: E731
    fv, fte, fe, kept = arr(fine.vertices, np.float64), arr(fine.tet_edges), arr(fine.edges), arr(fine_space.kept_edges)
    cv, ctt, cte, cs, ce2d = (arr(coarse.vertices, np.float64), arr(coarse.tets), arr(coarse.tet_edges),
                              arr(coarse.tet_edge_signs), arr(coarse_space.edge_to_dof))
    tm = arr(tet_map)
    rp, cl, vl = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)(), C.POINTER(C.c_double)()
    bad = C.c_int64(-1)
    I64, F64 = C.c_int64, C.c_double
    code = _lib.lib.mdd_coarse_restriction(
        fine.n_vertices, _lib.ptr(fv, F64), fine.n_tets, _lib.ptr(fte, I64), _lib.ptr(fe, I64), len(kept),
        _lib.ptr(kept, I64), _lib.ptr(cv, F64), coarse.n_tets, _lib.ptr(ctt, I64), _lib.ptr(cte, I64),
        _lib.ptr(cs, I64), _lib.ptr(ce2d, I64), coarse_space.ndof, _lib.ptr(tm, I64), continuity_tol,
        C.byref(rp), C.byref(cl), C.byref(vl), C.byref(bad))
    if code == 7:  # MDD_EDECOMP
        raise DecompositionError(f"tangential trace discontinuity on fine edge {bad.value}")
    _lib.check(code)
    ncs = coarse_space.ndof
    try:
        indptr = np.ctypeslib.as_array(rp, shape=(ncs + 1,)).copy()
        nnz = int(indptr[-1])
        indices = np.ctypeslib.as_array(cl, shape=(max(nnz, 1),))[:nnz].astype(np.int32)
        data = np.ctypeslib.as_array(vl, shape=(max(nnz, 1),))[:nnz].copy()
    finally:
        for p in (rp, cl, vl):
            _lib.lib.mdd_free(C.cast(p, C.c_void_p))
    return sp.csr_matrix((data, indices, indptr.astype(np.int32)), shape=(ncs, fine_space.ndof))


def _coarse_restriction_numpy(
    fine_space: EdgeSpace,
    coarse_space: EdgeSpace,
    tet_map: np.ndarray | None = None,
    continuity_tol: float = 1e-10,
) -> sp.csr_matrix:
    fine, coarse = fine_space.mesh, coarse_space.mesh
    if tet_map is None:
        tet_map = nesting_map(coarse, fine)
    # unique (fine edge, coarse tet) incidences, kept fine edges only
    fe = fine.tet_edges.ravel()
    ct = np.repeat(tet_map, 6)
    key = np.unique(fe.astype(np.int64) * coarse.n_tets + ct)
    fe, ct = key // coarse.n_tets, key % coarse.n_tets
    jdof = fine_space.edge_to_dof[fe]
    keep = jdof >= 0
    fe, ct, jdof = fe[keep], ct[keep], jdof[keep]
    # barycentric coordinates of the fine edge endpoints in the coarse tet
    cc = coarse.tet_coords()
    binv = np.linalg.inv(np.transpose(cc[:, 1:] - cc[:, :1], (0, 2, 1)))
    x0 = fine.vertices[fine.edges[fe, 0]]
    x1 = fine.vertices[fine.edges[fe, 1]]

    def bary(x):
        lam = np.einsum("pij,pj->pi", binv[ct], x - cc[ct, 0])
        return np.concatenate([1.0 - lam.sum(axis=1, keepdims=True), lam], axis=1)

    l0, l1 = bary(x0), bary(x1)
    a, b = LOCAL_EDGES[:, 0], LOCAL_EDGES[:, 1]
    vals = (l0[:, a] * l1[:, b] - l1[:, a] * l0[:, b]) * coarse.tet_edge_signs[ct]  # (npair, 6)
    pdof = coarse_space.edge_to_dof[coarse.tet_edges[ct]]  # (npair, 6)
    rows = pdof.ravel()
    cols = np.repeat(jdof, 6)
    v = vals.ravel()
    ok = rows >= 0
    rows, cols, v = rows[ok], cols[ok], v[ok]
    # merge duplicates (same fine edge, same coarse dof): first coarse tet wins,
    # the others must agree to continuity_tol (reference decomp.py:278-286)
    gkey = cols.astype(np.int64) * coarse_space.ndof + rows
    order = np.argsort(gkey, kind="stable")
    gkey, rows, cols, v = gkey[order], rows[order], cols[order], v[order]
    first = np.ones(len(gkey), dtype=bool)
    first[1:] = gkey[1:] != gkey[:-1]
    grp = np.cumsum(first) - 1
    ref = v[first][grp]
    bad = np.abs(v - ref) > continuity_tol * np.maximum(1.0, np.abs(ref))
    if np.any(bad):
        i = np.flatnonzero(bad)[0]
        j_edge = fine_space.kept_edges[cols[i]]
        raise DecompositionError(
            f"tangential trace discontinuity on fine edge {j_edge}: {ref[i]} vs {v[i]}"
        )
    rows, cols, v = rows[first], cols[first], v[first]
    nz = v != 0.0
    r0 = sp.csr_matrix((v[nz], (rows[nz], cols[nz])), shape=(coarse_space.ndof, fine_space.ndof))
    r0.sort_indices()
    return r0


_KUHN_ORDERS = {p: i for i, p in enumerate(__import__("itertools").permutations((0, 1, 2)))}


def coarse_restriction_nonnested(fine_space: EdgeSpace, coarse_space: EdgeSpace) -> sp.csr_matrix:
    """R0 for a coarse Kuhn mesh that does not nest in the fine one (extension:
    the reference requires nesting, mesh.py:231-242; BASELINE config 2 pairs a
    fine N=30 with a coarse N=8 mesh; the paper's non-nested setting, §6.2).

    Entry (p, j) is still the line integral of coarse basis p along fine edge j
    (reference decomp.py:212-297), now over a fine edge that may cross coarse
    tets.  The edge is split at every coarse cell plane (nc x_a integer) and
    every Kuhn diagonal plane (nc (x_a - x_b) integer), found exactly in integer
    lattice arithmetic; on each piece the coarse Whitney function is affine, so
    the midpoint rule is exact.  Pieces of one edge are summed.  A piece lying
    on a coarse face may be attributed to either neighbour: the tangential
    trace along it is continuous.
    """
    fine, coarse = fine_space.mesh, coarse_space.mesh
    nf, nc = fine.cells_per_axis, coarse.cells_per_axis
    kept = fine_space.kept_edges
    lat = fine.lattice()
    L0 = lat[fine.edges[kept, 0]]
    L1 = lat[fine.edges[kept, 1]]
    dirs = np.array([[1, 0, 0], [0, 1, 0], [0, 0, 1], [1, -1, 0], [0, 1, -1], [1, 0, -1]], dtype=np.int64)
    F0 = nc * (L0 @ dirs.T)  # nc * x . dir, in units of 1/nf (exact integers)
    F1 = nc * (L1 @ dirs.T)
    lo, hi = np.minimum(F0, F1), np.maximum(F0, F1)
    kmin = lo // nf + 1  # smallest integer k with k*nf > lo
    K = int(max(1, ((hi - 1) // nf - kmin + 1).max(initial=0)))
    ss = [np.zeros((len(kept), 1)), np.ones((len(kept), 1))]
    for r in range(K):
        k = (kmin + r) * nf
        ok = (k > lo) & (k < hi)
        den = np.where(F1 != F0, F1 - F0, 1)
        ss.append(np.where(ok, (k - F0) / den, 1.0))
    s = np.sort(np.concatenate(ss, axis=1), axis=1)  # (ne, npts)
    sa, sb = s[:, :-1], s[:, 1:]
    ln = sb - sa
    e_idx, piece = np.nonzero(ln > 0)
    mid = 0.5 * (sa[e_idx, piece] + sb[e_idx, piece])
    x0 = fine.vertices[fine.edges[kept[e_idx], 0]]
    d = fine.vertices[fine.edges[kept[e_idx], 1]] - x0
    xm = x0 + mid[:, None] * d
    u = xm * nc
    cell = np.clip(np.floor(u).astype(np.int64), 0, nc - 1)
    loc = u - cell
    order = np.argsort(-loc, axis=1, kind="stable")
    perm = np.array([_KUHN_ORDERS[tuple(o)] for o in map(tuple, order)]) if len(order) else np.zeros(0, int)
    ct = ((cell[:, 0] * nc + cell[:, 1]) * nc + cell[:, 2]) * 6 + perm
    cc = coarse.tet_coords()
    binv = np.linalg.inv(np.transpose(cc[:, 1:] - cc[:, :1], (0, 2, 1)))
    lam = np.einsum("pij,pj->pi", binv[ct], xm - cc[ct, 0])
    lam = np.concatenate([1.0 - lam.sum(axis=1, keepdims=True), lam], axis=1)
    g = np.empty((len(ct), 4, 3))
    g[:, 1:] = binv[ct]
    g[:, 0] = -binv[ct].sum(axis=1)
    a, b = LOCAL_EDGES[:, 0], LOCAL_EDGES[:, 1]
    w = lam[:, a, None] * g[:, b] - lam[:, b, None] * g[:, a]  # (npc, 6, 3)
    vals = np.einsum("pec,pc->pe", w, d) * ln[e_idx, piece][:, None] * coarse.tet_edge_signs[ct]
    rows = coarse_space.edge_to_dof[coarse.tet_edges[ct]].ravel()
    cols = np.repeat(fine_space.edge_to_dof[kept[e_idx]], 6)
    v = vals.ravel()
    ok = rows >= 0
    r0 = sp.csr_matrix((v[ok], (rows[ok], cols[ok])), shape=(coarse_space.ndof, fine_space.ndof))
    r0.sum_duplicates()
    r0.eliminate_zeros()
    r0.sort_indices()
    return r0


def build_decomposition(
    space: EdgeSpace, p_axis: int, layers: int, coarse_space: EdgeSpace | None = None,
    allow_nonnested: bool = False,
) -> Decomposition:
    """Box partition + overlap + DOF sets + PoU (+ coarse link) (reference decomp.py:304-332).

    ``allow_nonnested`` (extension): a coarse mesh whose resolution does not
    divide the fine one gets the split-edge R0 of
    :func:`coarse_restriction_nonnested` and ``tet_map=None`` (the reference,
    and the default here, raise ``MeshError`` from the nesting check)."""
    mesh = space.mesh
    elements = extend_overlap(mesh, box_partition(mesh, p_axis), layers)
    dofs = subdomain_dof_sets(space, elements)
    pou = build_pou(dofs, space.ndof)
    coarse = None
    if coarse_space is not None and allow_nonnested and mesh.cells_per_axis % coarse_space.mesh.cells_per_axis:
        p1 = space.lowest_order() if getattr(space, "order", 1) == 2 else space
        r1 = coarse_restriction_nonnested(p1, coarse_space)
        r0 = sp.csr_matrix((r1.data, r1.indices, r1.indptr), shape=(coarse_space.ndof, space.ndof))
        coarse = CoarseLink(space=coarse_space, R0=r0, tet_map=None)
    elif coarse_space is not None:
        tmap = nesting_map(coarse_space.mesh, mesh)
        if getattr(space, "order", 1) == 2:
            # the lowest-order coarse space is nested in the Whitney part of the
            # order-2 space (first n_edge_dofs unknowns): R0 = [R0_1 | 0]
            r1 = coarse_restriction(space.lowest_order(), coarse_space, tmap)
            r0 = sp.csr_matrix((r1.data, r1.indices, r1.indptr), shape=(coarse_space.ndof, space.ndof))
        else:
            r0 = coarse_restriction(space, coarse_space, tmap)
        coarse = CoarseLink(space=coarse_space, R0=r0, tet_map=tmap)
    return Decomposition(
        space=space,
        elements=elements,
        dofs=dofs,
        pou=pou,
        overlap_layers=layers,
        p_axis=p_axis,
        H_sub=float(np.sqrt(3.0) / p_axis),
        coarse=coarse,
    )
