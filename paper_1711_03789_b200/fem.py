"""Lowest-order Nedelec edge elements: spaces, coefficients and device assembly.

Public surface of reference ``maxwelldd.fem`` (/root/reference/pkg/src/
maxwelldd/fem.py:1-425).  ``assemble`` runs on the GPU (coloured element
scatter into CSR, csrc/assemble.cu) and returns :class:`SystemBundle` whose
matrices are :class:`~paper_1711_03789_b200.linalg.DeviceCSR`:

    A  = S_mu - M_w [- i*sign(xi)*k*Mb under an impedance boundary]
    Dk = S + k^2 M

with ``M_w`` weighted per element by ``k^2 eps + i(xi eps + k sigma)``
(reference fem.py:9-16, 233-279).  The load vector uses the reference's
4-point degree-2 rule (fem.py:367-390); a Python-callable source is evaluated
on the host at the quadrature points (user code), the rest is device work;
:class:`GaussianSource` (and :func:`gaussian_source`) is evaluated on the
device.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, replace

import numpy as np

from . import _lib
from .linalg import DeviceCSR, raise_for
from .mesh import LOCAL_EDGES, LOCAL_FACES, Mesh

__all__ = [
    "Coefficients",
    "EdgeSpace",
    "FemError",
    "GaussianSource",
    "NedelecSpace2",
    "SystemBundle",
    "assemble",
    "assemble_boundary_mass",
    "assemble_rhs",
    "build_edge_space",
    "element_matrices",
    "gaussian_source",
    "gradient_dof_vector",
    "interpolate_field",
]


class FemError(ValueError):
    """Reference fem.py:43."""


# ---------------------------------------------------------------- spaces
@dataclass(frozen=True)
class EdgeSpace:
    """Edge space with the boundary condition applied (reference fem.py:51-68)."""

    mesh: Mesh
    bc_kind: str
    kept_edges: np.ndarray
    edge_to_dof: np.ndarray
    _cache: dict = field(default_factory=dict, compare=False, repr=False)

    @property
    def ndof(self) -> int:
        return int(len(self.kept_edges))

    # device-resident copy of mesh + DOF map + CSR pattern
    def device(self) -> "DeviceSpace":
        d = self._cache.get("dev")
        if d is None:
            d = DeviceSpace(self)
            self._cache["dev"] = d
        return d

    def dof_half_coords(self) -> np.ndarray:
        """(ndof, 3) int32 edge midpoints in half-cell units (ND coordinates)."""
        c = self._cache.get("xyz")
        if c is None:
            c = np.ascontiguousarray(self.mesh.edge_half_coords()[self.kept_edges], dtype=np.int32)
            self._cache["xyz"] = c
        return c


class DeviceSpace:
    """Owner of the ``mdd_space`` handle for an :class:`EdgeSpace`."""

    def __init__(self, space: EdgeSpace):
        ctx = _lib.get_context()
        m = space.mesh
        self.ctx = ctx
        self._arrays = [
            np.ascontiguousarray(m.vertices, dtype=np.float64),
            np.ascontiguousarray(m.tets, dtype=np.int64),
            np.ascontiguousarray(m.tet_edges, dtype=np.int64),
            np.ascontiguousarray(m.tet_edge_signs, dtype=np.int64),
            np.ascontiguousarray(space.edge_to_dof, dtype=np.int64),
        ]
        v, t, te, sg, e2d = self._arrays
        h = C.c_void_p()
        try:
            _lib.check(
                _lib.lib.mdd_space_create(
                    ctx.handle,
                    m.cells_per_axis,
                    m.n_vertices,
                    _lib.ptr(v, C.c_double),
                    m.n_tets,
                    _lib.ptr(t, C.c_int64),
                    _lib.ptr(te, C.c_int64),
                    _lib.ptr(sg, C.c_int64),
                    m.n_edges,
                    _lib.ptr(e2d, C.c_int64),
                    space.ndof,
                    C.byref(h),
                )
            )
        except _lib.MddError as e:
            raise_for(e)
        self.handle = h
        self.nt = m.n_tets
        self.ndof = space.ndof

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            _lib.lib.mdd_space_destroy(h)
            self.handle = None


def build_edge_space(mesh: Mesh, bc: str = "pec", order: int = 1):
    """Reference fem.py:71-80: PEC drops boundary edges, impedance keeps all.

    ``order=2`` (extension, BASELINE config 2; the reference has Whitney
    elements only) returns a :class:`NedelecSpace2`.
    """
    if bc not in ("pec", "impedance"):
        raise FemError(f"unknown boundary condition {bc!r}")
    if order == 2:
        return build_nedelec2_space(mesh, bc)
    if order != 1:
        raise FemError(f"order must be 1 or 2, got {order!r}")
    kept = np.flatnonzero(~mesh.boundary_edge_flags) if bc == "pec" else np.arange(mesh.n_edges)
    e2d = np.full(mesh.n_edges, -1, dtype=np.int64)
    e2d[kept] = np.arange(len(kept))
    return EdgeSpace(mesh=mesh, bc_kind=bc, kept_edges=kept, edge_to_dof=e2d)


# ------------------------------------------------- second-order space
def stroud_rule(n: int = 3):
    """Conical-product (Stroud) rule on the tetrahedron: n^3 points, exact for
    degree 2n-1.  Returns barycentric points (n^3, 4) and weights summing to 1."""
    from scipy.special import roots_jacobi

    def gj(alpha):
        x, w = roots_jacobi(n, alpha, 0.0)  # weight (1-x)^alpha on [-1,1]
        return (1.0 + x) / 2.0, w / w.sum()

    u, wu = gj(2.0)
    v, wv = gj(1.0)
    t, wt = gj(0.0)
    pts, wts = [], []
    for i in range(n):
        for j in range(n):
            for k in range(n):
                x = u[i]
                y = v[j] * (1.0 - u[i])
                z = t[k] * (1.0 - u[i]) * (1.0 - v[j])
                pts.append((1.0 - x - y - z, x, y, z))
                wts.append(wu[i] * wv[j] * wt[k])
    return np.array(pts), np.array(wts)


@dataclass(frozen=True)
class NedelecSpace2:
    """Second-order Nedelec (first kind) space: 2 DoFs per edge, 2 per face.

    Extension for BASELINE config 2 (the reference implements Whitney elements
    only, reference fem.py:1-7).  Hierarchical basis in the frame
    of each tet's vertices sorted by global index (csrc/nedelec2.cu): Whitney
    w_ab, edge gradients grad(l_a l_b), face functions l_c w_ab and l_a w_bc.
    Global numbering: [Whitney DoFs in the lowest-order numbering | edge
    gradient DoFs | first face DoFs | second face DoFs], so the lowest-order
    space (and the lowest-order coarse space nested in it) sits on the first
    ``n_edge_dofs`` unknowns.
    """

    mesh: Mesh
    bc_kind: str
    kept_edges: np.ndarray
    edge_to_dof: np.ndarray
    faces: np.ndarray          # (nf, 3) sorted vertex triples
    tet_faces: np.ndarray      # (nt, 4) face ids in LOCAL_FACES order
    kept_faces: np.ndarray
    face_to_dof: np.ndarray    # index among kept faces, -1 if eliminated
    tet_dofs: np.ndarray       # (nt, 20) sorted-frame local -> global DoF (-1: eliminated)
    _cache: dict = field(default_factory=dict, compare=False, repr=False)

    order = 2

    @property
    def n_edge_dofs(self) -> int:
        return int(len(self.kept_edges))

    @property
    def n_face_dofs(self) -> int:
        return int(len(self.kept_faces))

    @property
    def ndof(self) -> int:
        return 2 * self.n_edge_dofs + 2 * self.n_face_dofs

    def lowest_order(self) -> EdgeSpace:
        """The Whitney space on the same mesh and boundary condition."""
        e = self._cache.get("p1")
        if e is None:
            e = EdgeSpace(mesh=self.mesh, bc_kind=self.bc_kind, kept_edges=self.kept_edges,
                          edge_to_dof=self.edge_to_dof)
            self._cache["p1"] = e
        return e

    def dof_coords(self) -> np.ndarray:
        """(ndof, 3) int32 DoF positions in sixth-cell units (edge midpoints,
        face centroids): vertex planes sit at multiples of 6 (ND separators)."""
        c = self._cache.get("xyz6")
        if c is None:
            lat = self.mesh.lattice()
            e = self.mesh.edges[self.kept_edges]
            ec = 3 * (lat[e[:, 0]] + lat[e[:, 1]])
            f = self.faces[self.kept_faces]
            fc = 2 * (lat[f[:, 0]] + lat[f[:, 1]] + lat[f[:, 2]])
            c = np.ascontiguousarray(np.concatenate([ec, ec, fc, fc]), dtype=np.int32)
            self._cache["xyz6"] = c
        return c

    def device(self) -> "DeviceSpace2":
        d = self._cache.get("dev")
        if d is None:
            d = DeviceSpace2(self)
            self._cache["dev"] = d
        return d


def build_nedelec2_space(mesh: Mesh, bc: str = "pec") -> NedelecSpace2:
    """Order-2 DoF map: PEC drops the DoFs of boundary edges and boundary faces."""
    if bc != "pec":
        raise FemError("order-2 spaces support bc='pec' only")
    p1 = build_edge_space(mesh, bc)
    nv = np.int64(mesh.n_vertices)
    tri = np.sort(mesh.tets[:, LOCAL_FACES], axis=2)  # (nt, 4, 3)
    fkeys = (tri[..., 0] * nv + tri[..., 1]) * nv + tri[..., 2]
    ukeys, tet_faces, cnt = np.unique(fkeys.ravel(), return_inverse=True, return_counts=True)
    tet_faces = tet_faces.reshape(-1, 4).astype(np.int64)
    faces = np.stack([ukeys // (nv * nv), (ukeys // nv) % nv, ukeys % nv], axis=1)
    kept_faces = np.flatnonzero(cnt == 2)
    f2d = np.full(len(faces), -1, dtype=np.int64)
    f2d[kept_faces] = np.arange(len(kept_faces))
    # sorted-frame local DoFs (csrc/nedelec2.cu): edges / faces of the sorted tet
    st = np.sort(mesh.tets, axis=1)
    ekeys = mesh.edges[:, 0] * nv + mesh.edges[:, 1]  # ascending
    a, b = LOCAL_EDGES[:, 0], LOCAL_EDGES[:, 1]
    eid = np.searchsorted(ekeys, st[:, a] * nv + st[:, b])  # (nt, 6)
    fa, fb, fc = LOCAL_FACES[:, 0], LOCAL_FACES[:, 1], LOCAL_FACES[:, 2]
    fid = np.searchsorted(ukeys, (st[:, fa] * nv + st[:, fb]) * nv + st[:, fc])  # (nt, 4)
    ned, nfd = len(p1.kept_edges), len(kept_faces)
    ed = p1.edge_to_dof[eid]
    fd = f2d[fid]
    td = np.empty((mesh.n_tets, 20), dtype=np.int64)
    td[:, 0:6] = ed
    td[:, 6:12] = np.where(ed >= 0, ed + ned, -1)
    td[:, 12:20:2] = np.where(fd >= 0, fd + 2 * ned, -1)
    td[:, 13:20:2] = np.where(fd >= 0, fd + 2 * ned + nfd, -1)
    return NedelecSpace2(mesh=mesh, bc_kind=bc, kept_edges=p1.kept_edges, edge_to_dof=p1.edge_to_dof,
                         faces=faces, tet_faces=tet_faces, kept_faces=kept_faces, face_to_dof=f2d,
                         tet_dofs=td)


_STROUD = None


def _rule():
    global _STROUD
    if _STROUD is None:
        _STROUD = stroud_rule(3)
    return _STROUD


class DeviceSpace2:
    """Owner of the ``mdd_space`` handle of a :class:`NedelecSpace2`."""

    def __init__(self, space: NedelecSpace2):
        ctx = _lib.get_context()
        m = space.mesh
        self.ctx = ctx
        qb, qw = _rule()
        self._arrays = [
            np.ascontiguousarray(m.vertices, dtype=np.float64),
            np.ascontiguousarray(m.tets, dtype=np.int64),
            np.ascontiguousarray(space.tet_dofs, dtype=np.int64),
            np.ascontiguousarray(qb, dtype=np.float64),
            np.ascontiguousarray(qw, dtype=np.float64),
        ]
        v, t, td, qbc, qwc = self._arrays
        h = C.c_void_p()
        try:
            _lib.check(
                _lib.lib.mdd_space2_create(
                    ctx.handle, m.cells_per_axis, m.n_vertices, _lib.ptr(v, C.c_double), m.n_tets,
                    _lib.ptr(t, C.c_int64), _lib.ptr(td, C.c_int64), space.ndof, len(qwc),
                    _lib.ptr(qbc, C.c_double), _lib.ptr(qwc, C.c_double), C.byref(h),
                )
            )
        except _lib.MddError as e:
            raise_for(e)
        self.handle = h
        self.nt = m.n_tets
        self.ndof = space.ndof

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            _lib.lib.mdd_space_destroy(h)
            self.handle = None


def element2_matrices(coords: np.ndarray):
    """20x20 order-2 element matrices (device) for tets (nt,4,3) in basis-frame vertex order."""
    ctx = _lib.get_context()
    c = np.ascontiguousarray(np.asarray(coords, dtype=np.float64).reshape(-1, 4, 3))
    nt = c.shape[0]
    s_el = np.empty((nt, 20, 20))
    m_el = np.empty((nt, 20, 20))
    _lib.check(_lib.lib.mdd_element2_matrices(ctx.handle, nt, _lib.ptr(c, C.c_double),
                                              _lib.ptr(s_el, C.c_double), _lib.ptr(m_el, C.c_double)))
    return s_el, m_el


@dataclass(frozen=True)
class Coefficients:
    """Per-element materials plus global k and xi (reference fem.py:83-123)."""

    k: float
    xi: float
    eps: np.ndarray | float = 1.0
    mu: np.ndarray | float = 1.0
    sigma: np.ndarray | float = 0.0

    def per_tet(self, n_tets: int):
        try:
            eps = np.broadcast_to(np.asarray(self.eps, dtype=float), (n_tets,))
            mu = np.broadcast_to(np.asarray(self.mu, dtype=float), (n_tets,))
            sigma = np.broadcast_to(np.asarray(self.sigma, dtype=float), (n_tets,))
        except ValueError as exc:
            raise FemError(f"coefficient arrays do not match {n_tets} elements") from exc
        if eps.min() <= 0 or mu.min() <= 0:
            raise FemError("eps and mu must be strictly positive")
        if sigma.min() < 0:
            raise FemError("sigma must be nonnegative")
        return eps, mu, sigma

    @property
    def homogeneous(self) -> bool:
        return (
            np.ndim(self.eps) == 0
            and np.ndim(self.mu) == 0
            and np.ndim(self.sigma) == 0
            and float(self.eps) == 1.0
            and float(self.mu) == 1.0
            and float(self.sigma) == 0.0
        )

    def with_xi(self, xi: float) -> "Coefficients":
        return replace(self, xi=xi)

    # C-ABI view (arrays kept alive by the returned holder)
    def to_c(self, n_tets: int):
        eps, mu, sigma = self.per_tet(n_tets)
        hold = []
        c = _lib.mdd_coeffs()
        c.k = float(self.k)
        c.xi = float(self.xi)
        c.homogeneous = 1 if self.homogeneous else 0
        for name, arr, scal in (("eps", eps, self.eps), ("mu", mu, self.mu), ("sigma", sigma, self.sigma)):
            if np.ndim(scal) == 0:
                setattr(c, name, C.POINTER(C.c_double)())
                setattr(c, name + "0", float(scal))
            else:
                a = np.ascontiguousarray(arr, dtype=np.float64)
                hold.append(a)
                setattr(c, name, _lib.ptr(a, C.c_double))
                setattr(c, name + "0", 0.0)
        return c, hold


@dataclass(frozen=True)
class SystemBundle:
    """Assembled matrices (reference fem.py:126-147); matrices live on the GPU."""

    space: EdgeSpace
    coefficients: Coefficients
    A: DeviceCSR
    S: DeviceCSR
    M: DeviceCSR
    Dk: DeviceCSR
    rhs: np.ndarray
    Mb: DeviceCSR | None = None

    @property
    def ndof(self) -> int:
        return self.space.ndof


# ----------------------------------------------------------- element data
def element_matrices(coords: np.ndarray):
    """S_e, M_e for one tet with local orientation (reference fem.py:198-207)."""
    c = np.ascontiguousarray(np.asarray(coords, dtype=float).reshape(1, 4, 3))
    b = c[0, 1:] - c[0, :1]
    if not np.linalg.det(b) > 0:
        raise FemError("tetrahedron with nonpositive volume")
    s_el, m_el, _ = element_matrices_batch(c, np.ones((1, 6)))
    return s_el[0], m_el[0]


def element_matrices_batch(coords: np.ndarray, signs: np.ndarray):
    """Device batch of element matrices (reference fem._element_matrices_batch)."""
    ctx = _lib.get_context()
    c = np.ascontiguousarray(coords, dtype=np.float64)
    sg = np.ascontiguousarray(signs, dtype=np.float64)
    nt = c.shape[0]
    s_el = np.empty((nt, 6, 6))
    m_el = np.empty((nt, 6, 6))
    vol = np.empty(nt)
    _lib.check(
        _lib.lib.mdd_element_matrices(
            ctx.handle, nt, _lib.ptr(c, C.c_double), _lib.ptr(sg, C.c_double),
            _lib.ptr(s_el, C.c_double), _lib.ptr(m_el, C.c_double), _lib.ptr(vol, C.c_double),
        )
    )
    return s_el, m_el, vol


# ------------------------------------------------------------------ sources
class GaussianSource:
    """``F(x) = amp * exp(-alpha |x - c|^2) * direction`` (device-evaluated).

    ``gaussian_source`` (reference fem.py:360-364) is amp=-1, alpha=400,
    c=(1/2,1/2,1/2), direction=(1,1,1).
    """

    def __init__(self, center=(0.5, 0.5, 0.5), alpha=400.0, amp=-1.0, direction=(1.0, 1.0, 1.0)):
        self.center = np.asarray(center, dtype=float)
        self.alpha = float(alpha)
        self.amp = float(amp)
        self.direction = np.asarray(direction, dtype=float)

    def __call__(self, points: np.ndarray) -> np.ndarray:
        r2 = ((points - self.center) ** 2).sum(axis=-1)
        f = self.amp * np.exp(-self.alpha * r2)
        return f[..., None] * self.direction


_GAUSS = GaussianSource()


def gaussian_source(points: np.ndarray) -> np.ndarray:
    """Reference fem.py:360-364 (host callable; assemble() evaluates it on device)."""
    return _GAUSS(points)


_QA = (5.0 + 3.0 * np.sqrt(5.0)) / 20.0
_QB = (5.0 - np.sqrt(5.0)) / 20.0
_QLAM = np.full((4, 4), _QB) + (_QA - _QB) * np.eye(4)


def assemble_rhs(space: EdgeSpace, source) -> np.ndarray:
    """Load vector with the 4-point degree-2 rule (reference fem.py:373-390)."""
    dev = space.device()
    rhs = np.empty(space.ndof, dtype=np.complex128)
    src = _GAUSS if source is gaussian_source else source
    try:
        if isinstance(src, GaussianSource):
            c = np.ascontiguousarray(src.center)
            d = np.ascontiguousarray(src.direction)
            _lib.check(
                _lib.lib.mdd_assemble_rhs_gaussian(
                    dev.handle, _lib.ptr(c, C.c_double), src.alpha, src.amp, _lib.ptr(d, C.c_double),
                    _lib.zptr(rhs),
                )
            )
        elif getattr(space, "order", 1) == 2:
            m = space.mesh
            coords = m.vertices[np.sort(m.tets, axis=1)]  # basis frame
            qb, _ = _rule()
            fv = np.empty((len(qb), m.n_tets, 3), dtype=np.complex128)
            for q in range(len(qb)):
                fv[q] = np.asarray(source(np.einsum("i,tic->tc", qb[q], coords)), dtype=complex)
            _lib.check(_lib.lib.mdd_assemble_rhs(dev.handle, _lib.zptr(fv), _lib.zptr(rhs)))
        else:
            coords = space.mesh.tet_coords()
            fv = np.empty((4, space.mesh.n_tets, 3), dtype=np.complex128)
            for q in range(4):
                pts = np.einsum("i,tic->tc", _QLAM[q], coords)
                fv[q] = np.asarray(source(pts), dtype=complex)
            _lib.check(_lib.lib.mdd_assemble_rhs(dev.handle, _lib.zptr(fv), _lib.zptr(rhs)))
    except _lib.MddError as e:
        raise_for(e)
    return rhs


# ----------------------------------------------------------------- assembly
def _bfaces(space: EdgeSpace) -> np.ndarray:
    return np.ascontiguousarray(space.mesh.boundary_faces, dtype=np.int64)


def assemble(space: EdgeSpace, coeffs: Coefficients, source=None, rows=None) -> SystemBundle:
    """Device assembly of the system bundle (reference fem.py:233-279).

    ``rows=(lo, hi)`` (sharded solves, no reference counterpart) assembles only the cells that
    touch an unknown in ``[lo, hi)``: those rows of the matrices are complete and bitwise equal
    to the full assembly, the others are not to be read (``distributed.needed_rows`` gives the
    range a rank needs).  Such an operator serves the sharded CGS2 loop, which multiplies a
    rank's owned rows only; the MGS2 loop with a sharded preconditioner keeps whole vectors and
    needs the whole matrix."""
    dev = space.device()
    cc, hold = coeffs.to_c(space.mesh.n_tets)
    imp = space.bc_kind == "impedance"
    bf = _bfaces(space) if imp else np.zeros((0, 3), dtype=np.int64)
    hA, hS, hM, hD, hMb = (C.c_void_p() for _ in range(5))
    try:
        if rows is not None:
            _lib.check(_lib.lib.mdd_space_set_row_window(dev.handle, int(rows[0]), int(rows[1])))
        try:
            _lib.check(
                _lib.lib.mdd_assemble(
                    dev.handle, C.byref(cc), 1 if imp else 0, len(bf), _lib.ptr(bf, C.c_int64),
                    C.byref(hA), C.byref(hS), C.byref(hM), C.byref(hD), C.byref(hMb),
                )
            )
        finally:
            if rows is not None:
                _lib.check(_lib.lib.mdd_space_set_row_window(dev.handle, -1, -1))
    except _lib.MddError as e:
        raise_for(e)
    ctx = dev.ctx
    A = DeviceCSR.from_handle(hA, ctx)
    S = DeviceCSR.from_handle(hS, ctx)
    M = DeviceCSR.from_handle(hM, ctx)
    Dk = DeviceCSR.from_handle(hD, ctx)
    Mb = DeviceCSR.from_handle(hMb, ctx) if imp else None
    rhs = assemble_rhs(space, source) if source is not None else np.zeros(space.ndof, dtype=complex)
    del hold
    return SystemBundle(space=space, coefficients=coeffs, A=A, S=S, M=M, Dk=Dk, rhs=rhs, Mb=Mb)


def assemble_boundary_mass(space: EdgeSpace) -> DeviceCSR:
    """Tangential boundary mass (reference fem.py:319-329), device-assembled."""
    if space.bc_kind != "impedance":
        raise FemError("boundary mass requires an impedance space")
    return assemble(space, Coefficients(k=1.0, xi=0.0)).Mb


# ------------------------------------------------------- interpolation (host)
def gradient_dof_vector(space: EdgeSpace, vertex_values: np.ndarray) -> np.ndarray:
    """Edge DOFs of grad(phi): phi[b] - phi[a] (reference fem.py:397-406)."""
    e = space.mesh.edges
    return (vertex_values[e[:, 1]] - vertex_values[e[:, 0]])[space.kept_edges]


def interpolate_field(space: EdgeSpace, field_fn) -> np.ndarray:
    """Two-point Gauss line integrals of the tangential field (reference fem.py:409-425)."""
    m = space.mesh
    a = m.vertices[m.edges[:, 0]]
    tang = m.vertices[m.edges[:, 1]] - a
    total = 0.0
    for s in 0.5 + np.array([-1.0, 1.0]) / (2.0 * np.sqrt(3.0)):
        total = total + 0.5 * np.einsum("ec,ec->e", np.asarray(field_fn(a + s * tang)), tang)
    return total[space.kept_edges]
