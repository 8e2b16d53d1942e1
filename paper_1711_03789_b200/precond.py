"""Overlapping Schwarz preconditioners (AS / RAS / ImpRAS, one or two levels).

Public surface of reference ``maxwelldd.precond`` (/root/reference/pkg/src/
maxwelldd/precond.py:1-257).  ``setup`` assembles the shifted system at
``xi_prec`` on the GPU (precond.py:155-159), then builds and numerically
factorises every local block and the coarse block on the device (batched
multifrontal elimination over a geometric nested-dissection ordering, see
csrc/frontal.h).  ``apply`` is a fixed linear map evaluated entirely on the
device; ``gmres`` recognises a :class:`PreconditionerState` (or its bound
``apply``) and keeps the whole Krylov loop on the device.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _lib
from .decomp import Decomposition, build_pou, impedance_dof_sets, subdomain_boundary_faces
from .fem import Coefficients, EdgeSpace, SystemBundle, assemble
from .linalg import DEFAULT_LU_CAP, DeviceCSR, as_device_csr, raise_for

__all__ = [
    "assemble_local",
    "PreconditionerSpec",
    "PreconditionerState",
    "setup",
]

FAMILIES = ("as", "ras", "impras")
CORRECTIONS = ("additive", "hybrid", "adef1")
_FAM = {"as": 0, "ras": 1, "impras": 2}
_CORR = {"additive": 0, "hybrid": 1, "adef1": 2}


@dataclass(frozen=True)
class PreconditionerSpec:
    """Reference precond.py:46-79."""

    family: str = "as"
    levels: str = "one"
    coarse_correction: str = "additive"
    xi_prec: float = 0.0
    side: str = "right"
    hybrid_matrix: str = "prob"

    def __post_init__(self):
        if self.family not in FAMILIES:
            raise ValueError(f"unknown family {self.family!r}")
        if self.levels not in ("one", "two"):
            raise ValueError(f"levels must be 'one' or 'two', got {self.levels!r}")
        if self.coarse_correction not in CORRECTIONS:
            raise ValueError(f"unknown coarse correction {self.coarse_correction!r}")
        if self.side not in ("left", "right"):
            raise ValueError(f"side must be 'left' or 'right', got {self.side!r}")
        if self.hybrid_matrix not in ("prob", "prec"):
            raise ValueError("hybrid_matrix must be 'prob' or 'prec'")

    def label(self) -> str:
        base = {"as": "AS", "ras": "RAS", "impras": "ImpRAS"}[self.family]
        if self.levels == "one":
            return f"{base}-1"
        return base + {"additive": "2", "hybrid": "-H", "adef1": "-ADEF1"}[self.coarse_correction]


def _local_kind(spec: PreconditionerSpec) -> str:
    return "pec" if spec.family in ("as", "ras") else "impedance"


class _Factors:
    """Owner of the device factor storage (``mdd_prec`` core); shared by variants."""

    def __init__(self, handle, ctx):
        self.handle = handle
        self.ctx = ctx

    def stats(self) -> dict:
        out = (C.c_double * 8)()
        _lib.check(_lib.lib.mdd_prec_stats(self.handle, out))
        keys = ("n_fronts", "max_front", "factor_entries", "factor_flops", "factor_ms", "levels",
                "sum_local_dofs", "coarse_n")
        d = dict(zip(keys, list(out)))
        fl = (C.c_double * 3)()
        _lib.check(_lib.lib.mdd_prec_flop_counts(self.handle, fl))
        d["lu_flops"], d["executed_flops"] = fl[1], fl[2]
        return d

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            _lib.lib.mdd_prec_destroy(h)
            self.handle = None


def _concat(sets, dtype=np.int64):
    ptr = np.zeros(len(sets) + 1, dtype=np.int64)
    ptr[1:] = np.cumsum([len(s) for s in sets])
    flat = np.concatenate([np.asarray(s, dtype=dtype) for s in sets]) if sets else np.zeros(0, dtype)
    return ptr, np.ascontiguousarray(flat, dtype=dtype)


class PreconditionerState:
    """Factorised Schwarz preconditioner; ``apply`` is a fixed linear map (reference precond.py:147-247)."""

    def __init__(self, problem: SystemBundle, decomp: Decomposition, spec: PreconditionerSpec,
                 lu_cap=DEFAULT_LU_CAP, leaf_size: int = 0, shard=None, _partial_cover: bool = False):
        """``shard`` (a :class:`distributed.Shard`) restricts the local solves to a
        subset of the subdomains and attaches the communicator whose allreduce
        completes the one-level sum; the coarse space stays replicated."""
        self.spec = spec
        self.shard = shard
        self.decomp = decomp
        self.ndof = problem.space.ndof
        space = problem.space
        prec_coeffs = problem.coefficients.with_xi(spec.xi_prec)
        self._prec_coeffs = prec_coeffs

        t0 = time.perf_counter()
        if getattr(space, "order", 1) == 2 and spec.family == "impras":
            raise ValueError("impras local problems are not available for order-2 spaces")
        if _local_kind(spec) == "pec":
            self.dof_sets = decomp.dofs
            self.pou_weights = decomp.pou
        else:
            self.dof_sets = impedance_dof_sets(space, decomp.elements)
            # _partial_cover: a single-subdomain state built by assemble_local (no PoU needed)
            self.pou_weights = ([np.ones(len(d)) for d in self.dof_sets] if _partial_cover
                                else build_pou(self.dof_sets, self.ndof))
        self._elements = decomp.elements
        if shard is not None:
            # PoU weights are global (computed over every subdomain) before the cut
            sel = [int(i) for i in shard.subdomains]
            self.dof_sets = [self.dof_sets[i] for i in sel]
            self.pou_weights = [self.pou_weights[i] for i in sel]
            self._elements = [decomp.elements[i] for i in sel]
        # A_prec (reference precond.py:150-152).  A rank of a sharded solve assembles only the cells
        # that touch the rows it needs (its subdomains' unknowns and the columns of its owned rows)
        self.assembly_rows = None
        if shard is not None and shard.nranks > 1 and getattr(space, "order", 1) == 1:
            from .distributed import needed_rows, row_block

            self.assembly_rows = needed_rows(space, self.dof_sets, *row_block(self.ndof, shard.nranks, shard.rank))
        t_asm = time.perf_counter()
        prec = assemble(space, prec_coeffs, rows=self.assembly_rows)
        t_asm = time.perf_counter() - t_asm  # not part of setup_time_s (reference precond.py:155-161)
        self.A_prec = prec.A
        self._A_prob = as_device_csr(problem.A, force_complex=True)
        self.A_corr = self._A_prob if spec.hybrid_matrix == "prob" else prec.A
        self.R0 = None
        if spec.levels == "two":
            if decomp.coarse is None:
                raise ValueError("two-level preconditioner needs a coarse link")
            self.R0 = decomp.coarse.R0
        handle = self._create(problem, decomp, spec, prec_coeffs, lu_cap, leaf_size)
        self.factors = _Factors(handle, prec.A._ctx)
        self._h = handle
        self.coarse_lu = self.factors if spec.levels == "two" else None
        if shard is not None and shard.comm is not None:
            _lib.check(_lib.lib.mdd_prec_set_comm(handle, shard.comm.handle))
            if shard.comm.nranks > 1 or shard.comm.is_nccl:
                self._set_halo(shard)
        self._check_static_pivoting(prec_coeffs, spec)
        self.setup_time_s = time.perf_counter() - t0 - t_asm

    #: pivot ratio below which a factor of a problem WITHOUT absorption is refused
    NO_ABSORPTION_PIVOT_TOL = 1e-10

    def _check_static_pivoting(self, prec_coeffs, spec):
        """The device factorisation pivots statically (no row exchanges).  That is backed by
        the paper's Lemma 2.5 whenever the preconditioning problem has absorption (xi_prec != 0
        or sigma > 0 somewhere) or impedance terms (impras local problems, impedance global
        boundary): every leading minor is then nonsingular and the minors are well behaved.
        Without any of these the blocks are real symmetric INDEFINITE once k^2 exceeds a
        subdomain's first Dirichlet eigenvalue; the reference's LAPACK LU pivots its way
        through such blocks (linalg.py:92), a static order need not.  In that case the factor
        is accepted only if no pivot came close to cancelling (ratio >= 1e-10, i.e. at most
        ~1e-6 of accuracy lost); otherwise a SingularMatrixError says why."""
        sig = np.asarray(prec_coeffs.sigma)
        absorbing = prec_coeffs.xi != 0.0 or bool(np.any(sig > 0.0))
        impedance = spec.family == "impras" or getattr(self.decomp.space, "bc_kind", "pec") == "impedance"
        self.static_pivoting_backed = bool(absorbing or impedance)
        if self.static_pivoting_backed:
            return
        a, b = C.c_double(), C.c_double()
        _lib.check(_lib.lib.mdd_prec_pivot_ratio(self._h, C.byref(a), C.byref(b)))
        self.pivot_ratio = (a.value, b.value)
        from .linalg import SingularMatrixError

        for what, r in (("subdomain blocks", a.value), ("coarse space", b.value)):
            if not r >= self.NO_ABSORPTION_PIVOT_TOL:
                raise SingularMatrixError(
                    f"{what}: pivot ratio {r:.2e} below {self.NO_ABSORPTION_PIVOT_TOL:.0e} in a problem without "
                    "absorption (xi_prec = 0, sigma = 0, PEC local problems): the blocks are real symmetric "
                    "indefinite and the device factorisation does not exchange rows; use a nonzero xi_prec or "
                    "impedance local problems")

    def _set_halo(self, shard):
        """Row ranges of the sharded data plane (libmdd ``mdd_prec_set_halo``): this rank's
        needed rows are its subdomains' unknowns and the columns of its rows of A (libmdd
        restricts R0 to this rank's owned columns for the coarse restriction)."""
        from .distributed import needed_rows, row_block

        lo, hi = row_block(self.ndof, shard.nranks, shard.rank)
        need_lo, need_hi = needed_rows(self.decomp.space, self.dof_sets, lo, hi)
        _lib.check(_lib.lib.mdd_prec_set_halo(self._h, int(need_lo), int(need_hi)))
        self.row_ranges = {"own": (lo, hi), "need": (int(need_lo), int(need_hi))}

    # ------------------------------------------------------------- setup
    def _create(self, problem, decomp, spec, prec_coeffs, lu_cap, leaf_size):
        space = problem.space
        dev = space.device()
        keep = []
        d = _lib.mdd_prec_desc()
        d.family = _FAM[spec.family]
        d.levels = 2 if spec.levels == "two" else 1
        d.correction = _CORR[spec.coarse_correction]
        d.lu_cap = int(lu_cap) if lu_cap is not None else 0
        d.leaf_size = int(leaf_size)
        d.A_prec = self.A_prec.handle
        d.A_corr = self.A_corr.handle
        d.nsub = len(self.dof_sets)
        sptr, sdofs = _concat(self.dof_sets)
        pou_flat = np.ascontiguousarray(np.concatenate(self.pou_weights), dtype=np.float64) \
            if len(self.pou_weights) else np.zeros(0)
        keep += [sptr, sdofs, pou_flat]
        d.sub_ptr = _lib.ptr(sptr, C.c_int64)
        d.sub_dofs = _lib.ptr(sdofs, C.c_int64)
        d.sub_pou = _lib.ptr(pou_flat, C.c_double)
        if getattr(space, "order", 1) == 2:
            # sixth-cell DoF positions; the Whitney companion space carries the
            # mesh for the coarse Galerkin product (R0 lives on the Whitney DoFs)
            xyz = space.dof_coords()
            d.dof_grid = 6
            p1dev = space.lowest_order().device()
            keep.append(p1dev)
            d.space = p1dev.handle
        else:
            xyz = space.dof_half_coords()
            d.dof_grid = 2
            d.space = dev.handle
        keep.append(xyz)
        d.dof_xyz = _lib.ptr(xyz, C.c_int32)
        cc, hold = prec_coeffs.to_c(space.mesh.n_tets)
        keep += [cc, hold]
        d.prec_coeffs = C.pointer(cc)
        if spec.family == "impras":
            tptr, tets = _concat(self._elements)
            bfs = [subdomain_boundary_faces(space.mesh, e) for e in self._elements]
            fptr = np.zeros(len(bfs) + 1, dtype=np.int64)
            fptr[1:] = np.cumsum([len(b) for b in bfs])
            fl = np.ascontiguousarray(np.concatenate(bfs) if bfs else np.zeros((0, 3)), dtype=np.int64)
            keep += [tptr, tets, fptr, fl]
            d.sub_tet_ptr = _lib.ptr(tptr, C.c_int64)
            d.sub_tets = _lib.ptr(tets, C.c_int64)
            d.sub_bface_ptr = _lib.ptr(fptr, C.c_int64)
            d.sub_bfaces = _lib.ptr(fl, C.c_int64)
        if spec.levels == "two":
            link = decomp.coarse
            r0 = as_device_csr(link.R0)
            cdev = link.space.device()
            cxyz = link.space.dof_half_coords()
            keep += [r0, cdev, cxyz]
            self._r0_dev = r0
            self._coarse_dev = cdev
            d.R0 = r0.handle
            d.coarse_space = cdev.handle
            if link.tet_map is not None:  # nested: element-wise Galerkin product
                tmap = np.ascontiguousarray(link.tet_map, dtype=np.int64)
                keep.append(tmap)
                d.tet_map = _lib.ptr(tmap, C.c_int64)
            # else (non-nested coarse mesh): tet_map stays NULL -> generic R0 A R0^T plan
            d.coarse_dof_xyz = _lib.ptr(cxyz, C.c_int32)
            if space.bc_kind == "impedance":
                gb = np.ascontiguousarray(space.mesh.boundary_faces, dtype=np.int64)
                keep.append(gb)
                d.nbf_global = len(gb)
                d.bfaces_global = _lib.ptr(gb, C.c_int64)
        self._space_dev = dev
        h = C.c_void_p()
        fctx = C.c_int32(-2)
        try:
            _lib.check(_lib.lib.mdd_prec_create(dev.ctx.handle, C.byref(d), C.byref(h), C.byref(fctx)))
        except _lib.MddError as e:
            raise_for(e)
        del keep
        return h

    def variant(self, spec: PreconditionerSpec) -> "PreconditionerState":
        """View sharing all factors (reference precond.py:195-213)."""
        if _local_kind(spec) != _local_kind(self.spec):
            raise ValueError("variant would need different local factorizations")
        if spec.xi_prec != self.spec.xi_prec:
            raise ValueError("variant would need factors at a different absorption")
        if spec.levels == "two" and self.coarse_lu is None:
            raise ValueError("variant needs a coarse factor the state does not hold")
        twin = object.__new__(PreconditionerState)
        twin.__dict__.update(self.__dict__)
        twin.spec = spec
        if spec.hybrid_matrix != self.spec.hybrid_matrix:
            twin.A_corr = self._A_prob if spec.hybrid_matrix == "prob" else self.A_prec
        h = C.c_void_p()
        _lib.check(
            _lib.lib.mdd_prec_variant(
                self._h, _FAM[spec.family], 2 if spec.levels == "two" else 1,
                _CORR[spec.coarse_correction], twin.A_corr.handle, C.byref(h),
            )
        )
        twin._h = h
        twin._variant_owner = _Factors(h, self.factors.ctx)
        return twin

    # ------------------------------------------------------- linear map
    @property
    def handle(self):
        return self._h

    def apply(self, v: np.ndarray) -> np.ndarray:
        v = np.asarray(v)
        if v.shape[0] != self.ndof:
            raise ValueError(f"vector has length {v.shape[0]}, expected {self.ndof}")
        x = np.ascontiguousarray(v, dtype=np.complex128)
        out = np.empty(self.ndof, dtype=np.complex128)
        _lib.check(_lib.lib.mdd_prec_apply(self._h, _lib.zptr(x), _lib.zptr(out)))
        return out

    __call__ = apply

    def coarse_solve(self, v: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(v, dtype=np.complex128)
        out = np.empty(self.ndof, dtype=np.complex128)
        _lib.check(_lib.lib.mdd_prec_coarse_apply(self._h, _lib.zptr(x), _lib.zptr(out)))
        return out

    def refactor(self, A_prec: DeviceCSR, prec_coeffs: Coefficients | None = None) -> None:
        """Numeric refactorisation for new values on the same pattern (benchmark step)."""
        co = prec_coeffs or self._prec_coeffs
        cc, hold = co.to_c(self.decomp.space.mesh.n_tets)
        try:
            _lib.check(_lib.lib.mdd_prec_refactor(self._h, A_prec.handle, C.byref(cc)))
        except _lib.MddError as e:
            raise_for(e)
        del hold

    def stats(self) -> dict:
        return self.factors.stats()


def assemble_local(space: EdgeSpace, coeffs: Coefficients, elems: np.ndarray, local_bc: str = "pec"):
    """System matrix on a subdomain submesh: ``(matrix, global_dofs)`` (reference precond.py:82-139).

    ``local_bc="pec"``: the unknowns with zero trace on the internal boundary; every tet around
    such an edge lies in the subdomain, so the matrix is the minor of the device-assembled
    global matrix on those unknowns (the reference's own test_decomp.py:240-253 checks that
    identity).  ``local_bc="impedance"``: all kept unknowns of the subdomain tets, element
    scatter over the subdomain tets plus the impedance mass over the subdomain boundary faces,
    assembled on the device exactly as the impras preconditioner does (csrc/precond.cu
    k_local_cells / k_local_faces) and read back through ``mdd_prec_local_matrix``."""
    from .decomp import Decomposition, subdomain_dof_sets
    from .fem import assemble as _assemble

    elems = np.ascontiguousarray(elems, dtype=np.int64)
    if local_bc == "pec":
        gdofs = subdomain_dof_sets(space, [elems])[0]
        a = _assemble(space, coeffs).A.to_scipy().tocsr()
        m = a[gdofs][:, gdofs].tocsr()
        m.sort_indices()
        return m, gdofs
    if local_bc != "impedance":
        raise ValueError(f"unknown local boundary condition {local_bc!r}")
    gdofs = impedance_dof_sets(space, [elems])[0]
    one = Decomposition(space=space, elements=[elems], dofs=[gdofs], pou=[np.ones(len(gdofs))], overlap_layers=1,
                        p_axis=1, H_sub=float(np.sqrt(3.0)))
    prob = _assemble(space, coeffs)
    st = PreconditionerState(prob, one, PreconditionerSpec("impras", "one", xi_prec=coeffs.xi), lu_cap=None,
                             _partial_cover=True)
    n, nnz = C.c_int64(), C.c_int64()
    _lib.check(_lib.lib.mdd_prec_local_matrix_size(st._h, 0, C.byref(n), C.byref(nnz)))
    rp = np.empty(n.value + 1, dtype=np.int32)
    cl = np.empty(max(nnz.value, 1), dtype=np.int32)
    vals = np.empty(max(nnz.value, 1), dtype=np.complex128)
    _lib.check(_lib.lib.mdd_prec_local_matrix(st._h, 0, _lib.ptr(rp, C.c_int32), _lib.ptr(cl, C.c_int32),
                                             vals.ctypes.data_as(C.c_void_p)))
    m = sp.csr_matrix((vals[: nnz.value], cl[: nnz.value], rp), shape=(n.value, n.value))
    m.sort_indices()
    return m, gdofs


def setup(problem: SystemBundle, decomp: Decomposition, spec: PreconditionerSpec,
          lu_cap=DEFAULT_LU_CAP) -> PreconditionerState:
    """Factorise all local (and coarse) blocks at ``spec.xi_prec`` (reference precond.py:250-257)."""
    return PreconditionerState(problem, decomp, spec, lu_cap=lu_cap)
