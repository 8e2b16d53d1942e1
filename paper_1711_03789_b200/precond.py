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
        return dict(zip(keys, list(out)))

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
                 lu_cap=DEFAULT_LU_CAP, leaf_size: int = 0, shard=None):
        """``shard`` (a :class:`distributed.Shard`) restricts the local solves to a
        subset of the subdomains and attaches the communicator whose allreduce
        completes the one-level sum; the coarse space stays replicated."""
        self.spec = spec
        self.shard = shard
        self.decomp = decomp
        self.ndof = problem.space.ndof
        space = problem.space
        prec_coeffs = problem.coefficients.with_xi(spec.xi_prec)
        prec = assemble(space, prec_coeffs)
        self.A_prec = prec.A
        self._A_prob = as_device_csr(problem.A, force_complex=True)
        self.A_corr = self._A_prob if spec.hybrid_matrix == "prob" else prec.A
        self._prec_coeffs = prec_coeffs

        t0 = time.perf_counter()
        if getattr(space, "order", 1) == 2 and spec.family == "impras":
            raise ValueError("impras local problems are not available for order-2 spaces")
        if _local_kind(spec) == "pec":
            self.dof_sets = decomp.dofs
            self.pou_weights = decomp.pou
        else:
            self.dof_sets = impedance_dof_sets(space, decomp.elements)
            self.pou_weights = build_pou(self.dof_sets, self.ndof)
        self._elements = decomp.elements
        if shard is not None:
            # PoU weights are global (computed over every subdomain) before the cut
            sel = [int(i) for i in shard.subdomains]
            self.dof_sets = [self.dof_sets[i] for i in sel]
            self.pou_weights = [self.pou_weights[i] for i in sel]
            self._elements = [decomp.elements[i] for i in sel]
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
        self.setup_time_s = time.perf_counter() - t0

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


def setup(problem: SystemBundle, decomp: Decomposition, spec: PreconditionerSpec,
          lu_cap=DEFAULT_LU_CAP) -> PreconditionerState:
    """Factorise all local (and coarse) blocks at ``spec.xi_prec`` (reference precond.py:250-257)."""
    return PreconditionerState(problem, decomp, spec, lu_cap=lu_cap)
