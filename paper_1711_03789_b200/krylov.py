"""Unrestarted GMRES on the device (reference ``maxwelldd.krylov``,
/root/reference/pkg/src/maxwelldd/krylov.py:1-209).

MGS with one reorthogonalisation pass in the optional D-inner product,
complex Givens rotations, happy breakdown, left/right preconditioning: the
same recurrences, executed by csrc/gmres.cu.  Operators and preconditioners
that live on the device (:class:`DeviceCSR`, scipy/numpy matrices uploaded
once, :class:`PreconditionerState`) keep the whole loop on the GPU; an opaque
Python callable is still honoured through a host round trip per application
(interop, not a CPU compute path).
"""

from __future__ import annotations

import ctypes as C
import warnings
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _lib
from .linalg import DeviceCSR, as_device_csr, raise_for

__all__ = ["KrylovConfig", "KrylovReport", "gmres"]


_last_drift = None


@dataclass(frozen=True)
class KrylovConfig:
    """Reference krylov.py:25-43 (+ ``check_orthogonality``, default on as in the reference).

    ``orthogonalization`` (extension, not in the reference): ``"mgs"`` — the
    reference's modified Gram-Schmidt with one reorthogonalisation pass
    (krylov.py:137-143), the default — or ``"cgs2"``: classical Gram-Schmidt
    with one reorthogonalisation pass, three reductions per iteration whatever
    the basis size.  With a sharded preconditioner (:mod:`.distributed`)
    ``"cgs2"`` also shards the Krylov vectors over the ranks by row blocks.
    Unweighted inner products only.
    """

    tol: float = 1e-6
    maxit: int = 200
    weight: object = None
    side: str = "right"
    initial_guess: str = "zero"
    seed: int = 0
    keep_basis: bool = False
    check_orthogonality: bool = True
    orthogonalization: str = "mgs"

    def __post_init__(self):
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if self.maxit < 1:
            raise ValueError("maxit must be >= 1")
        if self.side not in ("left", "right"):
            raise ValueError(f"side must be 'left' or 'right', got {self.side!r}")
        if self.initial_guess not in ("zero", "random"):
            raise ValueError(f"unknown initial guess {self.initial_guess!r}")
        if self.orthogonalization not in ("mgs", "cgs2"):
            raise ValueError(f"orthogonalization must be 'mgs' or 'cgs2', got {self.orthogonalization!r}")


@dataclass
class KrylovReport:
    """Reference krylov.py:46-55."""

    x: np.ndarray
    residual_history: np.ndarray
    iterations: int
    converged: bool
    gmres_time_s: float
    seed: int
    ortho_warning: bool = False
    basis: np.ndarray | None = None


def _device_prec(precond):
    from .precond import PreconditionerState

    if isinstance(precond, PreconditionerState):
        return precond
    owner = getattr(precond, "__self__", None)
    if isinstance(owner, PreconditionerState) and getattr(precond, "__func__", None) is PreconditionerState.apply:
        return owner
    return None


def _is_identity(m, n) -> bool:
    """An exact identity weight: the reference's D @ w is then bitwise w
    (krylov.py:80-81), so the unweighted path is bitwise-equivalent."""
    if isinstance(m, DeviceCSR):
        m = m.to_scipy()
    if sp.issparse(m):
        c = m.tocsr()
        c.sum_duplicates()
        return (c.shape == (n, n) and c.nnz == n and np.array_equal(c.indices, np.arange(n))
                and np.array_equal(c.indptr, np.arange(n + 1)) and np.all(c.data == 1.0))
    a = np.asarray(m)
    return a.shape == (n, n) and np.array_equal(a, np.eye(n))


def _is_matrix(op) -> bool:
    return isinstance(op, (DeviceCSR, np.ndarray)) or sp.issparse(op)


class _HostOp:
    """ctypes callback wrapping a Python callable; exceptions are re-raised after the call."""

    def __init__(self, fn):
        self.fn = fn
        self.error = None
        self.cb = _lib.HOST_OP(self._call)

    def _call(self, user, n, pin, pout):
        try:
            xin = np.ctypeslib.as_array(C.cast(pin, C.POINTER(C.c_double)), shape=(2 * n,)).view(np.complex128)
            y = np.asarray(self.fn(xin.copy()), dtype=np.complex128).reshape(-1)
            if y.shape[0] != n:
                raise ValueError(f"operator returned length {y.shape[0]}, expected {n}")
            out = np.ctypeslib.as_array(C.cast(pout, C.POINTER(C.c_double)), shape=(2 * n,)).view(np.complex128)
            out[:] = y
            return 0
        except BaseException as e:  # noqa: BLE001 - re-raised by gmres()
            self.error = e
            return 1


def gmres(operator, rhs, precond=None, config: KrylovConfig | None = None, *, out=None) -> KrylovReport:
    """Solve ``operator x = rhs`` by (weighted) GMRES (reference krylov.py:64-209).

    ``rhs`` may also be a device-resident :class:`_lib.DeviceBuffer` (then
    ``out`` must be one too and ``report.x`` is ``out``): the benchmark's
    HBM-resident path, with no host<->device copies of the vectors.  With a
    host ``rhs``, ``out`` may be a caller-owned complex128 array (e.g. pinned
    memory) that receives the solution (then ``report.x`` is ``out``).
    """
    cfg = config if config is not None else KrylovConfig()
    dio = isinstance(rhs, _lib.DeviceBuffer)
    if dio:
        if not isinstance(out, _lib.DeviceBuffer):
            raise ValueError("device-resident rhs needs a device-resident `out`")
        n = rhs.nbytes // 16
        if cfg.initial_guess != "zero":
            raise ValueError("device-resident solve supports initial_guess='zero' only")
        b = None
    else:
        b = np.ascontiguousarray(np.asarray(rhs, dtype=complex).reshape(-1))
        n = b.shape[0]
    ctx = _lib.get_context()
    keep = []
    ops = _lib.mdd_gmres_ops()
    if _is_matrix(operator):
        A = as_device_csr(operator, force_complex=False)
        if A.shape != (n, n):
            raise ValueError(f"dimension mismatch: operator is {A.shape}, rhs has {n}")
        keep.append(A)
        ops.A = A.handle
    elif callable(operator):
        h = _HostOp(operator)
        keep.append(h)
        ops.a_fn = h.cb
    else:
        raise TypeError("operator must be a matrix or a callable")
    host_ops = [k for k in keep if isinstance(k, _HostOp)]
    if precond is not None:
        P = _device_prec(precond)
        if P is not None:
            if P.ndof != n:
                raise ValueError(f"preconditioner has size {P.ndof}, rhs has {n}")
            ops.P = P.handle
            keep.append(P)
        elif _is_matrix(precond):
            Mm = as_device_csr(precond)
            keep.append(Mm)
            ops.Mcsr = Mm.handle
        elif callable(precond):
            h = _HostOp(precond)
            keep.append(h)
            host_ops.append(h)
            ops.m_fn = h.cb
        else:
            raise TypeError("precond must be a matrix, a PreconditionerState or a callable")
    if cfg.weight is not None and not _is_identity(cfg.weight, n):
        D = as_device_csr(cfg.weight)
        keep.append(D)
        ops.D = D.handle

    rng = np.random.default_rng(cfg.seed)
    x0 = None
    if cfg.initial_guess == "random":
        x0 = np.ascontiguousarray(rng.random(n) + 1j * rng.random(n))

    c = _lib.mdd_gmres_cfg()
    c.tol = float(cfg.tol)
    c.maxit = int(cfg.maxit)
    c.side = 0 if cfg.side == "right" else 1
    c.check_drift = 1 if cfg.check_orthogonality else 0
    c.keep_basis = 1 if cfg.keep_basis else 0
    c.device_io = 1 if dio else 0
    c.ortho = 1 if cfg.orthogonalization == "cgs2" else 0
    if dio:
        x = out
    elif isinstance(out, np.ndarray):
        # caller-owned host solution buffer (e.g. pinned memory for the end-to-end timing)
        if out.shape != (n,) or out.dtype != np.complex128 or not out.flags.c_contiguous:
            raise ValueError("host `out` must be a contiguous complex128 array of the rhs length")
        x = out
    else:
        x = np.empty(n, dtype=np.complex128)
    hist = np.empty(cfg.maxit + 1, dtype=np.float64)
    drift = np.full(cfg.maxit + 1, np.nan)
    basis = np.empty((cfg.maxit + 1, n), dtype=np.complex128) if cfg.keep_basis else None
    its, conv, secs = C.c_int32(), C.c_int32(), C.c_double()
    zp = (lambda buf: C.cast(buf.ptr, C.POINTER(_lib.mdd_complex))) if dio else _lib.zptr
    try:
        _lib.check(
            _lib.lib.mdd_gmres(
                ctx.handle, C.byref(ops), n, zp(rhs if dio else b),
                _lib.zptr(x0) if x0 is not None else C.POINTER(_lib.mdd_complex)(),
                C.byref(c), zp(x), _lib.ptr(hist, C.c_double), _lib.ptr(drift, C.c_double),
                _lib.zptr(basis) if basis is not None else C.POINTER(_lib.mdd_complex)(),
                C.byref(its), C.byref(conv), C.byref(secs),
            )
        )
    except _lib.MddError as e:
        for h in host_ops:
            if h.error is not None:
                raise h.error
        raise_for(e)
    m = its.value
    history = hist[: m + 1].copy() if m > 0 else np.array([0.0])
    global _last_drift
    _last_drift = drift[: m + 1].copy()  # per-step drift values of the last solve (tests, diagnostics)
    ortho = False
    for step in range(1, m + 1):
        dv = drift[step]
        if np.isfinite(dv) and dv > 1e-8:
            ortho = True
            warnings.warn(f"Arnoldi orthogonality drift {dv:.2e} at step {step}", RuntimeWarning, stacklevel=2)
    kept_basis = None
    if basis is not None and m > 0:
        nb = m if conv.value == 2 else m + 1  # no new vector after a happy breakdown
        kept_basis = basis[:nb].T.copy()
    return KrylovReport(
        x=x,
        residual_history=history,
        iterations=m,
        converged=bool(conv.value),
        gmres_time_s=float(secs.value),
        seed=cfg.seed,
        ortho_warning=ortho,
        basis=kept_basis,
    )
