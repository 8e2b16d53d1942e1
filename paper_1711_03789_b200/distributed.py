"""Multi-GPU sharding of the Schwarz preconditioner.

The reference runs on one process (SPEC.md:8 puts MPI out of scope); the
paper's production runs place one subdomain solve per processor
(PAPER.md:1754).  Here one process drives one GPU and:

* each rank factorises and solves a contiguous block of subdomains, balanced
  by local DoF count (:func:`shard_bounds`); subdomain ids are x-major, so a
  block is an x-slab of boxes;
* rank r owns the contiguous row block :func:`row_block` of every vector (the
  reference numbering is x-major too: an x-slab of unknowns) and needs the rows
  :func:`needed_rows` -- its subdomains' unknowns (2 overlap layers + 1) and the
  columns of its rows of A;
* the collectives of one iteration are neighbour exchanges of those row ranges
  (libmdd ``mdd_prec_set_halo``): a halo gather before the restriction and
  before the SpMV, an overlap sum (reverse halo, owner adds) after the
  prolongation, one ncclAllReduce of the ncs coarse values per coarse solve
  (the coarse factor is replicated, R0 is restricted to the owned columns),
  and three small ncclAllReduce calls for the two classical Gram-Schmidt
  projections and the norm (``orthogonalization="cgs2"``, libmdd gmres.cu
  ``gmres_cgs``).  No collective moves a whole vector inside the loop;
* ``orthogonalization="mgs"`` with a sharded preconditioner keeps the Krylov
  vectors replicated (every apply completes its output with one allgather of
  the owned blocks): a correctness path, not the fast one.

The NCCL unique id travels over the caller's ``torch.distributed`` process
group (any backend), NCCL itself is opened by libmdd with ``dlopen``.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["Communicator", "LoopbackGroup", "Shard", "shard_bounds", "shard_blocks", "make_shard", "setup_sharded",
           "row_block", "needed_rows"]


def shard_bounds(costs, nranks: int) -> np.ndarray:
    """Split ``len(costs)`` ordered subdomains into ``nranks`` contiguous blocks.

    Returns ``nranks + 1`` monotone boundaries; each block's summed cost is as
    close as possible to ``total / nranks`` (prefix-sum cut points).  Every
    rank receives at least one subdomain when there are enough of them.
    """
    costs = np.asarray(costs, dtype=np.float64)
    nsub = len(costs)
    if nranks < 1:
        raise ValueError("nranks must be >= 1")
    if nsub < nranks:
        raise ValueError(f"{nsub} subdomains cannot be shared by {nranks} ranks")
    pref = np.concatenate([[0.0], np.cumsum(costs)])
    total = pref[-1]
    b = np.zeros(nranks + 1, dtype=np.int64)
    b[-1] = nsub
    for r in range(1, nranks):
        target = total * r / nranks
        cut = int(np.searchsorted(pref, target))
        if cut > 0 and abs(pref[cut - 1] - target) <= abs(pref[min(cut, nsub)] - target):
            cut -= 1
        # keep at least one subdomain per rank on either side
        b[r] = min(max(cut, b[r - 1] + 1), nsub - (nranks - r))
    return b


def row_block(n: int, nranks: int, rank: int) -> tuple[int, int]:
    """Rows ``[lo, hi)`` of the Krylov vectors owned by ``rank`` in the sharded
    CGS2 loop: blocks of ``ceil(n / nranks)`` rows (the last one shorter), the
    layout ncclAllGather needs (equal per-rank counts, zero padding).  Mirrors
    ``gmres_cgs`` in csrc/gmres.cu."""
    if nranks < 1 or not 0 <= rank < nranks:
        raise ValueError("bad rank / world size")
    chunk = -(-n // nranks)
    lo = min(n, rank * chunk)
    return lo, min(n, lo + chunk)


def needed_rows(space, dof_sets, lo: int, hi: int) -> tuple[int, int]:
    """Rows ``[need_lo, need_hi)`` a rank must hold valid values of before it can apply its
    block of the preconditioner and its rows ``[lo, hi)`` of A: the unknowns of its subdomains
    (restriction, reference precond.py:220) and the column support of its rows (reference
    krylov.py:95-97; the columns of row i are the unknowns of the tets around edge i).  The
    reference numbering is x-major, so the set is an index range around the owned block."""
    need_lo, need_hi = lo, hi
    for d in dof_sets:
        if len(d):
            need_lo = min(need_lo, int(d[0]))
            need_hi = max(need_hi, int(d[-1]) + 1)
    if hi > lo:
        m = space.mesh
        mine = np.zeros(m.n_edges, dtype=bool)
        mine[space.kept_edges[lo:hi]] = True
        touched = mine[m.tet_edges].any(axis=1)
        cols = space.edge_to_dof[m.tet_edges[touched]]
        cols = cols[cols >= 0]
        if len(cols):
            need_lo = min(need_lo, int(cols.min()))
            need_hi = max(need_hi, int(cols.max()) + 1)
    return need_lo, need_hi


class Communicator:
    """libmdd NCCL communicator for the ranks of a ``torch.distributed`` group.

    ``force_nccl`` initialises NCCL even for a single rank (used by the tests
    to exercise the allreduce path on one GPU)."""

    def __init__(self, ctx=None, group=None, force_nccl: bool = False, loopback=None, standalone=None):
        self.ctx = ctx or _lib.get_context()
        self.is_nccl = False
        if standalone is not None:
            # (rank, nranks, unique id): ranks that found each other without torch.distributed
            self.rank, self.nranks, uid = int(standalone[0]), int(standalone[1]), bytes(standalone[2])
            h = C.c_void_p()
            _lib.check(_lib.lib.mdd_comm_create(self.ctx.handle, self.nranks, self.rank, uid, C.byref(h)))
            self.handle = h
            self.is_nccl = True
            return
        import torch.distributed as dist

        if loopback is not None:
            # (LoopbackGroup, rank): ranks are host threads sharing one GPU (tests)
            grp, rank = loopback
            self.rank, self.nranks, self._group = int(rank), grp.nranks, grp
            h = C.c_void_p()
            _lib.check(_lib.lib.mdd_comm_create_loopback(self.ctx.handle, grp.handle, self.rank, C.byref(h)))
            self.handle = h
            return
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.nranks = dist.get_world_size(group)
        else:
            self.rank, self.nranks = 0, 1
        uid = None
        if self.nranks > 1 or force_nccl:
            uid = broadcast_unique_id(_new_unique_id if self.rank == 0 else None, group)
        h = C.c_void_p()
        _lib.check(_lib.lib.mdd_comm_create(self.ctx.handle, self.nranks, self.rank, uid, C.byref(h)))
        self.handle = h
        self.is_nccl = uid is not None

    def abort(self):
        """Loopback groups: mark the group failed so the other ranks stop waiting (call from an
        ``except`` around a rank's work)."""
        _lib.lib.mdd_comm_abort(self.handle)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            _lib.lib.mdd_comm_destroy(h)
            self.handle = None


class LoopbackGroup:
    """Ranks as host threads on ONE GPU (test infrastructure, libmdd
    ``mdd_comm_loopback_group``): each thread uses its own context
    (``_lib.use_context``) and ``Communicator(loopback=(group, rank))``;
    collectives meet at a host barrier and move data with device copies, so
    the multi-rank code path (row blocks, allgather layout, partial-sum
    allreduce) runs for real without several GPUs."""

    def __init__(self, nranks: int):
        h = C.c_void_p()
        _lib.check(_lib.lib.mdd_comm_loopback_group(int(nranks), C.byref(h)))
        self.handle = h
        self.nranks = int(nranks)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            _lib.lib.mdd_comm_loopback_group_free(h)
            self.handle = None


def _new_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _lib.check(_lib.lib.mdd_comm_unique_id(buf))
    return buf.raw


def broadcast_unique_id(make_id, group=None) -> bytes:
    """Rank 0 calls ``make_id()``; the 128-byte id reaches every rank of ``group``."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return make_id()
    obj = [make_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0, group=group)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("NCCL unique id broadcast failed")
    return bytes(uid)


@dataclass(frozen=True)
class Shard:
    """The subdomains one rank owns and the communicator completing the sum."""

    rank: int
    nranks: int
    subdomains: np.ndarray
    comm: Communicator | None = None


def shard_blocks(dof_sets, ndof: int, nranks: int) -> np.ndarray:
    """Boundaries of the contiguous subdomain blocks of the ranks.

    Preferred: subdomain l goes to the rank whose owned row block (:func:`row_block`) holds
    the median unknown of I_l, so a rank's subdomains sit on top of the rows it owns and its
    needed row range (:func:`needed_rows`) exceeds them by the overlap only (cfg4 on 8 ranks:
    64 boxes = one x-layer per rank).  When that leaves a rank with less than half the
    average number of subdomains (more ranks than x-layers of boxes), fall back to blocks
    balanced by local DoF count (:func:`shard_bounds`)."""
    nsub = len(dof_sets)
    if nranks == 1:
        return np.array([0, nsub], dtype=np.int64)
    chunk = -(-ndof // nranks)
    med = np.array([d[len(d) // 2] if len(d) else 0 for d in dof_sets], dtype=np.int64)
    owner = np.minimum(med // chunk, nranks - 1)
    if np.all(np.diff(owner) >= 0):
        b = np.searchsorted(owner, np.arange(nranks + 1)).astype(np.int64)
        if np.diff(b).min() >= max(1, nsub // (2 * nranks)):
            return b
    return shard_bounds([len(d) for d in dof_sets], nranks)


def make_shard(decomp, rank: int, nranks: int, comm: Communicator | None = None) -> Shard:
    """Contiguous block of ``decomp``'s subdomains for ``rank`` (:func:`shard_blocks`)."""
    b = shard_blocks(decomp.dofs, decomp.space.ndof, nranks)
    return Shard(rank, nranks, np.arange(b[rank], b[rank + 1], dtype=np.int64), comm)


def setup_sharded(problem, decomp, spec, comm: Communicator | None = None, **kw):
    """:func:`precond.setup` over this rank's subdomains (all ranks call it)."""
    from .precond import PreconditionerState

    comm = comm or Communicator()
    shard = make_shard(decomp, comm.rank, comm.nranks, comm)
    return PreconditionerState(problem, decomp, spec, shard=shard, **kw)
