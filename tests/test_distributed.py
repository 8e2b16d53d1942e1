"""Sharded (multi-GPU) preconditioner and Krylov loop: host logic on CPU with
gloo, world_size 2.

The device path (libmdd ``mdd_prec_set_comm`` + ``mdd_prec_set_halo``) completes each
rank's partial one-level sum with a neighbour overlap-sum exchange, moves only halo row
ranges before restrictions and SpMVs, and allreduces the coarse restriction; these tests
check that decomposition of the work on the oracle: the per-rank partial sums reproduce
the full one-level, additive, hybrid and ADEF1 applications (allreduced, and through the
range exchanges restated on gloo send/recv).  The sharded CGS2 GMRES
of csrc/gmres.cu (``gmres_cgs``: row blocks of ``distributed.row_block``,
allgather of each new basis vector, allreduced projections and norms) is
restated step by step on gloo and must reproduce the oracle's MGS2 solve
(iterations +-1, solution <= 1e-8).
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import mesh_dict, rel
from oracle import maxwell_oracle as O
from paper_1711_03789_b200 import decomp, fem, mesh
from paper_1711_03789_b200.distributed import (broadcast_unique_id, make_shard, needed_rows, row_block, shard_blocks,
                                               shard_bounds)


def test_shard_bounds_cover_and_balance():
    rng = np.random.default_rng(1)
    for nsub, nranks in [(64, 1), (64, 2), (64, 8), (27, 4), (8, 8), (5, 3)]:
        costs = rng.uniform(1.0, 3.0, nsub)
        b = shard_bounds(costs, nranks)
        assert b[0] == 0 and b[-1] == nsub and len(b) == nranks + 1
        assert np.all(np.diff(b) >= 1)
        loads = np.add.reduceat(costs, b[:-1])
        assert loads.max() - loads.min() <= 2 * costs.max() + 1e-12
    assert list(shard_bounds(np.ones(64), 4)) == [0, 16, 32, 48, 64]
    with pytest.raises(ValueError):
        shard_bounds(np.ones(3), 4)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    s = fem.build_edge_space(mesh.build_cube_mesh(4), "pec")
    d = decomp.build_decomposition(s, 2, 1, coarse_space=fem.build_edge_space(mesh.build_cube_mesh(2), "pec"))
    a = O.assemble(mesh_dict(s.mesh), s.edge_to_dof, s.ndof, 3.0, 9.0)["A"]
    return s, d, a


def _allreduce_z(x):
    import torch

    t = torch.from_numpy(np.ascontiguousarray(x).view(np.float64).copy())
    dist.all_reduce(t)
    return t.numpy().view(np.complex128)


def _worker(rank, world, port, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        s, d, a = _problem()
        # unique-id broadcast (stub id: NCCL is not needed on CPU)
        uid = broadcast_unique_id((lambda: bytes(range(128))) if rank == 0 else None)
        assert uid == bytes(range(128))
        sh = make_shard(d, rank, world)
        sizes = [None] * world
        dist.all_gather_object(sizes, [int(i) for i in sh.subdomains])
        flat = sorted(i for blk in sizes for i in blk)
        assert flat == list(range(d.n_subdomains)), flat
        r0 = d.coarse.R0
        a0 = (r0 @ a @ r0.T).tocsr()
        v = np.random.default_rng(7).standard_normal(s.ndof) * (1 + 0.5j)
        for fam in ("as", "ras"):
            sel = list(sh.subdomains)
            local = O.Schwarz([d.dofs[i] for i in sel], [d.pou[i] for i in sel],
                              O.minors(a, [d.dofs[i] for i in sel]), fam, "two", "additive",
                              R0=r0, A0=a0, A_corr=a, ndof=s.ndof, solver="dense")
            for cor in ("additive", "hybrid", "adef1"):
                full = O.Schwarz(d.dofs, d.pou, O.minors(a, d.dofs), fam, "two", cor, R0=r0, A0=a0,
                                 A_corr=a, ndof=s.ndof, solver="dense")
                one = lambda x: _allreduce_z(local.one_level(x))  # noqa: E731
                gv = local.coarse_solve(v)  # replicated coarse space
                if cor == "additive":
                    got = one(v) + gv
                elif cor == "adef1":
                    got = one(v - a @ gv) + gv
                else:
                    y = one(v - a @ gv)
                    got = y - local.coarse_solve(a @ y) + gv
                err = rel(got, full.apply(v))
                assert err < 1e-12, (fam, cor, err)
            assert rel(_allreduce_z(local.one_level(v)), full.one_level(v)) < 1e-12
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as e:  # report to the parent
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise


def test_gloo_two_ranks_partial_sums():
    world = 2
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


def test_row_blocks_tile_the_vector():
    for n, w in [(10, 1), (10, 3), (433720, 8), (7, 8), (64, 4)]:
        blocks = [row_block(n, w, r) for r in range(w)]
        assert blocks[0][0] == 0 and blocks[-1][1] == n
        assert all(blocks[r][1] == blocks[r + 1][0] for r in range(w - 1))
        assert all(0 <= hi - lo <= -(-n // w) for lo, hi in blocks)


def _allgather_z(xl, n, world):
    """ncclAllGather of equal-size zero-padded blocks -> the first n entries."""
    import torch

    chunk = -(-n // world)
    pad = np.zeros(chunk, dtype=np.complex128)
    pad[: len(xl)] = xl
    t = torch.from_numpy(pad.view(np.float64).copy())
    parts = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    return np.concatenate([p.numpy().view(np.complex128) for p in parts])[:n]


def _cgs2_sharded(a, b, prec, tol, maxit, rank, world):
    """Restatement of gmres_cgs (csrc/gmres.cu) on this rank's row block."""
    n = len(b)
    lo, hi = row_block(n, world, rank)
    rows = a[lo:hi]
    dots = lambda X, y: _allreduce_z(np.array([np.vdot(x, y) for x in X]))  # noqa: E731
    r = b[lo:hi].copy()
    beta = np.sqrt(_allreduce_z(np.array([np.vdot(r, r)]))[0].real)
    V = [r / beta]
    H = np.zeros((maxit + 1, maxit), dtype=complex)
    g = np.zeros(maxit + 1, dtype=complex)
    g[0] = beta
    cs, sn = np.zeros(maxit, dtype=complex), np.zeros(maxit, dtype=complex)
    hist = [1.0]
    m = 0
    for j in range(maxit):
        w = rows @ prec(_allgather_z(V[j], n, world))
        h1 = dots(V, w)
        w = w - sum(h * v for h, v in zip(h1, V))
        h2 = dots(V, w)
        w = w - sum(h * v for h, v in zip(h2, V))
        col = np.zeros(j + 2, dtype=complex)
        col[: j + 1] = h1 + h2
        col[j + 1] = np.sqrt(_allreduce_z(np.array([np.vdot(w, w)]))[0].real)
        for i in range(j):  # krylov.py:162-187
            t = cs[i] * col[i] + sn[i] * col[i + 1]
            col[i + 1] = -np.conj(sn[i]) * col[i] + cs[i] * col[i + 1]
            col[i] = t
        am1, am = abs(col[j]), abs(col[j + 1])
        den = np.hypot(am1, am)
        cs[j] = am1 / den
        sn[j] = (col[j] / am1 if am1 > 0 else 1.0) * np.conj(col[j + 1]) / den
        H[: j + 2, j] = col
        H[j, j] = cs[j] * col[j] + sn[j] * col[j + 1]
        H[j + 1, j] = 0.0
        g[j + 1] = -np.conj(sn[j]) * g[j]
        g[j] = cs[j] * g[j]
        hist.append(min(abs(g[j + 1]) / beta, hist[-1]))
        m = j + 1
        V.append(w / np.sqrt(_allreduce_z(np.array([np.vdot(w, w)]))[0].real))
        if hist[-1] <= tol:
            break
    y = np.linalg.solve(np.triu(H[:m, :m]), g[:m])
    u = sum(yi * v for yi, v in zip(y, V[:m]))
    return prec(_allgather_z(u, n, world)), m


def _cgs_worker(rank, world, port, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        s, d, a = _problem()
        r0 = d.coarse.R0
        full = O.Schwarz(d.dofs, d.pou, O.minors(a, d.dofs), "as", "two", "additive", R0=r0,
                         A0=(r0 @ a @ r0.T).tocsr(), A_corr=a, ndof=s.ndof, solver="dense")
        b = np.random.default_rng(11).standard_normal(s.ndof) * (1 - 1j)
        x, it = _cgs2_sharded(a, b, full.apply, 1e-8, 200, rank, world)
        xr, _, itr, conv = O.gmres(a, b, full, tol=1e-8, maxit=200)
        assert conv and abs(it - itr) <= 1, (it, itr)
        assert rel(x, xr) <= 1e-8, rel(x, xr)
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as e:  # report to the parent
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise


def test_gloo_two_ranks_sharded_cgs2_gmres():
    world = 2
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_cgs_worker, args=(r, world, port, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


# ------------------------------------------------------------------ halo data plane
def test_needed_rows_cover_subdomains_and_matrix_columns():
    """needed_rows: the range contains the rank's subdomain unknowns and every column of its
    rows of A (checked against the assembled pattern), and stays an x-slab: far smaller than
    the whole vector once there are several ranks."""
    s = fem.build_edge_space(mesh.build_cube_mesh(8), "pec")
    d = decomp.build_decomposition(s, 4, 1)
    a = O.assemble(mesh_dict(s.mesh), s.edge_to_dof, s.ndof, 3.0, 9.0)["A"]
    world = 4
    for rank in range(world):
        lo, hi = row_block(s.ndof, world, rank)
        sh = make_shard(d, rank, world)
        sets = [d.dofs[i] for i in sh.subdomains]
        nlo, nhi = needed_rows(s, sets, lo, hi)
        assert nlo <= lo and hi <= nhi
        cols = a[lo:hi].indices
        assert cols.min() >= nlo and cols.max() < nhi
        for dd in sets:
            assert dd.min() >= nlo and dd.max() < nhi
        assert nhi - nlo < 0.8 * s.ndof


def _send_recv_ranges(vec, rank, world, ranges):
    """ranges: list of (peer, send_slice or None, recv_slice or None); blocking, lower rank sends first."""
    import torch

    for peer, snd, rcv in ranges:
        def do_send():
            if snd is not None and snd[1] > snd[0]:
                dist.send(torch.from_numpy(vec[snd[0]: snd[1]].view(np.float64).copy()), peer)

        def do_recv():
            if rcv is not None and rcv[1] > rcv[0]:
                buf = torch.zeros(2 * (rcv[1] - rcv[0]), dtype=torch.float64)
                dist.recv(buf, peer)
                return buf.numpy().view(np.complex128)
            return None

        if rank < peer:
            do_send()
            got = do_recv()
        else:
            got = do_recv()
            do_send()
        yield peer, got


def _halo_worker(rank, world, port, errq):
    """Restatement of the device data plane (csrc/comm.cu comm_halo_gather / comm_halo_reduce,
    csrc/precond.cu prec_apply_dist) on gloo: owned row blocks, needed row ranges, neighbour
    range exchanges, owner-side overlap sums in ascending rank order, coarse restriction as a
    local product with R0[:, owned] + allreduce."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        s = fem.build_edge_space(mesh.build_cube_mesh(6), "pec")
        d = decomp.build_decomposition(s, 3, 1, coarse_space=fem.build_edge_space(mesh.build_cube_mesh(2), "pec"))
        a = O.assemble(mesh_dict(s.mesh), s.edge_to_dof, s.ndof, 3.0, 9.0)["A"]
        n = s.ndof
        sh = make_shard(d, rank, world)
        sel = list(sh.subdomains)
        sets = [d.dofs[i] for i in sel]
        own = [row_block(n, world, q) for q in range(world)]
        need = [None] * world
        dist.all_gather_object(need, needed_rows(s, sets, *own[rank]))
        lo, hi = own[rank]
        r0 = d.coarse.R0.tocsr()
        a0 = (r0 @ a @ r0.T).tocsr()
        full = O.Schwarz(d.dofs, d.pou, O.minors(a, d.dofs), "ras", "two", "hybrid", R0=r0, A0=a0, A_corr=a,
                         ndof=n, solver="dense")
        local = O.Schwarz(sets, [d.pou[i] for i in sel], O.minors(a, sets), "ras", "two", "hybrid", R0=r0, A0=a0,
                          A_corr=a, ndof=n, solver="dense")
        isect = lambda p, q: (max(p[0], q[0]), min(p[1], q[1]))  # noqa: E731

        def gather(vec):  # owned-valid -> needed-valid, in place
            plan = [(q, isect(own[rank], need[q]), isect(own[q], need[rank])) for q in range(world) if q != rank]
            for (q, got), (_, _, rcv) in zip(_send_recv_ranges(vec, rank, world, plan), plan):
                if got is not None:
                    vec[rcv[0]: rcv[1]] = got
            return vec

        def reduce_(vec):  # partial on needed rows -> complete on owned rows
            plan = [(q, isect(own[q], need[rank]), isect(own[rank], need[q])) for q in range(world) if q != rank]
            acc = np.zeros(hi - lo, dtype=complex)
            parts = {q: (got, rcv) for (q, got), (_, _, rcv) in zip(_send_recv_ranges(vec, rank, world, plan), plan)}
            for q in range(world):  # ascending rank order, own partial in its place
                if q == rank:
                    acc += vec[lo:hi]
                elif parts[q][0] is not None:
                    rcv = parts[q][1]
                    acc[rcv[0] - lo: rcv[1] - lo] += parts[q][0]
            out = np.full(n, np.nan, dtype=complex)  # only owned rows are defined afterwards
            out[lo:hi] = acc
            return out

        def coarse(vec):  # owned-valid in, owned rows out
            part = r0[:, lo:hi] @ vec[lo:hi]
            y = local.coarse.solve(_allreduce_z(part))
            out = np.full(n, np.nan, dtype=complex)
            out[lo:hi] = r0.T.tocsr()[lo:hi] @ y
            return out

        def rows_of_a(vec):  # owned-valid in -> gather -> my rows
            out = np.full(n, np.nan, dtype=complex)
            out[lo:hi] = a[lo:hi] @ np.nan_to_num(gather(vec))[:]
            return out

        def one(vec):  # needed-valid in, owned-valid out
            return reduce_(local.one_level(np.nan_to_num(vec)))

        v = np.random.default_rng(21).standard_normal(n) * (1 - 0.3j)
        vin = np.full(n, np.nan, dtype=complex)
        vin[lo:hi] = v[lo:hi]
        vin = gather(vin)  # what the Krylov loop hands to the apply
        assert not np.isnan(vin[need[rank][0]: need[rank][1]]).any()
        gv = coarse(vin)
        t = rows_of_a(gv.copy())
        t[lo:hi] = vin[lo:hi] - t[lo:hi]
        t = gather(t)
        y = one(t)
        cy = coarse(rows_of_a(y.copy()))
        got = y[lo:hi] - cy[lo:hi] + gv[lo:hi]
        want = full.apply(v)[lo:hi]
        assert rel(got, want) < 1e-12, rel(got, want)
        # the ghost rows moved per exchange are a fraction of the vector
        assert (need[rank][1] - need[rank][0]) - (hi - lo) < n
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as e:  # report to the parent
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_halo_data_plane(world):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


def test_shard_blocks_follow_the_row_blocks():
    """8^3 boxes on 8 and 4 ranks: whole x-layers of boxes per rank, on top of the owned rows;
    on 8 ranks with 2^3 boxes the layers cannot be split, so the DoF-balanced blocks are used."""
    s = fem.build_edge_space(mesh.build_cube_mesh(16), "pec")
    d = decomp.build_decomposition(s, 8, 1)
    assert list(shard_blocks(d.dofs, s.ndof, 8)) == [64 * r for r in range(9)]
    assert list(shard_blocks(d.dofs, s.ndof, 4)) == [128 * r for r in range(5)]
    for world in (4, 8):
        for rank in range(world):
            lo, hi = row_block(s.ndof, world, rank)
            nlo, nhi = needed_rows(s, [d.dofs[i] for i in make_shard(d, rank, world).subdomains], lo, hi)
            assert (nhi - nlo) <= 2.6 * (hi - lo)  # owned rows + one overlap layer either side (boxes of 2 cells)
    d2 = decomp.build_decomposition(fem.build_edge_space(mesh.build_cube_mesh(8), "pec"), 2, 1)
    b = shard_blocks(d2.dofs, d2.space.ndof, 8)
    assert list(b) == list(range(9))
