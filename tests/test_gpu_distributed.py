"""Sharded preconditioner on one GPU: shard partial sums and the NCCL path.

Multi-rank runs need several GPUs (one process per GPU); on the single test
GPU these check (a) that per-shard one-level applications sum to the full
application, (b) that a one-rank NCCL communicator (real ncclAllReduce,
host-driven GMRES loop) reproduces the unsharded results bit for bit, and
(c) that a world-1 shard covers every subdomain.
"""

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


def _case_objects():
    from paper_1711_03789_b200 import decomp, fem, mesh

    s = fem.build_edge_space(mesh.build_cube_mesh(8), "pec")
    prob = fem.assemble(s, fem.Coefficients(k=4.0, xi=4.0), source=fem.gaussian_source)
    d = decomp.build_decomposition(s, 2, 2, coarse_space=fem.build_edge_space(mesh.build_cube_mesh(4), "pec"))
    return prob, d


@pytest.fixture(scope="module")
def case():
    return _case_objects()


@pytest.mark.parametrize("fam", ["as", "ras", "impras"])
def test_shard_partial_sums(gpu, case, fam):
    from paper_1711_03789_b200 import precond
    from paper_1711_03789_b200.distributed import Shard, shard_bounds

    prob, d = case
    spec = precond.PreconditionerSpec(fam, "one", xi_prec=4.0)
    full = precond.PreconditionerState(prob, d, spec)
    b = shard_bounds([len(x) for x in d.dofs], 3)
    parts = [precond.PreconditionerState(prob, d, spec, shard=Shard(r, 3, np.arange(b[r], b[r + 1])))
             for r in range(3)]
    v = np.random.default_rng(3).standard_normal(prob.space.ndof) * (1 - 2j)
    got = sum(p.apply(v) for p in parts)
    assert rel(got, full.apply(v)) < 1e-13


@pytest.mark.parametrize("fam,cor", [("as", "additive"), ("ras", "hybrid"), ("impras", "adef1")])
def test_one_rank_nccl_bitwise(gpu, case, fam, cor):
    from paper_1711_03789_b200 import KrylovConfig, gmres, precond
    from paper_1711_03789_b200.distributed import Communicator, setup_sharded

    prob, d = case
    spec = precond.PreconditionerSpec(fam, "two", cor, xi_prec=4.0)
    ref = precond.setup(prob, d, spec)
    comm = Communicator(force_nccl=True)
    st = setup_sharded(prob, d, spec, comm=comm)
    assert list(st.shard.subdomains) == list(range(d.n_subdomains))
    v = np.random.default_rng(5).standard_normal(prob.space.ndof) * (1 + 1j)
    assert np.array_equal(st.apply(v), ref.apply(v))
    cfg = KrylovConfig(tol=1e-8, maxit=80)
    r1 = gmres(prob.A, prob.rhs, precond=ref, config=cfg)   # device graph loop
    r2 = gmres(prob.A, prob.rhs, precond=st, config=cfg)    # host loop + ncclAllReduce
    assert r1.iterations == r2.iterations and r1.converged
    assert np.array_equal(r1.residual_history, r2.residual_history)
    assert np.array_equal(r1.x, r2.x)


@pytest.mark.parametrize("fam,cor", [("as", "additive"), ("ras", "hybrid")])
def test_one_rank_nccl_sharded_cgs2(gpu, case, fam, cor):
    """The sharded-vector CGS2 loop (ncclAllGather of each new basis vector,
    row-block SpMV, ncclAllReduce of the projections) on a one-rank NCCL
    communicator reproduces the unsharded CGS2 run bit for bit, and matches
    the MGS2 run to the north_star tolerances."""
    from paper_1711_03789_b200 import KrylovConfig, gmres, precond
    from paper_1711_03789_b200.distributed import Communicator, setup_sharded

    prob, d = case
    spec = precond.PreconditionerSpec(fam, "two", cor, xi_prec=4.0)
    ref = precond.setup(prob, d, spec)
    st = setup_sharded(prob, d, spec, comm=Communicator(force_nccl=True))
    cg = KrylovConfig(tol=1e-8, maxit=80, orthogonalization="cgs2")
    r1 = gmres(prob.A, prob.rhs, precond=ref, config=cg)
    r2 = gmres(prob.A, prob.rhs, precond=st, config=cg)
    assert r1.converged and r1.iterations == r2.iterations
    assert np.array_equal(r1.residual_history, r2.residual_history)
    assert np.array_equal(r1.x, r2.x)
    rm = gmres(prob.A, prob.rhs, precond=ref, config=KrylovConfig(tol=1e-8, maxit=80))
    assert abs(rm.iterations - r1.iterations) <= 1
    assert rel(r1.x, rm.x) <= 1e-8


@pytest.mark.parametrize("nranks,ortho,fam,cor", [
    (2, "cgs2", "as", "additive"),
    (3, "cgs2", "ras", "hybrid"),   # uneven row blocks and shards
    (2, "mgs", "impras", "adef1"),  # replicated Krylov vectors, sharded preconditioner
    (8, "cgs2", "as", "additive"),  # one subdomain per rank, as cfg0 on 8 GPUs
])
def test_loopback_ranks(gpu, case, nranks, ortho, fam, cor):
    """The multi-rank path for real on one GPU: each rank is a host thread with
    its own context and a loopback communicator (collectives = host barrier +
    device copies; no kernel waits on another rank).  Sharded applies sum to
    the unsharded one; every rank returns the same solution, and it matches
    the one-GPU solve to the north_star tolerances."""
    import threading

    from paper_1711_03789_b200 import KrylovConfig, _lib, fem, gmres, precond
    from paper_1711_03789_b200.distributed import Communicator, LoopbackGroup, setup_sharded

    prob, d = case
    spec = precond.PreconditionerSpec(fam, "two", cor, xi_prec=4.0)
    ref = precond.setup(prob, d, spec)
    cfg = KrylovConfig(tol=1e-8, maxit=80, orthogonalization=ortho)
    want = gmres(prob.A, prob.rhs, precond=ref, config=cfg)
    v = np.random.default_rng(7).standard_normal(prob.space.ndof) * (1 - 1j)
    want_apply = ref.apply(v)
    _lib.get_context().synchronize()

    group = LoopbackGroup(nranks)
    out, errors = [None] * nranks, []

    def rank_main(r):
        comm = None
        try:
            with _lib.use_context(_lib.Context(0)) as ctx:
                # device objects (spaces, matrices, factors) of this rank live on its own context
                pr, dr = _case_objects()
                comm = Communicator(ctx, loopback=(group, r))
                st = setup_sharded(pr, dr, spec, comm=comm)
                applied = st.apply(v)
                # sharded assembly: in the sharded CGS2 loop a rank multiplies its owned rows of A
                # only, so its operator holds the needed rows only (the MGS2 loop keeps replicated
                # Krylov vectors and multiplies whole vectors: it needs the whole matrix)
                assert st.assembly_rows is not None and st.assembly_rows == st.row_ranges["need"]
                A_r = fem.assemble(pr.space, pr.coefficients, rows=st.assembly_rows).A if ortho == "cgs2" else pr.A
                rep = gmres(A_r, pr.rhs, precond=st, config=cfg)
                ctx.synchronize()
                ghost = (st.row_ranges["need"][1] - st.row_ranges["need"][0]) - (st.row_ranges["own"][1] - st.row_ranges["own"][0])
                out[r] = (len(st.shard.subdomains), applied, rep, ghost)
        except Exception as exc:  # surfaced below
            errors.append((r, exc))
            if comm is not None:
                comm.abort()  # the other ranks fail fast instead of waiting at a barrier

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(nranks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=900)
    assert not errors, errors
    assert sum(o[0] for o in out) == d.n_subdomains
    if nranks > 1:  # the exchanges move row ranges, not vectors
        assert all(o[3] < prob.space.ndof for o in out), [o[3] for o in out]
    first = out[0][2]
    for _, applied, rep, _g in out:
        assert rel(applied, want_apply) < 1e-13
        assert rep.iterations == first.iterations and np.array_equal(rep.x, first.x)
        assert np.array_equal(rep.residual_history, first.residual_history)
    assert first.converged == want.converged
    assert abs(first.iterations - want.iterations) <= 1
    assert rel(first.x, want.x) <= 1e-8


@pytest.mark.parametrize("bc", ["pec", "impedance"])
def test_row_window_assembly_is_bitwise_on_its_rows(gpu, bc):
    """Sharded assembly (mdd_space_set_row_window): only the cells that touch the window are
    assembled; the window's rows equal the full assembly bit for bit (same cells, same order),
    rows far outside stay empty, and the window does not outlive the call."""
    from paper_1711_03789_b200 import fem, mesh

    s = fem.build_edge_space(mesh.build_cube_mesh(6), bc)
    rng = np.random.default_rng(1)
    co = fem.Coefficients(k=5.0, xi=2.0, eps=1 + rng.random(s.mesh.n_tets), sigma=rng.random(s.mesh.n_tets))
    full = fem.assemble(s, co)
    lo, hi = s.ndof // 3, s.ndof // 2
    part = fem.assemble(s, co, rows=(lo, hi))
    for name in ("A", "S", "M", "Dk"):
        f, p = getattr(full, name).to_scipy().tocsr(), getattr(part, name).to_scipy().tocsr()
        assert np.array_equal(f.indptr, p.indptr) and np.array_equal(f.indices, p.indices)
        a, b = f.indptr[lo], f.indptr[hi]
        assert np.array_equal(f.data[a:b], p.data[a:b]), name
    # the first rows are more than a cell layer away from the window: nothing was assembled there
    # (the impedance boundary term is added on every boundary face, window or not)
    if bc == "pec":
        Ap = part.A.to_scipy().tocsr()
        assert not Ap.data[: Ap.indptr[10]].any()
    again = fem.assemble(s, co)
    assert np.array_equal(again.A.to_scipy().data, full.A.to_scipy().data)
