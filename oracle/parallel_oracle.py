"""CPU ORACLE (config scale) — TEST INFRASTRUCTURE ONLY.

The reference pipeline (assemble -> decomposition -> PreconditionerState ->
gmres; reference fem.py:233-279, decomp.py:304-332, precond.py:147-247,
krylov.py:64-209) at the BASELINE.json sizes, where the reference as shipped
cannot run (its dense LU needs >= 285 GB from cfg1 on).  The
ONLY departure from the reference algorithm is the local/coarse factorisation:
``DenseLU`` (linalg.py:73-101) is replaced by SuperLU on the minor permuted by
a geometric nested dissection (grid planes are exact separators of the Kuhn
mesh) with diagonal pivots.  Validated at cfg0 against the reference's own
dense-LU solve (tests/golden/cfg0.npz): same 41 iterations, x to 1e-11
(tests/test_oracle_golden.py::test_parallel_oracle_cfg0).

The subdomain blocks are independent, so they are spread over worker
processes (all host cores); each apply still sums the local solutions in the
reference's order, subdomain 0 first (precond.py:220-224), so the result does
not depend on the worker count.

Only ``tests/``, ``tests/golden/*.py`` and ``bench.py`` (``cpu_baseline`` leg
and ``--impl reference`` arm) may import this module.  It imports nothing from
the product package.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import shutil
import tempfile
import time
from multiprocessing import shared_memory

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
from scipy.linalg import blas as _blas
from threadpoolctl import threadpool_limits

from . import geometry_oracle as G
from . import maxwell_oracle as O


# ------------------------------------------------------------ ND ordering
def nd_order(xyz, leaf=96):
    """Geometric nested dissection of DOFs given their half-cell coordinates.

    A DOF lies on the grid plane x_a = c iff its half-coordinate along a is 2c
    (every tet lies inside one cell), so {x_a == 2c} separates {x_a < 2c} from
    {x_a > 2c} exactly.  Returns the elimination order (left, right, separator)."""
    xyz = np.asarray(xyz)
    out = []

    def rec(idx):
        if len(idx) <= leaf:
            out.append(idx)
            return
        p = xyz[idx]
        lo, hi = p.min(axis=0), p.max(axis=0)
        for a in np.argsort(-(hi - lo), kind="stable"):
            c = (lo[a] + hi[a]) // 2
            c -= c & 1
            for cand in (c, c + 2, c - 2):
                if lo[a] < cand < hi[a]:
                    x = p[:, a]
                    rec(idx[x < cand])
                    rec(idx[x > cand])
                    out.append(idx[x == cand])
                    return
        out.append(idx)

    rec(np.arange(len(xyz)))
    return np.concatenate(out) if out else np.zeros(0, np.int64)


class NDLU:
    """SuperLU on the ND-permuted block, diagonal pivots (stands in for DenseLU, linalg.py:73-107)."""

    def __init__(self, a, xyz):
        self.perm = nd_order(xyz)
        ap = sp.csc_matrix(sp.csr_matrix(a)[self.perm][:, self.perm], dtype=complex)
        self.f = spla.splu(ap, permc_spec="NATURAL", diag_pivot_thresh=0.0, options=dict(SymmetricMode=True))
        self.entries = int(self.f.L.nnz + self.f.U.nnz)

    def solve(self, b):
        y = self.f.solve(np.asarray(b, dtype=complex)[self.perm])
        x = np.empty_like(y)
        x[self.perm] = y
        return x


# --------------------------------------------------------------- problem
def build_problem(c, seed=0, log=None):
    """Whole problem of a workloads.CONFIGS entry from plain arrays (no product import)."""
    import workloads as W

    t0 = time.perf_counter()
    mesh = G.cube_mesh(c["N"])
    space = G.edge_space(mesh, "pec")
    coarse = G.edge_space(G.cube_mesh(c["nc"]), "pec")
    t1 = time.perf_counter()
    dec = G.decomposition(space, c["p"], c["layers"], coarse, family=c["family"])
    t2 = time.perf_counter()
    if c.get("hetero"):
        eps, sigma = W.hetero_fields(c, G.barycenters(mesh), seed)
    else:
        eps, sigma = 1.0, 0.0
    n = space["ndof"]
    A = O.assemble(mesh, space["edge_to_dof"], n, c["k"], c["xi"], eps=eps, sigma=sigma)["A"]
    t3 = time.perf_counter()
    if c["rhs"][0] == "random":
        rhs = W.random_rhs(n, seed)
    else:
        rhs = O.rhs(mesh, space["edge_to_dof"], n, O.gaussian(alpha=c["rhs"][1], direction=(0.0, 0.0, 1.0)))
    if log:
        log(f"[oracle] {c['name']}: ndof={n} mesh {t1 - t0:.1f}s decomposition {t2 - t1:.1f}s "
            f"assemble {t3 - t2:.1f}s")
    # xi_prec == xi in every BASELINE config, so A_prec is A (precond.py:155-157)
    return {"c": c, "mesh": mesh, "space": space, "coarse_space": coarse, "dec": dec, "A": A, "rhs": rhs,
            "eps": eps, "sigma": sigma, "ndof": n,
            "times": {"mesh": t1 - t0, "decomposition": t2 - t1, "assemble": t3 - t2}}


# ------------------------------------------------------------ the workers
def _load_dir(d):
    return {f[:-4]: np.load(os.path.join(d, f), mmap_mode="r") for f in os.listdir(d) if f.endswith(".npy")}


def _worker_main(conn, tmpdir, subs, meta, shm_names):
    threadpool_limits(limits=1)  # one BLAS thread per worker whatever the inherited environment says
    arr = _load_dir(tmpdir)
    n, total = meta["ndof"], meta["total"]
    A = sp.csr_matrix((arr["A_data"], arr["A_indices"], arr["A_indptr"]), shape=(n, n))
    ptr = arr["dof_ptr"]
    flat = arr["dof_flat"]
    hc = arr["half_coords"]
    shm_v = shared_memory.SharedMemory(name=shm_names[0])
    shm_u = shared_memory.SharedMemory(name=shm_names[1])
    v = np.ndarray(n, dtype=complex, buffer=shm_v.buf)
    u = np.ndarray(total, dtype=complex, buffer=shm_u.buf)
    mesh = None
    if meta["family"] == "impras":
        mesh = {k: arr["mesh_" + k] for k in ("vertices", "tets", "edges", "tet_edges", "tet_edge_signs")}
        eptr, eflat = arr["el_ptr"], arr["el_flat"]
        eps = arr["eps"] if "eps" in arr else 1.0
        sigma = arr["sigma"] if "sigma" in arr else 0.0
    factors = {}

    def factor(ell):
        d = np.asarray(flat[ptr[ell]: ptr[ell + 1]])
        if meta["family"] == "impras":
            a = O.impedance_local_matrix(mesh, arr["edge_to_dof"], arr["kept_edges"], d,
                                         np.asarray(eflat[eptr[ell]: eptr[ell + 1]]), meta["k"], meta["xi"],
                                         eps=eps, sigma=sigma)
        else:
            a = A[d][:, d]
        return NDLU(a, hc[d])

    try:
        while True:
            msg = conn.recv()
            if msg[0] == "factor":
                t0 = time.perf_counter()
                ent = 0
                kept = 0
                for ell in subs:
                    f = factor(ell)
                    ent += f.entries
                    if kept + f.entries <= meta["budget"]:  # keep while the host-memory budget lasts
                        factors[ell] = f
                        kept += f.entries
                conn.send(("ok", time.perf_counter() - t0, ent))
            elif msg[0] == "apply":
                t0 = time.perf_counter()
                for ell in subs:
                    f = factors.get(ell) or factor(ell)
                    u[ptr[ell]: ptr[ell + 1]] = f.solve(v[flat[ptr[ell]: ptr[ell + 1]]])
                conn.send(("ok", time.perf_counter() - t0, 0))
            elif msg[0] == "stop":
                break
    except Exception as exc:  # noqa: BLE001
        conn.send(("error", repr(exc), 0))
    finally:
        shm_v.close()
        shm_u.close()


class ParallelSchwarz:
    """PreconditionerState (reference precond.py:147-247) with the local solves on worker processes.

    ``subdomains`` restricts the one-level sum to a subset (used only by
    bench.py's bounded reference-arm sample).  ``resident_entries`` caps the
    factor entries kept in host memory (about 33 B each in SuperLU); blocks
    beyond the cap are re-factored inside every apply (cfg3/cfg4 factors
    exceed this container's 62 GB)."""

    def __init__(self, prob, workers=None, resident_entries=None, subdomains=None, log=None):
        c = prob["c"]
        self.c, self.n = c, prob["ndof"]
        self.family, self.corr = c["family"], c["corr"]
        dec = prob["dec"]
        self.dofs, self.pou = dec["dofs"], dec["pou"]
        self.A = prob["A"]
        self.R0 = dec["R0"]
        self.active = list(range(len(self.dofs))) if subdomains is None else list(subdomains)
        W = max(1, min(len(self.active), workers or (os.cpu_count() or 1)))
        self.workers = W
        ptr = np.zeros(len(self.dofs) + 1, dtype=np.int64)
        ptr[1:] = np.cumsum([len(d) for d in self.dofs])
        self.ptr = ptr
        space, mesh = prob["space"], prob["mesh"]
        self.tmp = tempfile.mkdtemp(prefix="mdd_oracle_")
        save = lambda k, a: np.save(os.path.join(self.tmp, k + ".npy"), np.ascontiguousarray(a))  # noqa: E731
        save("A_data", self.A.data)
        save("A_indices", self.A.indices)
        save("A_indptr", self.A.indptr)
        save("dof_ptr", ptr)
        save("dof_flat", np.concatenate(self.dofs))
        save("half_coords", G.edge_half_coords(mesh)[space["kept_edges"]])
        if self.family == "impras":
            for k in ("vertices", "tets", "edges", "tet_edges", "tet_edge_signs"):
                save("mesh_" + k, mesh[k])
            save("edge_to_dof", space["edge_to_dof"])
            save("kept_edges", space["kept_edges"])
            ep = np.zeros(len(dec["elements"]) + 1, dtype=np.int64)
            ep[1:] = np.cumsum([len(e) for e in dec["elements"]])
            save("el_ptr", ep)
            save("el_flat", np.concatenate(dec["elements"]))
            if np.ndim(prob["eps"]):
                save("eps", prob["eps"])
            if np.ndim(prob["sigma"]):
                save("sigma", prob["sigma"])
        meta = {"ndof": self.n, "total": int(ptr[-1]), "family": self.family, "k": c["k"], "xi": c["xi"],
                "budget": float("inf") if resident_entries is None else float(resident_entries) / W}
        self.shm_v = shared_memory.SharedMemory(create=True, size=16 * self.n)
        self.shm_u = shared_memory.SharedMemory(create=True, size=16 * int(ptr[-1]))
        self.v = np.ndarray(self.n, dtype=complex, buffer=self.shm_v.buf)
        self.u = np.ndarray(int(ptr[-1]), dtype=complex, buffer=self.shm_u.buf)
        # largest blocks first, dealt round-robin: balanced workers, fixed ownership
        order = sorted(self.active, key=lambda ell: -len(self.dofs[ell]))
        ctx = mp.get_context("spawn")
        saved = {k: os.environ.get(k) for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS")}
        for k in saved:
            os.environ[k] = "1"  # one BLAS thread per worker: the parallelism is the pool
        self.procs, self.conns = [], []
        try:
            for w in range(W):
                a, b = ctx.Pipe()
                p = ctx.Process(target=_worker_main, args=(b, self.tmp, order[w::W], meta,
                                                           (self.shm_v.name, self.shm_u.name)), daemon=True)
                p.start()
                self.procs.append(p)
                self.conns.append(a)
        finally:
            for k, val in saved.items():
                if val is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = val
        t0 = time.perf_counter()
        res = self._round(("factor",))
        t_sub = time.perf_counter() - t0
        self.factor_entries = sum(r[2] for r in res)
        self.coarse = None
        if self.R0 is not None:
            a0 = (self.R0 @ self.A @ self.R0.T).tocsr()  # triple_product(R0, A_prec), precond.py:189-192
            # The sparse triple product keeps a structural entry wherever two coarse supports come
            # within one fine cell of each other; the Galerkin value there is rounding noise
            # (<= 1e-16 of the largest entry: the supports share no tet).  The reference's dense LU
            # does not care; a sparse factorisation would fill in on them (cfg1: 309,080 stored
            # entries, 90,802 above 1e-14; factor 4.9 s -> 0.17 s, solution unchanged to 8e-15).
            a0.data[np.abs(a0.data) <= 1e-13 * np.abs(a0.data).max()] = 0.0
            a0.eliminate_zeros()
            cs = prob["coarse_space"]
            # SuperLU calls BLAS on small supernodes: one thread (a threaded BLAS only adds sync cost there)
            with threadpool_limits(limits=1):
                self.coarse = NDLU(a0, G.edge_half_coords(cs["mesh"])[cs["kept_edges"]])
            self.factor_entries += self.coarse.entries
        self.setup_time_s = time.perf_counter() - t0
        self.setup_split = {"subdomains_s": t_sub, "coarse_s": self.setup_time_s - t_sub,
                            "worker_factor_s": [round(r[1], 2) for r in res]}
        if log:
            log(f"[oracle] setup {self.setup_time_s:.1f}s on {W} workers (subdomain blocks {t_sub:.1f}s, coarse "
                f"{self.setup_time_s - t_sub:.1f}s), factor entries {self.factor_entries:.3e}")

    def _round(self, msg):
        for cn in self.conns:
            cn.send(msg)
        res = [cn.recv() for cn in self.conns]
        for r in res:
            if r[0] != "ok":
                raise RuntimeError(f"oracle worker failed: {r[1]}")
        return res

    # reference precond.py:217-225
    def one_level(self, v):
        self.v[:] = v
        self._round(("apply",))
        out = np.zeros(self.n, dtype=complex)
        weighted = self.family in ("ras", "impras")
        for ell in self.active:
            ul = self.u[self.ptr[ell]: self.ptr[ell + 1]]
            out[self.dofs[ell]] += self.pou[ell] * ul if weighted else ul
        return out

    # reference precond.py:227-228
    def coarse_solve(self, v):
        with threadpool_limits(limits=1):
            y = self.coarse.solve(self.R0 @ v)
        return self.R0.T @ y

    # reference precond.py:230-245
    def apply(self, v):
        v = np.asarray(v, dtype=complex)
        if self.coarse is None:
            return self.one_level(v)
        gv = self.coarse_solve(v)
        if self.corr == "additive":
            return self.one_level(v) + gv
        if self.corr == "adef1":
            return self.one_level(v - self.A @ gv) + gv
        y = self.one_level(v - self.A @ gv)
        return y - self.coarse_solve(self.A @ y) + gv

    __call__ = apply

    def close(self):
        for cn in self.conns:
            try:
                cn.send(("stop",))
            except Exception:  # noqa: BLE001
                pass
        for p in self.procs:
            p.join(timeout=10)
            if p.is_alive():
                p.terminate()
        self.procs, self.conns = [], []
        for s in (self.shm_v, self.shm_u):
            try:
                s.close()
                s.unlink()
            except Exception:  # noqa: BLE001
                pass
        shutil.rmtree(self.tmp, ignore_errors=True)

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


# ------------------------------------------------------------------ GMRES
def gmres(op, b, precond, tol=1e-6, maxit=200, max_iters=None, deadline=None, min_iters=1, log=None,
          snapshots=None):
    """Right-preconditioned MGS2 GMRES, zero initial guess, Euclidean inner product —
    the BASELINE setting of reference krylov.py:64-209, same step order as
    oracle.maxwell_oracle.gmres (pinned to reference runs) with the level-1
    work on threaded BLAS (zdotc / zaxpy) and the basis in one array.

    ``max_iters`` truncates the run; ``deadline`` (a time.perf_counter() value)
    truncates it at the first iteration boundary past that time, after at least
    ``min_iters`` iterations (bench.py's time-boxed CPU sample).  The iterate
    returned is the GMRES iterate of the iterations done.  ``snapshots`` (a dict
    with iteration numbers as keys) is filled with the GMRES iterate x_m at those
    iterations (what a run with maxit=m returns), at the cost of one apply each.
    Returns (x, history, iterations, converged, seconds-by-phase)."""
    b = np.asarray(b, dtype=complex)
    n = len(b)
    limit = maxit if max_iters is None else min(maxit, max_iters)
    beta = float(np.sqrt(np.vdot(b, b).real))
    tm = {"operator": 0.0, "precond": 0.0, "arnoldi": 0.0}
    if beta == 0.0:
        return np.zeros(n, complex), np.array([0.0]), 0, True, tm
    V = np.empty((limit + 1, n), dtype=complex)
    V[0] = b / beta
    H = np.zeros((limit + 1, limit), dtype=complex)
    cs = np.zeros(limit, dtype=complex)
    sn = np.zeros(limit, dtype=complex)
    g = np.zeros(limit + 1, dtype=complex)
    g[0] = beta
    hist = [1.0]
    conv = False
    m = 0

    def iterate(k):
        # x_k = M (V_k y_k), y_k from the rotated Hessenberg system (krylov.py:189-198)
        y = np.zeros(k, dtype=complex)
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1: k] @ y[i + 1: k]) / H[i, i]
        upd = np.zeros(n, dtype=complex)
        for i in range(k):
            upd += y[i] * V[i]
        return precond(upd)

    for m in range(1, limit + 1):
        t0 = time.perf_counter()
        z = precond(V[m - 1])
        t1 = time.perf_counter()
        w = np.ascontiguousarray(op @ z)
        t2 = time.perf_counter()
        col = np.zeros(m + 1, dtype=complex)
        for _ in range(2):
            for j in range(m):
                h = _blas.zdotc(V[j], w)
                col[j] += h
                _blas.zaxpy(V[j], w, a=-h)  # in place on w
        hl = float(np.sqrt(max(_blas.zdotc(w, w).real, 0.0)))
        col[m] = hl
        brk = hl <= 1e-13 * np.abs(col).max()
        if not brk:
            V[m] = w / hl
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
        t3 = time.perf_counter()
        tm["precond"] += t1 - t0
        tm["operator"] += t2 - t1
        tm["arnoldi"] += t3 - t2
        if log and (m % 10 == 0 or m == 1):
            log(f"[oracle] it {m}: rel.res {hist[-1]:.4e}  (precond {tm['precond']:.0f}s arnoldi {tm['arnoldi']:.0f}s)")
        if snapshots is not None and m in snapshots:
            snapshots[m] = iterate(m)
        if brk or hist[-1] <= tol:
            conv = True
            break
        if deadline is not None and m >= min_iters and time.perf_counter() > deadline:
            break
    t0 = time.perf_counter()
    x = iterate(m)
    tm["precond"] += time.perf_counter() - t0
    return x, np.array(hist), m, conv, tm
