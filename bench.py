"""Benchmark: preconditioned GMRES time-to-solve on the BASELINE configs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1] [--impl mine|reference]

One *step* = one complete numeric solve on a fixed mesh + decomposition:
device assembly of the problem matrix A and of the shifted A_prec
(fem.assemble), numeric factorisation of every subdomain block, element-wise
Galerkin coarse block and its factorisation (PreconditionerState.refactor),
and right-preconditioned GMRES (tol 1e-6, maxit 200, zero initial guess).
Mesh, DOF pattern, decomposition and the nested-dissection symbolic analysis
are per-mesh setup, done once before timing (SURVEY.md §3.6's "setup" phase
is the numeric factorisation, which is timed).

value : DoFs/s = n_gpus * ndof / (device time per step), inputs resident in HBM.
e2e   : same metric through the public API with host buffers (rhs H2D and
        x D2H inside the timed region), wall clock.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs (SURVEY.md §8d for the conventions chosen where BASELINE is silent)
CONFIGS = {
    0: dict(name="cfg0", N=20, k=10.0, xi=10.0, p=2, layers=2, nc=5, family="as", corr="additive",
            rhs=("gauss", 100.0)),
    1: dict(name="cfg1", N=40, k=20.0, xi=20.0, p=4, layers=2, nc=10, family="as", corr="additive",
            rhs=("random", 0)),
    # second-order Nedelec fine space (extension: the reference has Whitney elements only),
    # lowest-order coarse space nested in its Whitney part; Gaussian source as cfg0
    2: dict(name="cfg2", N=30, k=20.0, xi=20.0, p=3, layers=1, nc=8, family="as", corr="additive",
            rhs=("gauss", 100.0), order=2),
    3: dict(name="cfg3", N=60, k=30.0, xi=math.sqrt(30.0), p=4, layers=2, nc=15, family="impras",
            corr="hybrid", rhs=("random", 0)),  # ImpHRAS: the paper's coarse combination for ImpRAS
    4: dict(name="cfg4", N=80, k=40.0, xi=0.0, p=8, layers=2, nc=20, family="as", corr="additive",
            rhs=("gauss", 400.0), hetero=True),
}
METRIC = "precond_gmres_time_to_solve"
UNIT = "DoF/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------- problem
def build_problem(c, seed=0):
    from paper_1711_03789_b200 import decomp, fem, mesh

    m = mesh.build_cube_mesh(c["N"])
    space = fem.build_edge_space(m, "pec", order=c.get("order", 1))
    nt = m.n_tets
    if c.get("hetero"):
        # eps_r per 4x4x4 block ~ U[1,4]; absorption per block ~ U[k/2, 2k] carried by
        # sigma = absorption / k, so k*sigma is the block absorption (fem.py:254)
        rng = np.random.default_rng(seed)
        blk = np.clip((m.barycenters() * 4).astype(int), 0, 3)
        bid = (blk[:, 0] * 4 + blk[:, 1]) * 4 + blk[:, 2]
        eps_b = 1.0 + 3.0 * rng.random(64)
        abs_b = c["k"] * (0.5 + 1.5 * rng.random(64))
        coeffs = fem.Coefficients(k=c["k"], xi=c["xi"], eps=eps_b[bid], sigma=abs_b[bid] / c["k"])
    else:
        coeffs = fem.Coefficients(k=c["k"], xi=c["xi"])
    if c["rhs"][0] == "random":
        rng = np.random.default_rng(seed)
        rhs = (rng.standard_normal(space.ndof) + 1j * rng.standard_normal(space.ndof)) / np.sqrt(2.0)
    else:
        rhs = fem.assemble_rhs(space, fem.GaussianSource(alpha=c["rhs"][1], direction=(0.0, 0.0, 1.0)))
    coarse = fem.build_edge_space(mesh.build_cube_mesh(c["nc"]), "pec")
    t0 = time.perf_counter()
    dec = decomp.build_decomposition(space, c["p"], c["layers"], coarse_space=coarse, allow_nonnested=True)
    t_dec = time.perf_counter() - t0
    return space, coeffs, np.ascontiguousarray(rhs), dec, t_dec


# --------------------------------------------------------------- clocks
class ClockSampler:
    """One long-lived `nvidia-smi -lms 200` process, started before the timed
    region and stopped after it (B200_PROFILING.md's clocks line): a single
    fork outside the timed region instead of one per sample."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, device):
        self.device = device
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=10)
        except Exception:  # noqa: BLE001
            self.proc.kill()
            out, _ = self.proc.communicate()
        for line in out.splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and "Active" in s[3 + i]
                          and "Not" not in s[3 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------ CPU baseline
def _cpu_block_job(args):
    """Worker: SuperLU factorisation + one solve of one subdomain block (oracle)."""
    import time as _t

    import numpy as _np
    import scipy.sparse as _sp

    from oracle import maxwell_oracle as O

    data, indices, indptr, shape = args
    a = _sp.csr_matrix((data, indices, indptr), shape=shape)
    t0 = _t.perf_counter()
    f = O._Sparse(a)
    t1 = _t.perf_counter()
    f.solve(_np.ones(shape[0], dtype=complex))
    return t1 - t0, _t.perf_counter() - t1


def cpu_sample(c, space, coeffs, rhs, dec, budget_s=12.0, workers=None):
    """Bounded oracle sample on host cores -> extrapolated time-to-solve.

    Times (a) SuperLU factorisation + solve of `workers` subdomain blocks,
    concurrently, one per process (the blocks are independent, so all host
    cores are used; scaled to all subdomains assuming perfect parallel
    speed-up, which favours the CPU), (b) one SpMV and one coarse solve,
    (c) the MGS2 Arnoldi step at two basis sizes (linear in m); then sums the
    full solve at the GPU run's iteration count.
    """
    from concurrent.futures import ProcessPoolExecutor

    from oracle import maxwell_oracle as O

    t_start = time.perf_counter()
    md = {k: getattr(space.mesh, k) for k in ("vertices", "tets", "edges", "tet_edges", "tet_edge_signs",
                                              "boundary_faces")}
    t0 = time.perf_counter()
    if getattr(space, "order", 1) == 2:
        from oracle import nedelec2_oracle as O2

        sysm = O2.assemble(space.mesh.vertices, space.mesh.tets, space.tet_dofs, space.ndof, coeffs.k, coeffs.xi,
                           eps=coeffs.eps, mu=coeffs.mu, sigma=coeffs.sigma)
    else:
        sysm = O.assemble(md, space.edge_to_dof, space.ndof, coeffs.k, coeffs.xi, eps=coeffs.eps, mu=coeffs.mu,
                          sigma=coeffs.sigma)
    t_asm = time.perf_counter() - t0
    A = sysm["A"]
    nsub = len(dec.dofs)
    P = max(1, min(nsub, workers or (os.cpu_count() or 1)))
    jobs = []
    for ell in range(P):
        a_l = A[dec.dofs[ell]][:, dec.dofs[ell]].tocsr()
        jobs.append((a_l.data, a_l.indices, a_l.indptr, a_l.shape))
    if P > 1:
        import multiprocessing as mp

        # spawn, not fork (forking after BLAS threads exist can deadlock the
        # children); one BLAS thread per worker: the parallelism is the pool
        saved = {k: os.environ.get(k) for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS")}
        for k in saved:
            os.environ[k] = "1"
        try:
            with ProcessPoolExecutor(max_workers=P, mp_context=mp.get_context("spawn")) as ex:
                res = list(ex.map(_cpu_block_job, jobs))
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
    else:
        res = [_cpu_block_job(jobs[0])]
    fac_times = [r[0] for r in res]
    solve_times = [r[1] for r in res]
    rng = np.random.default_rng(0)
    r0 = dec.coarse.R0
    t0 = time.perf_counter()
    a0 = (r0 @ A @ r0.T).tocsc()
    f0 = O._Sparse(a0)
    t_coarse_fac = time.perf_counter() - t0
    x = rng.standard_normal(space.ndof) + 1j * rng.standard_normal(space.ndof)
    t0 = time.perf_counter()
    for _ in range(3):
        A @ x
    t_spmv = (time.perf_counter() - t0) / 3
    t0 = time.perf_counter()
    r0.T @ f0.solve(r0 @ x)
    t_coarse = time.perf_counter() - t0

    def mgs(m):
        V = [rng.standard_normal(space.ndof) + 0j for _ in range(m)]
        w = x.copy()
        t = time.perf_counter()
        for _ in range(2):
            for j in range(m):
                h = np.vdot(V[j], w)
                w = w - h * V[j]
        return time.perf_counter() - t

    m1, m2 = 8, 24
    tm1, tm2 = mgs(m1), mgs(m2)
    slope = max((tm2 - tm1) / (m2 - m1), 0.0)
    return {
        "t_asm": t_asm, "t_fac_sub": float(np.mean(fac_times)), "t_solve_sub": float(np.mean(solve_times)),
        "t_coarse_fac": t_coarse_fac, "t_coarse": t_coarse, "t_spmv": t_spmv, "mgs_slope": slope,
        "mgs_icpt": max(tm1 - slope * m1, 0.0), "nsub": nsub, "n_sampled": len(fac_times), "workers": P,
        "sample_s": time.perf_counter() - t_start,
    }


def cpu_extrapolate(s, iterations):
    par = s["nsub"] / s["workers"]  # subdomain work spread over the worker processes
    t_fac = 2 * s["t_asm"] + par * s["t_fac_sub"] + s["t_coarse_fac"]
    t_apply = par * s["t_solve_sub"] + s["t_coarse"]
    t_it = (iterations + 1) * (t_apply + s["t_spmv"])
    t_arn = sum(s["mgs_icpt"] + s["mgs_slope"] * m for m in range(1, iterations + 1)) * 1.5  # + drift check
    return t_fac + t_it + t_arn


# ---------------------------------------------------------------- our arm
def run_mine(args, rank, world):
    from paper_1711_03789_b200 import _lib, fem, krylov, precond

    c = CONFIGS[args.config]
    ctx = _lib.get_context()
    t0 = time.perf_counter()
    space, coeffs, rhs, dec, t_dec = build_problem(c)
    n = space.ndof
    spec = precond.PreconditionerSpec(c["family"], "two", c["corr"], xi_prec=c["xi"])
    prob = fem.assemble(space, coeffs)
    t1 = time.perf_counter()
    if world > 1:
        # strong scaling: each rank factorises/solves its block of subdomains; the
        # one-level sum is completed by one ncclAllReduce per apply (distributed.py)
        from paper_1711_03789_b200 import distributed

        comm = distributed.Communicator(ctx)
        st = distributed.setup_sharded(prob, dec, spec, comm=comm, lu_cap=None)
    else:
        st = precond.setup(prob, dec, spec, lu_cap=None)
    t_setup = time.perf_counter() - t1
    t_prep = time.perf_counter() - t0
    stats = st.stats()
    # one GPU: the reference's MGS2 (default); sharded runs: CGS2 over row-block
    # sharded Krylov vectors (three small allreduces per iteration instead of
    # one per MGS step), validated against MGS2 in tests/test_gpu_gmres.py
    ortho = args.ortho or ("cgs2" if world > 1 else "mgs")
    kcfg = krylov.KrylovConfig(tol=1e-6, maxit=200, side="right", initial_guess="zero", orthogonalization=ortho)
    rhs_dev = _lib.DeviceBuffer(ctx, 16 * n)
    rhs_dev.upload(rhs)
    x_dev = _lib.DeviceBuffer(ctx, 16 * n)
    prec_coeffs = coeffs.with_xi(spec.xi_prec)

    def step(device_io=True):
        p = fem.assemble(space, coeffs)
        ctx.record(1)
        a_prec = fem.assemble(space, prec_coeffs).A
        ctx.record(4)
        st.refactor(a_prec, prec_coeffs)
        ctx.record(2)
        if device_io:
            rep = krylov.gmres(p.A, rhs_dev, precond=st, config=kcfg, out=x_dev)
        else:
            rep = krylov.gmres(p.A, rhs_pin, precond=st.apply, config=kcfg, out=x_pin)
        return rep

    log(f"[bench] {c['name']}: ndof={n} nsub={len(dec.dofs)} prep {t_prep:.1f}s (decomp {t_dec:.1f}s, "
        f"setup {t_setup:.1f}s) fronts={stats['n_fronts']:.0f} max_front={stats['max_front']:.0f} "
        f"factor_entries={stats['factor_entries']:.3e}")
    for _ in range(args.warmup):
        step()
    dist_barrier(world)
    ctx.synchronize()
    launches0 = ctx.kernel_launches()
    ms_steps, phases, reps = [], [], []
    host = np.zeros(4)
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        for _ in range(args.steps):
            ctx.record(0)
            rep = step()
            ctx.record(3)
            ms = ctx.elapsed_ms(0, 3)
            ms_steps.append(ms)
            phases.append((ctx.elapsed_ms(0, 1), ctx.elapsed_ms(1, 2), ctx.elapsed_ms(2, 3), ctx.elapsed_ms(4, 2)))
            host += np.array(ctx.timers()[3:7])
            reps.append(rep)
    ctx.synchronize()
    dist_barrier(world)
    launches = ctx.kernel_launches() - launches0
    # one extra instrumented step (host-driven loop with per-phase CUDA events) for the
    # per-kernel-family breakdown; not part of the timed value
    ctx.set_timing(True)
    step()
    timers = np.array(ctx.timers()[:3])
    ctx.set_timing(False)
    ms_step = max_over_ranks(float(np.mean(ms_steps)), world)
    # e2e through the public API with host buffers: rhs and solution in pinned host
    # memory, so the per-step H2D / D2H copies are DMA transfers
    import torch

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))  # pin through this rank's GPU context
    rhs_pin = torch.empty(n, dtype=torch.complex128, pin_memory=True).numpy()
    rhs_pin[:] = rhs
    x_pin = torch.empty(n, dtype=torch.complex128, pin_memory=True).numpy()
    e2e_t = []
    import gc

    gc.collect()
    gc.disable()  # no collector pauses inside the wall-clock region
    try:
        for _ in range(max(1, args.steps)):
            t = time.perf_counter()
            rep_e = step(device_io=False)
            e2e_t.append(time.perf_counter() - t)
    finally:
        gc.enable()
    e2e_s = max_over_ranks(float(np.mean(e2e_t)), world)
    rep = reps[-1]
    x = np.empty(n, dtype=np.complex128)
    x_dev.download(x)
    its = rep.iterations
    # roofline of the dominant kernel family
    t_op, t_prec, t_arn = timers
    h_setup, h_loop, h_final, h_graph = host / args.steps
    fe = stats["factor_entries"]
    sum_loc = stats["sum_local_dofs"]
    r0nnz = dec.coarse.R0.nnz
    b_prec = 16 * fe + 40 * sum_loc + 40 * r0nnz + 48 * n
    # two MGS passes stream V_0..V_{m-1} once each; the drift rides along the first pass; + w in, V_m out
    b_arn = sum((32 * m + 64) * n for m in range(1, its + 1))
    b_spmv = (20 * prob.A.nnz + 36 * n) * its
    peak = read_peaks()
    # kernel families per GMRES iteration: one preconditioner apply, one SpMV,
    # one Arnoldi launch (bytes: SURVEY.md §8d formulas)
    cands = {
        "precond_apply": (b_prec, t_prec / its, "k_solve_tma fwd/bwd levels + k_scatter_owner + coarse R0/R0^T "
                                                  "SpMV and coarse solve, one apply"),
        "k_arnoldi": (b_arn / its, t_arn / its, "one k_arnoldi launch (MGS2 + drift + Givens), mean over the "
                                                 "solve's iterations"),
        "k_spmv": (b_spmv / its, t_op / its, "one complex CSR SpMV"),
    }
    dom = max(cands, key=lambda k: cands[k][1])
    traffic = read_traffic(c["name"])
    roof_all = {}
    for k, (b, t, what) in cands.items():
        ach = b / (t / 1e3) / 1e9 if t > 0 else 0.0
        roof_all[k] = {"achieved": ach, "frac": ach / peak["hbm_gbs"], "ms_per_launch": t,
                       "algorithmic_bytes_per_launch": b, "ms_per_step": t * its, "launch": what,
                       "traffic": traffic.get(k)}
    fpk = read_fp64_peak()
    fac_ms = float(np.mean([p[3] for p in phases]))  # numeric refactorisation inside the timed steps
    f_ach = stats["factor_flops"] / (fac_ms / 1e3) / 1e12 if fac_ms > 0 else 0.0
    roof_factor = {"bound": "tensor", "kernel": "numeric factorisation (k_front_init, GJ sweeps k_gj_small/k_panel/"
                                                "k_update, k_gemm DMMA F_PU/Schur, k_transpose_up), subdomains + coarse",
                   "achieved": f_ach, "peak": fpk["tflops"], "unit": "TFLOP/s", "frac": f_ach / fpk["tflops"],
                   "flops": stats["factor_flops"], "ms": fac_ms, "peak_source": fpk["source"]}
    hist = rep.residual_history
    res = {
        "metric": METRIC,
        "value": n / (ms_step / 1e3),  # one solve per step, shared by all ranks
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "c128",
        "data": "synthetic (seeded; BASELINE.json configs)",
        "config": {
            "workload": f"{c['name']}: N={c['N']} ({n} DoFs), k={c['k']}, xi={c['xi']:.4g}, "
                        f"{c['p']}^3 subdomains, {c['layers']} overlap layers, coarse N={c['nc']}, "
                        f"{spec.label()}, right GMRES tol 1e-6 maxit 200",
            "ndof": n, "subdomains": len(dec.dofs), "iterations": its, "converged": bool(rep.converged),
            "final_rel_residual": float(hist[-1]),
            "parallelism": (f"subdomains sharded over {world} GPUs (NCCL allreduce per apply), coarse replicated, "
                            + ("Krylov vectors sharded by row blocks (CGS2: allgather per iteration + 3 small "
                               "allreduces)" if ortho == "cgs2" else "MGS2 GMRES replicated"))
                           if world > 1 else "single-gpu",
            "orthogonalization": ortho,
            "local_subdomains": int(len(st.dof_sets)),
            "l2": "working set (V basis, factors) >> 126 MB L2; no flush needed",
        },
        "iters_per_s": its / (ms_step / 1e3),
        "ms_steps": [round(x, 3) for x in ms_steps],
        "phases_ms": {"assemble_A": float(np.mean([p[0] for p in phases])),
                      "assemble_Aprec_factor": float(np.mean([p[1] for p in phases])),
                      "gmres": float(np.mean([p[2] for p in phases])),
                      "factor": float(np.mean([p[3] for p in phases])),
                      "gmres_spmv": t_op, "gmres_precond": t_prec, "gmres_arnoldi": t_arn,
                      "gmres_host_setup": h_setup, "gmres_host_loop": h_loop, "gmres_host_final": h_final,
                      "gmres_graph_build": h_graph},
        "setup_s": {"decomposition": t_dec, "first_setup_incl_symbolic": t_setup},
        "factor": {k: stats[k] for k in ("n_fronts", "max_front", "factor_entries", "factor_flops", "factor_ms")},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": roof_all[dom]["achieved"], "peak": peak["hbm_gbs"],
                     "unit": "GB/s", "frac": roof_all[dom]["frac"], "traffic": roof_all[dom]["traffic"],
                     "algorithmic_bytes_per_launch": roof_all[dom]["algorithmic_bytes_per_launch"],
                     "launch": roof_all[dom]["launch"], "peak_source": peak["source"],
                     "traffic_source": "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch "
                                       "(profiles/traffic.json)" if roof_all[dom]["traffic"] else None},
        "roofline_all": roof_all,
        "roofline_factor": roof_factor,
        "e2e": {"value": n / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": 16 * n,
                "s_per_step": e2e_s, "s_steps": [round(v, 4) for v in e2e_t], "iterations": rep_e.iterations},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        s = cpu_sample(c, space, coeffs, rhs, dec)
        t_cpu = cpu_extrapolate(s, its)
        res["cpu_baseline"] = {"value": n / t_cpu, "unit": UNIT, "cores": s["workers"], "kind": "port",
                               "sample": f"oracle (numpy/SuperLU) on {s['n_sampled']} of {s['nsub']} subdomain "
                                         f"factorisations+solves ({s['workers']} processes), 1 SpMV, 1 coarse "
                                         f"solve, MGS2 at m=8,24; "
                                         f"extrapolated to {its} iterations ({s['sample_s']:.1f}s sampled, "
                                         f"est. {t_cpu:.0f}s per solve)",
                               "est_s_per_solve": t_cpu}
    return res


def read_traffic(cfg_name):
    """Measured DRAM bytes per launch of each kernel family (ncu launch list of
    one bench step, tools/traffic_from_ncu.py -> profiles/traffic.json)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return d.get(cfg_name, {})
    except Exception:  # noqa: BLE001
        return {}


def read_fp64_peak():
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
        return {"tflops": float(d["fp64_tflops"]), "source": "measured DMMA peak (profiles/fp64_peak.json)"}
    except Exception:  # noqa: BLE001
        return {"tflops": 40.0, "source": "nominal B200 FP64 tensor peak (no measurement found)"}


def read_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:  # noqa: BLE001
        return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


# ---------------------------------------------------------- reference arm
def run_reference(args):
    """The reference's CPU path (the oracle port: the reference is pure Python and
    cannot travel to the GPU box) on a bounded sample of the same workload."""
    c = CONFIGS[args.config]
    space, coeffs, rhs, dec, _ = build_problem(c)
    n = space.ndof
    its = 200 if args.config == 1 else 60
    vals = []
    workers = 1
    for i in range(args.warmup + args.steps):
        s = cpu_sample(c, space, coeffs, rhs, dec, budget_s=8.0)
        workers = s["workers"]
        if i >= args.warmup:
            vals.append(cpu_extrapolate(s, its))
    t = float(np.mean(vals))
    return {
        "metric": METRIC, "impl": "reference", "value": n / t, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded; BASELINE.json configs)",
        "config": {"workload": f"{c['name']} (same as the GPU arm)", "ndof": n, "iterations_assumed": its},
        "cpu_baseline": {"value": n / t, "unit": UNIT, "cores": workers, "kind": "port",
                         "sample": f"oracle restatement of the reference (numpy + SuperLU), bounded sample per step: "
                                   f"{workers} subdomain factorisations+solves in {workers} processes, SpMV, coarse "
                                   f"solve, MGS2 timings, extrapolated to a full solve"},
        "e2e": {"value": n / t, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# ------------------------------------------------------------ distributed
def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)
    return rank, world


def dist_barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(v, world):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=1, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ortho", choices=["mgs", "cgs2"], default=None,
                    help="Gram-Schmidt variant (default: mgs on one GPU, cgs2 sharded)")
    args = ap.parse_args()
    rank, world = dist_init()
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return
    res = run_mine(args, rank, world)
    if rank == 0:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
