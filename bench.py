"""Benchmark: preconditioned GMRES time-to-solve on the BASELINE configs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl mine|reference]

One *step* = one complete numeric solve on a fixed mesh + decomposition:
device assembly of the problem matrix A and of the shifted A_prec
(fem.assemble), numeric factorisation of every subdomain block, element-wise
Galerkin coarse block and its factorisation (PreconditionerState.refactor),
and right-preconditioned GMRES (tol 1e-6, maxit 200, zero initial guess).
Mesh, DOF pattern, decomposition and the nested-dissection symbolic analysis
are per-mesh setup, done once before timing (SURVEY.md §3.6's "setup" phase
is the numeric factorisation, which is timed).

value : DoF-iterations/s = ndof * GMRES iterations / (device time per step), SURVEY.md
        §8d's "DoFs/s", inputs resident in HBM; `time_to_solve` holds seconds per solve.
e2e   : same metric through the public API with host buffers (rhs H2D and
        x D2H inside the timed region), wall clock.

--gpus N > 1 without a torchrun environment re-launches itself under
`python -m torch.distributed.run --nproc-per-node N` (one rank per GPU).
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

from workloads import CONFIGS, MAXIT, TOL, describe, hetero_fields, random_rhs  # noqa: E402  (plain data, numpy only)

DEFAULT_CONFIG = 4  # the largest BASELINE config; fits one B200 (factors 46 GB + Krylov basis 11 GB of 180 GB)
METRIC = "precond_gmres_dof_iterations_per_s"
UNIT = "DoF*it/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------- problem
def build_problem(c, seed=0):
    from paper_1711_03789_b200 import decomp, fem, mesh

    m = mesh.build_cube_mesh(c["N"])
    space = fem.build_edge_space(m, "pec", order=c.get("order", 1))
    if c.get("hetero"):
        eps, sigma = hetero_fields(c, m.barycenters(), seed)
        coeffs = fem.Coefficients(k=c["k"], xi=c["xi"], eps=eps, sigma=sigma)
    else:
        coeffs = fem.Coefficients(k=c["k"], xi=c["xi"])
    if c["rhs"][0] == "random":
        rhs = random_rhs(space.ndof, seed)
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
def cpu_time_boxed_solve(c, box_s, min_iters=3):
    """The reference's CPU path (oracle/parallel_oracle.py: the reference pipeline with
    DenseLU swapped for ND-permuted SuperLU, all host cores) on a bounded sample of the
    workload: the REAL step from the start -- assembly, every subdomain factorisation,
    the coarse factorisation -- then GMRES iterations until the time box is spent (or
    the solve ends).  Nothing is extrapolated: value = ndof * iterations done / wall time
    of exactly that work.  Imports nothing from the product package."""
    import psutil

    from oracle import parallel_oracle as P

    t0 = time.perf_counter()
    prob = P.build_problem(c, log=log)
    t_build = time.perf_counter() - t0
    n = prob["ndof"]
    cores = os.cpu_count() or 1
    # SuperLU keeps ~33 B per factor entry; blocks beyond half the free memory are re-factored per apply
    budget = 0.5 * psutil.virtual_memory().available / 33.0
    t1 = time.perf_counter()  # the timed step starts here (mesh + decomposition are per-mesh setup in both arms)
    from oracle import maxwell_oracle as O

    A = O.assemble(prob["mesh"], prob["space"]["edge_to_dof"], n, c["k"], c["xi"], eps=prob["eps"],
                   sigma=prob["sigma"])["A"]  # the step re-assembles, as the device arm's step does
    prob["A"] = A
    t_asm = time.perf_counter() - t1
    with P.ParallelSchwarz(prob, workers=cores, resident_entries=budget, log=log) as M:
        t_setup = time.perf_counter() - t1
        t2 = time.perf_counter()
        # ONE solve, stopped at the first iteration boundary past the time box
        x, hist, its, conv, tm = P.gmres(A, prob["rhs"], M.apply, tol=TOL, maxit=MAXIT, deadline=t1 + box_s,
                                         min_iters=min_iters)
        t_gmres = time.perf_counter() - t2
        entries = M.factor_entries
        workers = M.workers
    wall = t_setup + t_gmres  # assembly + every factorisation + the (truncated) solve
    return {"value": n * its / wall, "ndof": n, "iterations": int(its), "converged": bool(conv), "wall_s": wall,
            "assemble_s": t_asm, "setup_s": t_setup, "gmres_s": t_gmres, "phases": tm, "cores": cores,
            "workers": workers, "build_s": t_build, "factor_entries": entries, "final_rel_residual": float(hist[-1]),
            "resident_entries_cap": budget}


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
        # strong scaling: each rank factorises/solves its block of subdomains and owns a row
        # block of every vector; halo gathers and overlap sums with the neighbours, no
        # whole-vector collective in the loop (distributed.py)
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
    kcfg = krylov.KrylovConfig(tol=TOL, maxit=MAXIT, side="right", initial_guess="zero", orthogonalization=ortho,
                               check_orthogonality=not args.no_drift)
    rhs_dev = _lib.DeviceBuffer(ctx, 16 * n)
    rhs_dev.upload(rhs)
    x_dev = _lib.DeviceBuffer(ctx, 16 * n)
    prec_coeffs = coeffs.with_xi(spec.xi_prec)

    # a rank of a sharded run assembles the cells that touch its needed rows only
    # (the sharded CGS2 loop multiplies owned rows only; MGS2 keeps whole vectors and the whole A)
    rows = getattr(st, "assembly_rows", None) if world > 1 and ortho == "cgs2" else None

    def step(device_io=True):
        p = fem.assemble(space, coeffs, rows=rows)
        ctx.record(1)
        a_prec = fem.assemble(space, prec_coeffs, rows=rows).A
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
    with ClockSampler(int(ctx.device)) as clk:
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

    torch.cuda.set_device(int(ctx.device))  # pin through the solver context's own GPU
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
    # three flop counts (include/mdd.h: mdd_prec_flop_counts): what the kernels executed (the
    # rate the tensor pipe ran at: `achieved`), the partial-LU count of the same fronts (what the
    # reference's zgetrf would need) and the nominal 8 np m^2 of a full elimination
    tf = lambda fl: fl / (fac_ms / 1e3) / 1e12 if fac_ms > 0 else 0.0  # noqa: E731
    f_ach = tf(stats["executed_flops"])
    roof_factor = {"bound": "tensor", "kernel": "numeric factorisation (k_front_init, GJ sweeps k_gj_small/k_panel/"
                                                "k_update, k_gemm DMMA F_PU/Schur, k_transpose_up), subdomains + coarse",
                   "achieved": f_ach, "peak": fpk["tflops"], "unit": "TFLOP/s", "frac": f_ach / fpk["tflops"],
                   "flops": stats["executed_flops"], "ms": fac_ms, "peak_source": fpk["source"],
                   "lu_flops": stats["lu_flops"], "lu_equivalent_tflops": tf(stats["lu_flops"]),
                   "lu_equivalent_frac": tf(stats["lu_flops"]) / fpk["tflops"],
                   "nominal_flops_8npm2": stats["factor_flops"], "nominal_tflops": tf(stats["factor_flops"])}
    hist = rep.residual_history
    res = {
        "metric": METRIC,
        "value": n * its / (ms_step / 1e3),  # DoFs/s = n * iterations / solve time; one solve per step
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
            "workload": describe(c, n, spec.label()),
            "ndof": n, "subdomains": len(dec.dofs), "iterations": its, "converged": bool(rep.converged),
            "final_rel_residual": float(hist[-1]),
            "parallelism": (f"subdomains sharded over {world} GPUs as x-slabs of boxes, rows owned in blocks; per "
                            "apply: neighbour halo gather (ncclSend/Recv) for restriction and SpMV, neighbour "
                            "overlap sum for prolongation, allreduce of the coarse restriction (coarse factor "
                            "replicated); "
                            + ("Krylov vectors sharded by owned rows (CGS2: 3 small allreduces per iteration)"
                               if ortho == "cgs2" else "MGS2 GMRES replicated (whole-vector completion per apply)"))
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
        "time_to_solve": {"s_per_solve": ms_step / 1e3, "dofs_per_s": n / (ms_step / 1e3),
                          "cold_s": t_dec + t_setup + ms_step / 1e3,
                          "cold_includes": "decomposition + first setup (symbolic ND analysis, allocation, first "
                                           "numeric factorisation) + one timed step"},
        "e2e": {"value": n * rep_e.iterations / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": 16 * n,
                "s_per_step": e2e_s, "s_steps": [round(v, 4) for v in e2e_t], "iterations": rep_e.iterations},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        if c.get("order", 1) != 1:
            res["cpu_baseline"] = None  # no CPU reference exists for the order-2 extension
        else:
            res["cpu_baseline"] = cpu_baseline_record(cpu_time_boxed_solve(c, args.cpu_box))
    return res


def cpu_baseline_record(s):
    return {"value": s["value"], "unit": UNIT, "cores": s["cores"], "kind": "port",
            "sample": f"oracle port of the reference (numpy + ND-SuperLU, {s['workers']} worker processes + threaded "
                      f"BLAS) on the same workload, one real step from the start: assembly {s['assemble_s']:.1f}s, all "
                      f"subdomain + coarse factorisations (setup {s['setup_s']:.1f}s incl. assembly), then the first "
                      f"{s['iterations']} GMRES iterations ({s['gmres_s']:.1f}s) of the solve; value = ndof*iterations"
                      f"/wall ({s['wall_s']:.1f}s), nothing extrapolated",
            "iterations": s["iterations"], "wall_s": s["wall_s"], "setup_s": s["setup_s"], "gmres_s": s["gmres_s"],
            "phases_s": s["phases"], "final_rel_residual": s["final_rel_residual"], "converged": s["converged"]}


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
    """The reference's CPU implementation of the path on this box's host cores.  The
    reference package is pure Python and cannot travel to the GPU box, and its dense LU
    cannot hold any config beyond cfg0, so this is the oracle port (kind "port"), built
    product-free (oracle/geometry_oracle.py: no libmdd.so is loaded by this arm).

    A full CPU step at the headline config takes minutes, so the whole run is ONE real
    step from the start, time-boxed (--ref-box seconds): assembly, all factorisations,
    then GMRES iterations until the box is spent.  --steps/--warmup are echoed but not
    multiplied: "steps_run" says what ran.  value = ndof * iterations / wall."""
    c = CONFIGS[args.config]
    if c.get("order", 1) != 1:
        return {"impl": "reference", "unavailable": "no CPU reference exists for the order-2 extension (cfg2)"}
    s = cpu_time_boxed_solve(c, args.ref_box, min_iters=5)
    label = {"additive": "2", "hybrid": "-H", "adef1": "-ADEF1"}[c["corr"]]
    label = {"as": "AS", "ras": "RAS", "impras": "ImpRAS"}[c["family"]] + label
    return {
        "metric": METRIC, "impl": "reference", "value": s["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "steps_run": 1, "warmup_run": 0,
        "ms_per_step": s["wall_s"] * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded; BASELINE.json configs)",
        "config": {"workload": describe(c, s["ndof"], label), "ndof": s["ndof"], "iterations": s["iterations"],
                   "converged": s["converged"], "final_rel_residual": s["final_rel_residual"],
                   "time_box_s": args.ref_box},
        "cpu_baseline": cpu_baseline_record(s),
        "e2e": {"value": s["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "product_imported": "paper_1711_03789_b200" in sys.modules,
        "repo_so_mapped": _mapped_repo_libraries(),
    }


def _mapped_repo_libraries():
    try:
        with open("/proc/self/maps") as f:
            return sorted({ln.split()[-1] for ln in f if ".so" in ln and ROOT in ln})
    except OSError:
        return None


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


def torchrun_command(n, argv, port=None):
    """The launch line the driver itself uses for N > 1 (one rank per GPU, NCCL over NVLink)."""
    if port is None:
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]


def visible_gpus():
    from paper_1711_03789_b200 import _lib

    return _lib.device_count()


def relaunch_under_torchrun(n, argv, count=visible_gpus, run=subprocess.call):
    have = count()
    if have < n:
        print(f"bench.py: --gpus {n} requested but only {have} CUDA device(s) are visible", file=sys.stderr)
        return 2
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # keep NCCL's transport lines (NVLS / P2P) in the log
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return run(torchrun_command(n, argv), env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--cpu-box", type=float, default=120.0,
                    help="time box (s) of the cpu_baseline leg's real CPU step (setup + first GMRES iterations)")
    ap.add_argument("--ref-box", type=float, default=180.0,
                    help="time box (s) of the --impl reference arm's one real CPU step")
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-drift", action="store_true",
                    help="experiment: skip the reference's orthogonality-drift check (krylov.py:152-160)")
    ap.add_argument("--ortho", choices=["mgs", "cgs2"], default=None,
                    help="Gram-Schmidt variant (default: mgs on one GPU, cgs2 sharded)")
    args = ap.parse_args()
    if args.impl == "mine" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args.gpus, sys.argv[1:]))
    rank, world = dist_init()
    if args.impl == "mine" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return
    res = run_mine(args, rank, world)
    if rank == 0:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
