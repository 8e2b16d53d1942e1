"""Config-scale golden fixtures: the pinned CPU oracle at the BASELINE sizes.

    python tests/golden/make_golden_configs.py 1            # cfg1, 200 iterations (~3 min on 8 cores)
    python tests/golden/make_golden_configs.py 3 --maxit 200
    python tests/golden/make_golden_configs.py 4 --maxit 40 --resident-entries 1e9   # factors exceed 62 GB of host memory
    python tests/golden/make_golden_configs.py 1 --check-reference     # + geometry/assembly hashes vs /root/reference

What runs is oracle/parallel_oracle.py: the reference pipeline with DenseLU
replaced by ND-permuted SuperLU (validated against the reference's own dense
solve at cfg0 to 3e-12 / same 41 iterations).  The reference as shipped
cannot run these sizes.

Stored per config in tests/golden/cfgK_oracle.npz (a few hundred KiB):

    hist            residual history of the (possibly truncated) solve
    its, conv       iteration count, convergence flag
    x_proj, x_samp  16 seeded projections <p_i, x> and a strided sample of x
    ap_proj, ap_samp the same for one preconditioner apply M^{-1} v on a seeded v
    xnorm, apnorm   2-norms
    times           oracle wall times (setup, gmres by phase), cores
    maxit           iteration cap of this run (200 = the full BASELINE solve)

x is the solution after `its` iterations; when the run was capped (maxit <
200) the GPU test solves with the same cap.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402
from oracle import parallel_oracle as P  # noqa: E402


def log(*a):
    print(*a, flush=True)


def digest(arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def check_against_reference(c, prob):
    """Mesh, DOF sets, PoU, R0 and A of the oracle-side problem vs the reference package itself."""
    sys.path.insert(0, "/root/reference/pkg/src")
    from maxwelldd import decomp as rdecomp
    from maxwelldd import fem as rfem
    from maxwelldd import mesh as rmesh

    t0 = time.time()
    m = rmesh.build_cube_mesh(c["N"])
    s = rfem.build_edge_space(m, "pec")
    cs = rfem.build_edge_space(rmesh.build_cube_mesh(c["nc"]), "pec")
    if c.get("hetero"):
        eps, sigma = W.hetero_fields(c, m.barycenters(), 0)
        co = rfem.Coefficients(k=c["k"], xi=c["xi"], eps=eps, sigma=sigma)
    else:
        co = rfem.Coefficients(k=c["k"], xi=c["xi"])
    ra = rfem.assemble(s, co).A
    a = prob["A"]
    out = {"A_pattern_equal": bool(np.array_equal(ra.indptr, a.indptr) and np.array_equal(ra.indices, a.indices)),
           "A_max_rel_diff": float(np.abs(ra.data - a.data).max() / np.abs(ra.data).max())}
    log(f"[check] assembly vs reference: {out}  ({time.time() - t0:.0f}s)")
    d = rdecomp.build_decomposition(s, c["p"], c["layers"], coarse_space=cs)
    dofs = rdecomp.impedance_dof_sets(s, d.elements) if c["family"] == "impras" else d.dofs
    out["elements_equal"] = digest(d.elements) == digest(prob["dec"]["elements"])
    out["dofs_equal"] = digest(dofs) == digest(prob["dec"]["dofs"])
    out["R0_max_abs_diff"] = float(abs(d.coarse.R0 - prob["dec"]["R0"]).max())
    out["reference_decomposition_s"] = time.time() - t0
    log(f"[check] decomposition vs reference: {out}")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int, choices=[0, 1, 3, 4])
    ap.add_argument("--maxit", type=int, default=W.MAXIT)
    ap.add_argument("--workers", type=int, default=None)
    ap.add_argument("--resident-entries", type=float, default=None,
                    help="cap on factor entries kept in host memory (~33 B each); the rest is re-factored per apply")
    ap.add_argument("--check-reference", action="store_true")
    ap.add_argument("--short", type=int, default=20)
    ap.add_argument("--short-only", action="store_true")
    ap.add_argument("--update", action="store_true", help="with --sensitivity: add to the existing file, no main run")
    ap.add_argument("--sensitivity", type=int, default=0, metavar="K",
                    help="add hist_pert: the oracle's own history over K iterations when every preconditioner "
                         "output is perturbed by a relative 1e-13 (the size of the device/oracle apply difference)")
    args = ap.parse_args()
    c = W.CONFIGS[args.config]
    t_all = time.time()
    prob = P.build_problem(c, log=log)
    n = prob["ndof"]
    extra = {}
    if args.check_reference:
        extra = check_against_reference(c, prob)
    probes = W.probe_vectors(n)
    stride = W.sample_stride(n)
    with P.ParallelSchwarz(prob, workers=args.workers, resident_entries=args.resident_entries, log=log) as M:
        v = W.random_rhs(n, seed=777)
        t0 = time.time()
        av = M.apply(v)
        t_apply = time.time() - t0
        log(f"[oracle] one apply {t_apply:.2f}s")
        out = os.path.join(HERE, f"{c['name']}_oracle.npz")
        snaps = {args.short: None}
        def perturbed_history(k):
            rng = np.random.default_rng(99)

            def noisy(vv):
                y = M.apply(vv)
                return y * (1.0 + 1e-13 * rng.standard_normal(len(y)))

            return P.gmres(prob["A"], prob["rhs"], noisy, tol=W.TOL, maxit=W.MAXIT, max_iters=k, log=log)[1]

        if args.short_only or (args.sensitivity and args.update):
            old = dict(np.load(out, allow_pickle=False))
            if args.short_only:
                xs = P.gmres(prob["A"], prob["rhs"], M.apply, tol=W.TOL, maxit=W.MAXIT, max_iters=args.short,
                             log=log)[0]
                old.update(xs_proj=probes.conj() @ xs, xs_samp=xs[::stride], xsnorm=np.linalg.norm(xs),
                           short=args.short)
            if args.sensitivity:
                hp = perturbed_history(args.sensitivity)
                old.update(hist_pert=hp, pert_level=1e-13)
                k = min(len(hp), len(old["hist"]))
                log("max rel deviation under the perturbation:", float(np.abs(hp[:k] / old["hist"][:k] - 1).max()))
            np.savez_compressed(out, **old)
            log("updated", out, f"{os.path.getsize(out) / 1024:.1f} KiB")
            return
        t0 = time.time()
        x, hist, its, conv, tm = P.gmres(prob["A"], prob["rhs"], M.apply, tol=W.TOL, maxit=args.maxit, log=log,
                                         snapshots=snaps)
        t_gmres = time.time() - t0
        xs = snaps[args.short] if snaps[args.short] is not None else x
        hist_pert = perturbed_history(args.sensitivity) if args.sensitivity else None
        res = np.linalg.norm(prob["rhs"] - prob["A"] @ x) / np.linalg.norm(prob["rhs"])
        log(f"[oracle] {c['name']}: {its} iterations conv={conv} hist[-1]={hist[-1]:.6e} true rel.res {res:.6e} "
            f"gmres {t_gmres:.1f}s setup {M.setup_time_s:.1f}s")
        times = {"setup_s": M.setup_time_s, "gmres_s": t_gmres, "apply_s": t_apply, "phases": tm,
                 "workers": M.workers, "cores": os.cpu_count(), "build": prob["times"],
                 "factor_entries": M.factor_entries, "resident_entries_cap": args.resident_entries,
                 "total_s": time.time() - t_all, **extra}
    np.savez_compressed(out, hist=hist, its=its, conv=conv, maxit=args.maxit, ndof=n,
                        x_proj=probes.conj() @ x, x_samp=x[::stride], xnorm=np.linalg.norm(x),
                        ap_proj=probes.conj() @ av, ap_samp=av[::stride], apnorm=np.linalg.norm(av),
                        xs_proj=probes.conj() @ xs, xs_samp=xs[::stride], xsnorm=np.linalg.norm(xs),
                        short=min(args.short, its), true_rel_res=res, times=json.dumps(times),
                        **({"hist_pert": hist_pert, "pert_level": 1e-13} if hist_pert is not None else {}))
    log("wrote", out, f"{os.path.getsize(out) / 1024:.1f} KiB", json.dumps(times))


if __name__ == "__main__":
    main()
