"""Per-rank device time of the sharded multi-GPU step, measured on ONE GPU.

Each rank r of N runs alone (distributed.Communicator(emulate=(r, N))): its
block of subdomains is factorised and solved, the coarse space replicated, the
Krylov vectors sharded by row blocks (CGS2), and every collective is reduced
to its local part (allreduce: nothing; allgather: own block).  The computed
numbers are not the solve's; the step is forced to 200 iterations (tol 1e-300)
as cfg1's solve does.  Output: ms per step per rank, and the max over ranks
(the compute part of an N-GPU step; collective time is NOT included).

    python tools/rank_emulation.py [--config 1] [--ranks 1,2,4,8]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1711_03789_b200 import _lib, distributed, fem, krylov, precond  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--only-rank", type=int, default=None, help="time this rank only (profiling)")
    args = ap.parse_args()
    c = bench.CONFIGS[args.config]
    ctx = _lib.get_context()
    space, coeffs, rhs, dec, _ = bench.build_problem(c)
    n = space.ndof
    spec = precond.PreconditionerSpec(c["family"], "two", c["corr"], xi_prec=c["xi"])
    prec_coeffs = coeffs.with_xi(spec.xi_prec)
    rhs_dev = _lib.DeviceBuffer(ctx, 16 * n)
    rhs_dev.upload(rhs)
    x_dev = _lib.DeviceBuffer(ctx, 16 * n)
    kcfg = krylov.KrylovConfig(tol=1e-300, maxit=200, orthogonalization="cgs2")
    out = {"config": c["name"], "ndof": n, "collectives": "excluded (local part only)", "ranks": {}}
    for N in [int(x) for x in args.ranks.split(",")]:
        per_rank = []
        for r in (range(N) if args.only_rank is None else [args.only_rank]):
            prob = fem.assemble(space, coeffs)
            comm = distributed.Communicator(ctx, emulate=(r, N)) if N > 1 else None
            st = (distributed.setup_sharded(prob, dec, spec, comm=comm, lu_cap=None) if N > 1
                  else precond.setup(prob, dec, spec, lu_cap=None))

            def step():
                p = fem.assemble(space, coeffs)
                st.refactor(fem.assemble(space, prec_coeffs).A, prec_coeffs)
                return krylov.gmres(p.A, rhs_dev, precond=st, config=kcfg, out=x_dev)

            step()
            ctx.synchronize()
            ms = []
            for _ in range(args.steps):
                ctx.record(0)
                rep = step()
                ctx.record(3)
                ms.append(ctx.elapsed_ms(0, 3))
            per_rank.append({"rank": r, "ms": float(np.mean(ms)), "iterations": int(rep.iterations),
                             "subdomains": int(len(distributed.make_shard(dec, r, N).subdomains))})
            del st, comm
            print(N, r, per_rank[-1], flush=True)
        out["ranks"][N] = {"per_rank": per_rank, "max_ms": max(p["ms"] for p in per_rank)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
