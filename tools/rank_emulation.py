"""Per-rank device time of the sharded multi-GPU step, measured on ONE GPU.

Each rank r of N runs alone against tools/nccl_stub (a stand-in libnccl whose collectives do
only their local part; libmdd loads it through MDD_NCCL_LIB -- the product library holds no
emulation code): its block of subdomains is factorised and solved, the coarse space replicated,
the Krylov vectors sharded by row blocks (CGS2), halo and overlap-sum exchanges reduced to
nothing.  The computed numbers are not the solve's; the step is forced to 200 iterations
(tol 1e-300).  Output: ms per step per rank, the max over ranks (the compute part of an N-GPU
step) and the bytes each rank would exchange per iteration (from mdd_prec_halo_info), costed at
NVLink 5's 900 GB/s per direction.

    python tools/rank_emulation.py [--config 4] [--ranks 1,2,4,8] [--sample-ranks 2]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import ctypes as C  # noqa: E402
import subprocess  # noqa: E402

STUB_DIR = os.path.join(ROOT, "tools", "nccl_stub")
STUB = os.path.join(STUB_DIR, "_build", "libnccl_stub.so")
if not os.path.exists(STUB):
    os.makedirs(os.path.dirname(STUB), exist_ok=True)
    subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-I/usr/local/cuda/include",
                           os.path.join(STUB_DIR, "nccl_stub.c"), "-o", STUB, "-L/usr/local/cuda/lib64", "-lcudart"])
os.environ["MDD_NCCL_LIB"] = STUB

import bench  # noqa: E402
from paper_1711_03789_b200 import _lib, distributed, fem, krylov, precond  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--sample-ranks", type=int, default=0, help="time only this many ranks per N (first, middle, ...)")
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
    out = {"config": c["name"], "ndof": n, "collectives": "excluded from ms (tools/nccl_stub); bytes reported",
           "ranks": {}}
    for N in [int(x) for x in args.ranks.split(",")]:
        per_rank = []
        ranks = list(range(N)) if args.only_rank is None else [args.only_rank]
        if args.sample_ranks and len(ranks) > args.sample_ranks:
            ranks = sorted({ranks[int(round(i * (len(ranks) - 1) / max(1, args.sample_ranks - 1)))]
                            for i in range(args.sample_ranks)} | {len(ranks) // 2})
        for r in ranks:
            prob = fem.assemble(space, coeffs)
            comm = distributed.Communicator(ctx, standalone=(r, N, b"\x07" * 128)) if N > 1 else None
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
            rec = {"rank": r, "ms": float(np.mean(ms)), "iterations": int(rep.iterations),
                   "subdomains": int(len(distributed.make_shard(dec, r, N).subdomains))}
            if N > 1:
                v = [C.c_int64() for _ in range(5)]
                _lib.check(_lib.lib.mdd_prec_halo_info(st._h, *[C.byref(x) for x in v]))
                own, need, ghost = v[1].value - v[0].value, v[3].value - v[2].value, v[4].value
                # per iteration (additive, right): halo gather of v, overlap sum of M^-1 v, halo gather of z
                xbytes = 3 * 16 * ghost
                rec.update(owned_rows=own, needed_rows=need, ghost_rows=ghost, exchange_bytes_per_iteration=xbytes,
                           exchange_ms_per_step_at_900GBs=1e3 * rep.iterations * xbytes / 900e9,
                           whole_vector_bytes_per_iteration_before=2 * 16 * n)
            per_rank.append(rec)
            del st, comm
            print(N, r, per_rank[-1], flush=True)
        out["ranks"][N] = {"per_rank": per_rank, "max_ms": max(p["ms"] for p in per_rank)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
