"""One host-driven (MDD_NO_GRAPH=1) GMRES solve of a BASELINE config, for ncu captures of the
loop kernels (kernels inside a conditional graph node are invisible to ncu).

    MDD_NO_GRAPH=1 python tools/prof_arnoldi.py 4 120     # config, maxit
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MDD_NO_GRAPH", "1")

import bench  # noqa: E402
import workloads as W  # noqa: E402
from paper_1711_03789_b200 import fem, krylov, precond  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 120
c = W.CONFIGS[cfg]
space, coeffs, rhs, dec, _ = bench.build_problem(c)
prob = fem.assemble(space, coeffs)
st = precond.setup(prob, dec, precond.PreconditionerSpec(c["family"], "two", c["corr"], xi_prec=c["xi"]), lu_cap=None)
t = time.time()
rep = krylov.gmres(prob.A, rhs, precond=st, config=krylov.KrylovConfig(tol=W.TOL, maxit=maxit))
print(f"{c['name']}: {rep.iterations} iterations in {time.time() - t:.2f}s, final {rep.residual_history[-1]:.6e}")
