"""Profiling driver: cfg1 setup + a short preconditioned GMRES (k_arnoldi launches)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1711_03789_b200 import fem, precond, krylov

c = bench.CONFIGS[1]
space, coeffs, rhs, dec, _ = bench.build_problem(c)
prob = fem.assemble(space, coeffs)
st = precond.setup(prob, dec, precond.PreconditionerSpec("as", "two", "additive", xi_prec=c["xi"]), lu_cap=None)
rep = krylov.gmres(prob.A, rhs, precond=st, config=krylov.KrylovConfig(tol=1e-6, maxit=int(os.environ.get("MAXIT", "60"))))
print("done", rep.iterations)
