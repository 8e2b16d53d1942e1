"""Profiling driver: cfg setup (one factorisation), then REFACTORS numeric refactorisations."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1711_03789_b200 import fem, precond, _lib

c = bench.CONFIGS[int(os.environ.get("CFG", "1"))]
space, coeffs, rhs, dec, _ = bench.build_problem(c)
prob = fem.assemble(space, coeffs)
st = precond.setup(prob, dec, precond.PreconditionerSpec(c["family"], "two", c["corr"], xi_prec=c["xi"]), lu_cap=None)
pc = coeffs.with_xi(c["xi"])
for _ in range(int(os.environ.get("REFACTORS", "1"))):
    st.refactor(fem.assemble(space, pc).A, pc)
_lib.get_context().synchronize()
print("done", st.stats())
