"""Profiling driver: cfg1 setup, then a few preconditioner applies and one
numeric refactorisation (run under ncu with -k filters)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_1711_03789_b200 import fem, precond, _lib

c = bench.CONFIGS[int(os.environ.get("CFG", "1"))]
space, coeffs, rhs, dec, _ = bench.build_problem(c)
prob = fem.assemble(space, coeffs)
st = precond.setup(prob, dec, precond.PreconditionerSpec(c["family"], "two", c["corr"], xi_prec=c["xi"]), lu_cap=None)
ctx = _lib.get_context()
for _ in range(int(os.environ.get("APPLIES", "3"))):
    st.apply(rhs)
if os.environ.get("REFACTOR"):
    st.refactor(fem.assemble(space, coeffs.with_xi(c["xi"])).A)
ctx.synchronize()
print("done", st.stats())
