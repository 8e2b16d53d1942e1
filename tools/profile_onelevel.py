"""Profiling driver: cfg1 setup, then restriction + subdomain solves only
(mdd_prec_apply_bench which=1: 3 warm-up applies, REPS timed)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1711_03789_b200 import fem, precond, _lib

c = bench.CONFIGS[int(os.environ.get("CFG", "1"))]
space, coeffs, rhs, dec, _ = bench.build_problem(c)
prob = fem.assemble(space, coeffs)
st = precond.setup(prob, dec, precond.PreconditionerSpec(c["family"], "two", c["corr"], xi_prec=c["xi"]), lu_cap=None)
ms = C.c_double()
_lib.check(_lib.lib.mdd_prec_apply_bench(st._h, 1, int(os.environ.get("REPS", "0")), C.byref(ms)))
print("done", ms.value)
