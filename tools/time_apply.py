"""Device-timed preconditioner applies on a BASELINE config (CFG env, default 1):
full apply, restriction + subdomain solves, coarse solve (ms per call)."""
import json, os, sys
import ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1711_03789_b200 import fem, precond, _lib

c = bench.CONFIGS[int(os.environ.get("CFG", "1"))]
space, coeffs, rhs, dec, _ = bench.build_problem(c)
prob = fem.assemble(space, coeffs)
st = precond.setup(prob, dec, precond.PreconditionerSpec(c["family"], "two", c["corr"], xi_prec=c["xi"]), lu_cap=None)
out = {"cfg": c["name"], "env": {k: v for k, v in os.environ.items() if k.startswith("MDD_")}}
for which, name in ((0, "apply"), (1, "one_level"), (2, "coarse")):
    ms = C.c_double()
    _lib.check(_lib.lib.mdd_prec_apply_bench(st._h, which, int(os.environ.get("REPS", "20")), C.byref(ms)))
    out[name + "_ms"] = ms.value
s = st.stats()
out["factor_entries"] = s["factor_entries"]
out["apply_GBps_factor_only"] = 16 * s["factor_entries"] / (out["apply_ms"] * 1e-3) / 1e9
print(json.dumps(out), flush=True)
