"""Residual histories of MGS2, CGS2 sweeps and CGS2 row-tiled on one mid-size case (debug aid)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1711_03789_b200 import decomp, fem, mesh, precond
from paper_1711_03789_b200.krylov import KrylovConfig, gmres

s = fem.build_edge_space(mesh.build_cube_mesh(8), "pec")
prob = fem.assemble(s, fem.Coefficients(k=6.0, xi=6.0), source=fem.gaussian_source)
d = decomp.build_decomposition(s, 2, 2, coarse_space=fem.build_edge_space(mesh.build_cube_mesh(2), "pec"))
st = precond.setup(prob, d, precond.PreconditionerSpec("as", "two", "additive", xi_prec=6.0), lu_cap=None)
out = {}
for name, env, ortho in [("mgs", "1", "mgs"), ("tiled", "1", "cgs2"), ("tiled2", "1", "cgs2"), ("sweeps", "0", "cgs2"), ("sweeps2", "0", "cgs2")]:
    os.environ["MDD_CGS_FUSED"] = env
    r = gmres(prob.A, prob.rhs, precond=st, config=KrylovConfig(tol=1e-10, maxit=200, orthogonalization=ortho))
    out[name] = {"it": r.iterations, "hist": r.residual_history.tolist(), "x0": [r.x[0].real, r.x[0].imag]}
json.dump(out, open("gpurun_out/cgs_compare.json", "w"))
for k, v in out.items():
    print(k, v["it"], ["%.6e" % h for h in v["hist"][18:28]])
