"""Small end-to-end case for compute-sanitizer (one tool per gpurun call, B200_PROFILING.md):
assembly (k_assemble_cells), preconditioner setup and applies (k_solve_tma, k_scatter_owner),
host-driven GMRES (k_arnoldi register path, then the wide path forced through the test hooks).

    MDD_NO_GRAPH=1 compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MDD_NO_GRAPH", "1")

import numpy as np  # noqa: E402

from paper_1711_03789_b200 import decomp, fem, krylov, mesh, precond  # noqa: E402

s = fem.build_edge_space(mesh.build_cube_mesh(6), "pec")
prob = fem.assemble(s, fem.Coefficients(k=4.0, xi=4.0), source=fem.gaussian_source)
d = decomp.build_decomposition(s, 2, 1, coarse_space=fem.build_edge_space(mesh.build_cube_mesh(2), "pec"))
for fam, cor in (("as", "additive"), ("impras", "hybrid")):
    st = precond.setup(prob, d, precond.PreconditionerSpec(fam, "two", cor, xi_prec=4.0), lu_cap=None)
    rep = krylov.gmres(prob.A, prob.rhs, precond=st, config=krylov.KrylovConfig(tol=1e-8, maxit=60))
    print(fam, cor, "register path:", rep.iterations, rep.converged, float(rep.residual_history[-1]))
os.environ["MDD_ARNOLDI_MODE"] = "2"
os.environ["MDD_ARN_GRID"] = "3"
os.environ["MDD_ARNOLDI_WCAP"] = "200"
os.environ["MDD_ARN_ZIGZAG"] = "1"
rep2 = krylov.gmres(prob.A, prob.rhs, precond=st, config=krylov.KrylovConfig(tol=1e-8, maxit=60))
print("wide path:", rep2.iterations, rep2.converged, float(np.abs(rep2.x - rep.x).max()))
