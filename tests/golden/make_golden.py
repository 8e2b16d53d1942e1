"""Generate golden fixtures by running the REFERENCE package itself.

    python tests/golden/make_golden.py           # small fixtures (seconds)
    python tests/golden/make_golden.py --cfg0    # + the full config-0 solve (minutes)

Needs /root/reference (read-only) in this container; the fixtures are
committed so the GPU box (which has no /root/reference) can use them.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, "/root/reference/pkg/src")

from maxwelldd import decomp as rdecomp  # noqa: E402
from maxwelldd import fem as rfem  # noqa: E402
from maxwelldd import krylov as rkrylov  # noqa: E402
from maxwelldd import mesh as rmesh  # noqa: E402
from maxwelldd import precond as rprecond  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def csr_fields(prefix, m):
    m = sp.csr_matrix(m)
    return {f"{prefix}_indptr": m.indptr, f"{prefix}_indices": m.indices, f"{prefix}_data": m.data,
            f"{prefix}_shape": np.array(m.shape)}


def ragged(prefix, sets, dtype=np.int64):
    ptr = np.zeros(len(sets) + 1, dtype=np.int64)
    ptr[1:] = np.cumsum([len(s) for s in sets])
    flat = np.concatenate([np.asarray(s, dtype=dtype) for s in sets]) if sets else np.zeros(0, dtype)
    return {f"{prefix}_ptr": ptr, f"{prefix}_flat": flat}


def save(name, **arrs):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrs)
    print("wrote", path, f"{os.path.getsize(path) / 1024:.1f} KiB")


def mesh_fixture():
    out = {}
    for n in (1, 3):
        m = rmesh.build_cube_mesh(n)
        for f in ("vertices", "tets", "edges", "tet_edges", "tet_edge_signs", "boundary_edge_flags",
                  "boundary_faces", "boundary_face_normals"):
            out[f"n{n}_{f}"] = getattr(m, f)
    out["nest_3_1"] = rmesh.nesting_map(rmesh.build_cube_mesh(1), rmesh.build_cube_mesh(3))
    save("mesh.npz", **out)


def system_fixture():
    out = {}
    m3 = rmesh.build_cube_mesh(3)
    sp3 = rfem.build_edge_space(m3, "pec")
    b = rfem.assemble(sp3, rfem.Coefficients(k=2.0, xi=4.0), source=rfem.gaussian_source)
    for k in ("A", "S", "M", "Dk"):
        out.update(csr_fields(f"hom_{k}", getattr(b, k)))
    out["hom_rhs"] = b.rhs
    rng = np.random.default_rng(1)
    nt = m3.n_tets
    eps, mu, sig = 1 + 3 * rng.random(nt), 0.5 + rng.random(nt), rng.random(nt)
    out.update(het_eps=eps, het_mu=mu, het_sigma=sig)
    bh = rfem.assemble(sp3, rfem.Coefficients(k=3.0, xi=2.0, eps=eps, mu=mu, sigma=sig))
    for k in ("A", "S", "M", "Dk"):
        out.update(csr_fields(f"het_{k}", getattr(bh, k)))
    m2 = rmesh.build_cube_mesh(2)
    si = rfem.build_edge_space(m2, "impedance")
    for tag, xi in (("imp", 4.0), ("impneg", -4.0)):
        bi = rfem.assemble(si, rfem.Coefficients(k=2.0, xi=xi), source=rfem.gaussian_source)
        out.update(csr_fields(f"{tag}_A", bi.A))
        out.update(csr_fields(f"{tag}_Mb", bi.Mb))
        out[f"{tag}_rhs"] = bi.rhs
    # z-directed Gaussian of the BASELINE configs (width 0.1 -> exp(-100 r^2))
    zsrc = lambda p: np.stack([0 * p[:, 0], 0 * p[:, 0], -np.exp(-100.0 * ((p - 0.5) ** 2).sum(axis=1))], axis=1)
    out["zrhs"] = rfem.assemble_rhs(sp3, zsrc)
    s_el, m_el = rfem.element_matrices(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1.0]]))
    out.update(ref_tet_S=s_el, ref_tet_M=m_el)
    save("system.npz", **out)


def decomp_fixture():
    out = {}
    cases = {"a": (4, 2, 2, 2), "b": (3, 3, 1, 1), "c": (6, 3, 2, 3)}
    for tag, (n, p, layers, nc) in cases.items():
        s = rfem.build_edge_space(rmesh.build_cube_mesh(n), "pec")
        c = rfem.build_edge_space(rmesh.build_cube_mesh(nc), "pec")
        d = rdecomp.build_decomposition(s, p, layers, coarse_space=c)
        out.update(ragged(f"{tag}_elements", d.elements))
        out.update(ragged(f"{tag}_dofs", d.dofs))
        out.update(ragged(f"{tag}_pou", d.pou, dtype=np.float64))
        out.update(ragged(f"{tag}_impdofs", rdecomp.impedance_dof_sets(s, d.elements)))
        out.update(csr_fields(f"{tag}_R0", d.coarse.R0))
        out[f"{tag}_tetmap"] = d.coarse.tet_map
        out[f"{tag}_case"] = np.array([n, p, layers, nc])
    # impedance global space decomposition
    si = rfem.build_edge_space(rmesh.build_cube_mesh(4), "impedance")
    ci = rfem.build_edge_space(rmesh.build_cube_mesh(2), "impedance")
    di = rdecomp.build_decomposition(si, 2, 1, coarse_space=ci)
    out.update(ragged("imp_dofs", di.dofs))
    out.update(csr_fields("imp_R0", di.coarse.R0))
    save("decomp.npz", **out)


def precond_fixture():
    """All 12 family x level x correction maps on n=3, p=3, layers=1, coarse n=1
    (the reference's dense-oracle case, test_precond.py:49-80), plus a global
    impedance hybrid case."""
    out = {}
    m = rmesh.build_cube_mesh(3)
    s = rfem.build_edge_space(m, "pec")
    prob = rfem.assemble(s, rfem.Coefficients(k=2.0, xi=4.0), source=rfem.gaussian_source)
    c = rfem.build_edge_space(rmesh.build_cube_mesh(1), "pec")
    d = rdecomp.build_decomposition(s, 3, 1, coarse_space=c)
    rng = np.random.default_rng(8)
    V = rng.standard_normal((3, s.ndof)) + 1j * rng.standard_normal((3, s.ndof))
    out["v"] = V
    for fam in ("as", "ras", "impras"):
        for lev, cor in (("one", "additive"), ("two", "additive"), ("two", "hybrid"), ("two", "adef1")):
            st = rprecond.setup(prob, d, rprecond.PreconditionerSpec(fam, lev, cor, xi_prec=4.0))
            out[f"{fam}_{lev}_{cor}"] = np.stack([st.apply(v) for v in V])
    # impras local matrices of subdomain 0 (for the oracle)
    a0, g0 = rprecond.assemble_local(s, rfem.Coefficients(k=2.0, xi=4.0), d.elements[0], "impedance")
    out.update(csr_fields("imp_local0", a0))
    out["imp_local0_gdofs"] = g0
    # global impedance space, two-level hybrid impras
    mi = rmesh.build_cube_mesh(2)
    si = rfem.build_edge_space(mi, "impedance")
    pi = rfem.assemble(si, rfem.Coefficients(k=2.0, xi=4.0), source=rfem.gaussian_source)
    ci = rfem.build_edge_space(rmesh.build_cube_mesh(1), "impedance")
    di = rdecomp.build_decomposition(si, 2, 1, coarse_space=ci)
    vi = rng.standard_normal(si.ndof) + 1j * rng.standard_normal(si.ndof)
    out["gimp_v"] = vi
    for fam in ("as", "impras"):
        st = rprecond.setup(pi, di, rprecond.PreconditionerSpec(fam, "two", "hybrid", xi_prec=4.0))
        out[f"gimp_{fam}"] = st.apply(vi)
    save("precond.npz", **out)


def gmres_fixture():
    out = {}
    rng = np.random.default_rng(0)
    n = 40
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)) + 6 * np.eye(n)
    bb = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    r = rkrylov.gmres(a, bb, config=rkrylov.KrylovConfig(tol=1e-12, maxit=120))
    out.update(dense_a=a, dense_b=bb, dense_x=r.x, dense_hist=r.residual_history, dense_it=r.iterations)
    m = rmesh.build_cube_mesh(4)
    s = rfem.build_edge_space(m, "pec")
    prob = rfem.assemble(s, rfem.Coefficients(k=3.0, xi=9.0), source=rfem.gaussian_source)
    c = rfem.build_edge_space(rmesh.build_cube_mesh(2), "pec")
    d = rdecomp.build_decomposition(s, 2, 1, coarse_space=c)
    for fam, lev, cor, side, wt in (
        ("as", "two", "additive", "right", None),
        ("ras", "two", "hybrid", "left", None),
        ("ras", "one", "additive", "right", "dk"),
        ("as", "two", "adef1", "right", None),
    ):
        st = rprecond.setup(prob, d, rprecond.PreconditionerSpec(fam, lev, cor, xi_prec=9.0, side=side))
        cfg = rkrylov.KrylovConfig(tol=1e-8, maxit=200, side=side, weight=prob.Dk if wt else None)
        rr = rkrylov.gmres(prob.A, prob.rhs, precond=st.apply, config=cfg)
        tag = f"{fam}_{lev}_{cor}_{side}_{wt or 'id'}"
        out[f"{tag}_x"] = rr.x
        out[f"{tag}_hist"] = rr.residual_history
        out[f"{tag}_it"] = rr.iterations
    # random initial guess path (krylov.py:88-92)
    rr = rkrylov.gmres(prob.A, prob.rhs, precond=None,
                       config=rkrylov.KrylovConfig(tol=1e-6, maxit=60, initial_guess="random", seed=5))
    out.update(rand_x=rr.x, rand_hist=rr.residual_history, rand_it=rr.iterations)
    save("gmres.npz", **out)


def cfg0_fixture():
    """BASELINE configs[0], solved by the reference as shipped (dense LU, lu_cap raised)."""
    t0 = time.time()
    m = rmesh.build_cube_mesh(20)
    s = rfem.build_edge_space(m, "pec")
    src = lambda p: np.stack([0 * p[:, 0], 0 * p[:, 0], -np.exp(-100.0 * ((p - 0.5) ** 2).sum(axis=1))], axis=1)
    prob = rfem.assemble(s, rfem.Coefficients(k=10.0, xi=10.0), source=src)
    c = rfem.build_edge_space(rmesh.build_cube_mesh(5), "pec")
    d = rdecomp.build_decomposition(s, 2, 2, coarse_space=c)
    t1 = time.time()
    st = rprecond.setup(prob, d, rprecond.PreconditionerSpec("as", "two", "additive", xi_prec=10.0), lu_cap=20000)
    t2 = time.time()
    rr = rkrylov.gmres(prob.A, prob.rhs, precond=st.apply,
                       config=rkrylov.KrylovConfig(tol=1e-6, maxit=200, side="right", initial_guess="zero"))
    t3 = time.time()
    print(f"cfg0: decomposition {t1 - t0:.1f}s setup {t2 - t1:.1f}s gmres {t3 - t2:.1f}s its {rr.iterations}")
    save("cfg0.npz", x=rr.x, hist=rr.residual_history, it=rr.iterations, conv=rr.converged,
         rhs=prob.rhs, times=np.array([t1 - t0, t2 - t1, t3 - t2]))


if __name__ == "__main__":
    mesh_fixture()
    system_fixture()
    decomp_fixture()
    precond_fixture()
    gmres_fixture()
    if "--cfg0" in sys.argv:
        cfg0_fixture()
