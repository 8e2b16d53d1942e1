"""Config-scale parity at the BASELINE sizes against committed oracle goldens.

tests/golden/cfg{1,3,4}_oracle.npz come from tests/golden/make_golden_configs.py
(the pinned CPU oracle, oracle/parallel_oracle.py, run at full size in the
build container; reference path: krylov.py:134-198 over precond.py:217-245).
Each case builds the same problem through the product API, then checks

* one preconditioner apply on a seeded vector     (<= 1e-10 of |M^-1 v|),
* the residual history of the solve: rtol 1e-8 over the first 20 points; after that within
  the oracle's OWN sensitivity envelope.  These solves stagnate for a long time and their
  later history is chaotic in the rounding: perturbing every preconditioner output of the
  oracle by a relative 1e-13 (the device/oracle apply difference is 3e-14 .. 3e-13) moves its
  cfg1 history by 6e-10 up to iteration 50, 6.5e-3 by iteration 100 and 4e-2 by iteration 200.
  The goldens store that perturbed history (`hist_pert`, make_golden_configs.py
  --sensitivity); the device history may deviate by 50x what the oracle itself moved up to
  the same iteration (floor 1e-8, cap 0.1), and by at most 0.1 beyond the stored range;
* the iterate after 20 iterations (a run with maxit=20): <= 1e-8 of |x| (north_star),
  and the final iterate within the late-history sensitivity (5e-2 of |x|),

through 16 seeded projections and a strided sample of the vectors (the full
vectors are not committed: 3.5M complex entries at cfg4).
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _load(name):
    path = os.path.join(GOLDEN, f"{name}_oracle.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    return dict(np.load(path, allow_pickle=False))


def _check_vector(got, g, prefix, norm, tol):
    import workloads as W

    n = len(got)
    probes = W.probe_vectors(n)
    stride = W.sample_stride(n)
    samp = got[::stride]
    e_samp = np.linalg.norm(samp - g[prefix + "_samp"]) / np.linalg.norm(g[prefix + "_samp"])
    e_proj = np.abs(probes.conj() @ got - g[prefix + "_proj"]).max() / norm  # |p_i| ~ 1
    assert e_samp <= tol, f"{prefix} sample differs by {e_samp:.3e}"
    assert e_proj <= tol, f"{prefix} projections differ by {e_proj:.3e}"
    return e_samp, e_proj


@pytest.mark.parametrize("cfg", [1, 3, 4])
def test_config_matches_oracle_golden(gpu, cfg):
    import bench
    import workloads as W
    from paper_1711_03789_b200 import fem, krylov, precond

    c = W.CONFIGS[cfg]
    g = _load(c["name"])
    space, coeffs, rhs, dec, _ = bench.build_problem(c)
    n = space.ndof
    assert n == int(g["ndof"])
    prob = fem.assemble(space, coeffs)
    st = precond.setup(prob, dec, precond.PreconditionerSpec(c["family"], "two", c["corr"], xi_prec=c["xi"]),
                       lu_cap=None)
    v = W.random_rhs(n, seed=777)
    e_ap = _check_vector(st.apply(v), g, "ap", float(g["apnorm"]), 1e-10)
    maxit = int(g["maxit"])
    rep = krylov.gmres(prob.A, rhs, precond=st, config=krylov.KrylovConfig(tol=W.TOL, maxit=maxit, side="right",
                                                                          initial_guess="zero"))
    hist = g["hist"]
    assert rep.converged == bool(g["conv"])
    assert abs(rep.iterations - int(g["its"])) <= 1
    k = min(len(hist), len(rep.residual_history))
    h = np.asarray(rep.residual_history)
    dev = np.abs(h[:k] / hist[:k] - 1)
    print(json.dumps({"cfg": c["name"], "apply_err": e_ap, "iterations": rep.iterations, "final": float(h[-1]),
                      "golden_final": float(hist[-1]), "hist_dev_to_20": float(dev[:21].max()),
                      "hist_dev_to_50": float(dev[:51].max()), "hist_dev_all": float(dev.max())}))
    assert dev[:21].max() <= 1e-8
    tol = np.full(k, 0.1)
    if "hist_pert" in g:
        kp = min(k, len(g["hist_pert"]))
        own = np.maximum.accumulate(np.abs(g["hist_pert"][:kp] / hist[:kp] - 1))
        tol[:kp] = np.clip(50.0 * own, 1e-8, 0.1)
    else:
        tol[:51] = 1e-6  # measured for cfg1; configs without a stored envelope are held to it
    worst = int(np.argmax(dev / tol))
    assert np.all(dev <= tol), f"history deviates by {dev[worst]:.3e} at iteration {worst} (allowed {tol[worst]:.3e})"
    if rep.iterations == int(g["its"]):
        print(json.dumps({"x_err_final": _check_vector(rep.x, g, "x", float(g["xnorm"]), 5e-2)}))
    if "xs_samp" in g:
        short = int(g["short"])
        rs = krylov.gmres(prob.A, rhs, precond=st, config=krylov.KrylovConfig(tol=W.TOL, maxit=short, side="right",
                                                                             initial_guess="zero"))
        assert rs.iterations == short
        print(json.dumps({"x_err_short": _check_vector(rs.x, g, "xs", float(g["xsnorm"]), 1e-8)}))
