"""Per-CTA timeline of one k_arnoldi_wide launch (tools build with -DMDD_ARN_TRACE).

    python tools/arn_trace.py build                 # here: tools/_trace/libmdd_trace.so
    MDD_LIB_PATH=tools/_trace/libmdd_trace.so python tools/arn_trace.py run 4 100   # on the GPU box

The kernel stamps %globaltimer per CTA and MGS step after the exchange (sweep start) and after
the CTA's block sum (sweep end); the last launch's stamps are summarised: sweep time per CTA
(min / median / max), the exchange (slowest sweep end -> median next start), the share of the
step a median CTA spends waiting for the slowest one.
"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.environ.get("MDD_TRACE_LIB") or os.path.join(ROOT, "tools", "_trace", "libmdd_trace.so")
if not os.path.isabs(OUT):
    OUT = os.path.join(ROOT, OUT)


def build(extra=()):
    from paper_1711_03789_b200 import build as B  # noqa: F401  (normal objects first)
    B.build()
    obj = OUT[:-3] + ".o"
    os.makedirs(os.path.dirname(obj), exist_ok=True)
    r = subprocess.run([B.NVCC, *B.CUFLAGS, "-DMDD_ARN_TRACE", *extra, "-c", os.path.join(B.CSRC, "gmres.cu"), "-o", obj],
                       check=True, capture_output=True, text=True)
    for ln in r.stderr.splitlines():
        if "k_arnoldi_wide" in ln:
            print(ln)
        elif "spill" in ln and getattr(build, "_w", False):
            print(ln)
        build._w = "k_arnoldi_wide" in ln
    objs = [os.path.join(B.OBJ, s + ".o") for s in B.SOURCES if s != "gmres.cu"] + [obj]
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", OUT, *objs, "-cudart", "static", "-lpthread", "-ldl"], check=True)
    print(OUT)


def run(cfg, maxit):
    os.environ["MDD_NO_GRAPH"] = "1"
    os.environ["MDD_LIB_PATH"] = OUT
    import numpy as np

    import bench
    import workloads as W
    from paper_1711_03789_b200 import _lib, fem, krylov, precond

    c = W.CONFIGS[cfg]
    space, coeffs, rhs, dec, _ = bench.build_problem(c)
    prob = fem.assemble(space, coeffs)
    st = precond.setup(prob, dec, precond.PreconditionerSpec(c["family"], "two", c["corr"], xi_prec=c["xi"]), lu_cap=None)
    rep = krylov.gmres(prob.A, rhs, precond=st, config=krylov.KrylovConfig(tol=W.TOL, maxit=maxit))
    m = rep.iterations
    lib = ctypes.CDLL(OUT)
    K = 160
    cnt = (2 * 512 + 1) * K * 2
    buf = np.zeros(cnt, dtype=np.uint64)
    rc = lib.mdd_debug_arn_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(cnt))
    assert rc == 0, rc
    t = buf.reshape(2 * 512 + 1, K, 2).astype(np.int64)
    G = 148
    smid = t[1024, :G, 0]
    t0 = t[1024, :G, 1]
    ns = 2 * m
    start = t[:ns, :G, 0]   # sweep start (after the exchange)
    end = t[:ns, :G, 1]     # sweep end
    sweep = (end - start) / 1e3
    print(f"cfg{cfg} n={space.ndof} m={m} steps={ns}; us")
    step = (start[1:].min(axis=1) - start[:-1].min(axis=1)) / 1e3
    print("step time (first starter to first starter): median %.2f mean %.2f" % (np.median(step), step.mean()))
    print("sweep per CTA: min %.2f  p10 %.2f  median %.2f  p90 %.2f  max %.2f" % tuple(
        np.percentile(sweep[2:], q) for q in (0, 10, 50, 90, 100)))
    smax = sweep.max(axis=1)
    smed = np.median(sweep, axis=1)
    print("per step: median-CTA sweep %.2f, slowest-CTA sweep %.2f (median over steps)" % (np.median(smed), np.median(smax)))
    exch = (start[1:].min(axis=1) - end[:-1].max(axis=1)) / 1e3
    exch_med = (np.median(start[1:], axis=1) - end[:-1].max(axis=1)) / 1e3
    print("exchange: last sweep end -> first next start %.2f, -> median next start %.2f" % (np.median(exch), np.median(exch_med)))
    spread = (start.max(axis=1) - start.min(axis=1)) / 1e3
    print("start spread across CTAs: median %.2f" % np.median(spread))
    # which CTAs are slow, consistently?
    rank = sweep[2:].mean(axis=0)
    order = np.argsort(rank)
    print("fastest CTAs (cta, smid, mean sweep):", [(int(i), int(smid[i]), round(float(rank[i]), 2)) for i in order[:8]])
    print("slowest CTAs (cta, smid, mean sweep):", [(int(i), int(smid[i]), round(float(rank[i]), 2)) for i in order[-8:]])
    for k in (0, 1, ns // 2, ns // 2 + 1, ns - 2):
        print(f"  step {k}: sweep min {sweep[k].min():.2f} med {np.median(sweep[k]):.2f} max {sweep[k].max():.2f}")
    np.save(os.path.join(ROOT, "gpurun_out", f"arn_trace_cfg{cfg}.npy"), t[:, :G])


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(tuple(sys.argv[2:]))
    else:
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        run(int(sys.argv[2]), int(sys.argv[3]))
