"""Diagnostic: N loopback ranks on one GPU with per-rank progress prints and a stack dump on stall."""
import faulthandler, os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from paper_1711_03789_b200 import KrylovConfig, _lib, gmres, precond
from paper_1711_03789_b200.distributed import Communicator, LoopbackGroup, setup_sharded
from test_gpu_distributed import _case_objects

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
faulthandler.dump_traceback_later(90, exit=True)
prob, d = _case_objects()
spec = precond.PreconditionerSpec("as", "two", "additive", xi_prec=4.0)
cfg = KrylovConfig(tol=1e-8, maxit=80, orthogonalization="cgs2")
v = np.random.default_rng(7).standard_normal(prob.space.ndof) * (1 - 1j)
_lib.get_context().synchronize()
group = LoopbackGroup(N)
t0 = time.time()
def log(*a): print(f"[{time.time()-t0:7.2f}]", *a, flush=True)
def rank_main(r):
    with _lib.use_context(_lib.Context(0)) as ctx:
        log(r, "objects"); pr, dr = _case_objects()
        log(r, "setup"); st = setup_sharded(pr, dr, spec, comm=Communicator(ctx, loopback=(group, r)))
        log(r, "apply"); st.apply(v)
        log(r, "gmres"); rep = gmres(pr.A, pr.rhs, precond=st, config=cfg)
        log(r, "done", rep.iterations)
th = [threading.Thread(target=rank_main, args=(r,)) for r in range(N)]
[t.start() for t in th]; [t.join() for t in th]
log("all done")
