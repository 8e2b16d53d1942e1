"""Device-timed complex SpMV on a BASELINE config's A (CFG env): ms per call and GB/s."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1711_03789_b200 import fem, _lib

c = bench.CONFIGS[int(os.environ.get("CFG", "1"))]
space, coeffs, rhs, dec, _ = bench.build_problem(c)
A = fem.assemble(space, coeffs).A
ms = C.c_double()
_lib.check(_lib.lib.mdd_spmv_bench(_lib.get_context().handle, A.handle, 50, C.byref(ms)))
n = space.ndof
b = 20 * A.nnz + 36 * n
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("MDD_")}, "ms": ms.value,
                  "GBps": b / (ms.value * 1e-3) / 1e9}))
