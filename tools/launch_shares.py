"""Per-kernel shares of an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_*):

    python tools/launch_shares.py gpurun_out/launches_cfg4.csv

Prints, per kernel name, launches, total time, share of the listed time and DRAM bytes per
launch, and the totals of the bench's kernel families (precond_apply, k_arnoldi, k_spmv,
factorisation, assembly).  ncu times are cold-cache and serialised: compare SHARES."""
import csv
import re
import sys
from collections import OrderedDict, defaultdict

U = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3,
     'ms': 1.0, 'msecond': 1.0, 's': 1e3, 'second': 1e3}
rows = list(csv.reader(open(sys.argv[1], errors="replace")))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
ki, mi, vi, ui, ii = (h.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
L = OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = L.setdefault(r[ii], {"name": r[ki]})
    try:
        d[r[mi]] = float(r[vi].replace(',', '')) * U.get(r[ui], 1)
    except ValueError:
        pass


def short(n):
    n = re.sub(r"^void ", "", n)
    n = re.sub(r"\(.*$", "", n)
    return n.replace("mdd::", "")


def family(n):
    if n.startswith(("k_arnoldi", "k_drift")):
        return "k_arnoldi (+ drift panels)"
    if n.startswith(("k_solve_tma", "k_scatter_owner", "k_spmv<0", "k_spmv<false", "k_sub_add", "k_vec")):
        return "precond_apply (solve levels, scatter, R0 / R0^T)"
    if n.startswith(("k_spmv<1", "k_spmv<true")):
        return "k_spmv (complex)"
    if n.startswith(("k_front", "k_gemm", "k_gj", "k_panel", "k_update", "k_copy_b", "k_transpose", "k_symcheck",
                     "k_invert", "k_galerkin", "k_scatter_blocks", "k_rap", "k_local")):
        return "factorisation (+ coarse operator, local matrices)"
    if n.startswith(("k_assemble", "k_combine", "k_rhs")):
        return "assembly"
    return "other"


per = defaultdict(lambda: [0, 0.0, 0.0])
fam = defaultdict(lambda: [0, 0.0, 0.0])
for d in L.values():
    n = short(d["name"])
    t = d.get("gpu__time_duration.sum", 0.0)
    b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    for acc, key in ((per, n), (fam, family(n))):
        acc[key][0] += 1
        acc[key][1] += t
        acc[key][2] += b
tot = sum(v[1] for v in per.values())
print(f"# {sys.argv[1]}: {len(L)} launches, {tot:.1f} ms of kernel time listed\n")
print("| family | launches | ms | share | DRAM GB |\n|---|---|---|---|---|")
for k, v in sorted(fam.items(), key=lambda kv: -kv[1][1]):
    print(f"| {k} | {v[0]} | {v[1]:.1f} | {100 * v[1] / tot:.1f}% | {v[2] / 1e9:.2f} |")
print("\n| kernel | launches | ms | share | us / launch | DRAM MB / launch |\n|---|---|---|---|---|---|")
for k, v in sorted(per.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"| {k} | {v[0]} | {v[1]:.1f} | {100 * v[1] / tot:.1f}% | {1e3 * v[1] / v[0]:.1f} | {v[2] / v[0] / 1e6:.2f} |")
