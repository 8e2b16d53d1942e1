"""Per-family DRAM bytes per launch from an ncu launch list of one bench step
(run with MDD_NO_GRAPH=1 so the GMRES loop is host-driven and visible):

    MDD_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none -c N --csv python bench.py --steps 1 --warmup 0 --no-cpu > launches.csv

    python tools/traffic_from_ncu.py launches.csv cfg1 ITERATIONS [profiles/traffic.json]

Families per GMRES iteration: precond_apply (k_solve_tma, k_scatter_owner,
real SpMV k_spmv<0,*> for R0 / R0^T, k_sub_add), k_spmv (complex SpMV
k_spmv<1,*>), k_arnoldi.  Bytes are averaged over the GMRES phase's launches
(the first complete GMRES solve in the list)."""
import csv, json, os, sys
from collections import OrderedDict

U = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0,
     'ms': 1e3, 'msecond': 1e3}
path, cfg, its = sys.argv[1], sys.argv[2], int(sys.argv[3])
out = sys.argv[4] if len(sys.argv) > 4 else None
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
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
launches = list(L.values())
isfac = [d["name"].startswith(("k_update", "k_pack_up", "k_front_init")) for d in launches]
first_arn = next(k for k, d in enumerate(launches) if d["name"].startswith("void k_arnoldi"))
a = max((k for k in range(first_arn) if isfac[k]), default=-1) + 1
b = next((k for k in range(first_arn, len(launches)) if isfac[k]), len(launches))
gm = launches[a:b]  # the first complete GMRES solve
n_arn = sum(d["name"].startswith("void k_arnoldi") for d in gm)
if n_arn != its:
    sys.exit(f"launch list covers {n_arn} Arnoldi launches in the first solve, expected {its}")


def fam(name):
    if name.startswith("void k_arnoldi"):
        return "k_arnoldi"
    if name.startswith("void k_spmv<1") or name.startswith("void k_spmv<true"):
        return "k_spmv"
    if name.startswith(("void mdd::k_solve_tma", "void k_solve_tma", "k_scatter_owner", "void k_spmv<0", "k_sub_add")):
        return "precond_apply"
    return None


acc = {}
for d in gm:
    f = fam(d["name"])
    if f:
        b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        acc.setdefault(f, [0.0, 0.0, 0])
        acc[f][0] += b
        acc[f][1] += d.get("gpu__time_duration.sum", 0)
        acc[f][2] += 1
res = {f: v[0] / its for f, v in acc.items()}
print(json.dumps({cfg: res, "launch_counts": {f: v[2] for f, v in acc.items()},
                  "us_per_iteration": {f: v[1] / its for f, v in acc.items()}}, indent=1))
if out:
    d = json.load(open(out)) if os.path.exists(out) else {}
    d[cfg] = res
    json.dump(d, open(out, "w"), indent=1)
