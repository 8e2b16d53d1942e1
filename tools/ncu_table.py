"""Summarise an ncu --csv metrics log: per launch time, DRAM bytes, GB/s."""
import csv, sys
from collections import OrderedDict
U = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3,
     'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, '': 1}
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, mi, ui, ii, mn, gi = (h.index(x) for x in ('Kernel Name', 'Metric Value', 'Metric Unit', 'ID', 'Metric Name', 'Grid Size'))
L = OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= mi:
        continue
    d = L.setdefault((r[ii], r[ki].split('(')[0], r[gi]), {})
    try:
        d[r[mn]] = float(r[mi].replace(',', '')) * U.get(r[ui], 1)
    except ValueError:
        pass
tt = tb = 0
for (i, k, g), d in L.items():
    t = d.get('gpu__time_duration.sum', 0)
    b = d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0)
    tt += t; tb += b
    print(f"{i:>5} {k:26s} grid={g:14s} t={t:9.1f}us dram={b/1e6:8.1f}MB {b/t/1e3 if t else 0:7.1f} GB/s")
print(f"total {tt:.1f} us, {tb/1e9:.3f} GB, {tb/tt/1e3:.1f} GB/s")
