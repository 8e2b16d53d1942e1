"""Hot SASS lines of an ncu report (stall samples / executed instructions)."""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; data = rows[2:]
si = h.index("Warp Stall Sampling (All Samples)"); ii = h.index("Instructions Executed")
num = lambda x: int(x) if x.isdigit() else 0
ts = sum(num(r[si]) for r in data); ti = sum(num(r[ii]) for r in data)
print(f"samples {ts} warp-instructions {ti}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for k, r in enumerate(data):
    if num(r[si]) >= ts * 0.008 or num(r[ii]) >= ti * 0.02:
        print(f"{num(r[si]):7d} {num(r[ii]):10d} {r[0][-5:]} {r[1][:80]}")
