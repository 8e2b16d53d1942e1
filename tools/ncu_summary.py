"""Key metrics of an ncu --set full report (run here, no GPU needed)."""
import csv, subprocess, sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Grid Size", "Block Size", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Warp Cycles Per Issued Instruction", "Executed Ipc Active"]


def summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    res = {}
    kname = None
    for r in rows[1:]:
        kname = r[ki]
        if r[mi] in WANT and r[mi] not in res:
            res[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    hh, vals = rr[0], rr[2] if len(rr) > 2 else []
    stalls = {}
    for i, name in enumerate(hh):
        if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("_not_issued"):
            try:
                stalls[name] = float(vals[i])
            except (ValueError, IndexError):
                pass
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        if k in hh:
            res[k] = f"{vals[hh.index(k)]} {rr[1][hh.index(k)]}"
    tot = sum(stalls.values()) or 1.0
    top = [(n, 100.0 * v / tot) for n, v in sorted(stalls.items(), key=lambda x: -x[1])[:6]]
    return kname, res, top


if __name__ == "__main__":
    for p in sys.argv[1:]:
        k, res, top = summary(p)
        print(f"## {p.split('/')[-1]} — `{k.split('(')[0]}`")
        for kk, v in res.items():
            print(f"- {kk}: {v}")
        print("- top stall reasons (% of PC samples):",
              ", ".join(f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')} {v:.0f}%" for n, v in top))
        print()
