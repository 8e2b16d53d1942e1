"""Run paper-table presets through the device path (experiments.run_table) and write their CSVs.

    python tools/run_tables.py table1 table6      # -> gpurun_out/tables/<preset>.csv (+ _times.csv)
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1711_03789_b200.experiments import config_from_preset, run_table  # noqa: E402

out = os.path.join(ROOT, "gpurun_out", "tables")
os.makedirs(out, exist_ok=True)
for name in sys.argv[1:]:
    for times in ("false", "true"):
        t0 = time.time()
        _, csv = run_table(config_from_preset(name, None, {"times": times}))
        suffix = "" if times == "false" else "_times"
        with open(os.path.join(out, f"{name}{suffix}.csv"), "w", encoding="utf-8", newline="\n") as fh:
            fh.write(csv)
        print(name, times, f"{time.time() - t0:.1f}s", flush=True)
