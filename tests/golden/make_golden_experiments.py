"""Golden CSV tables for the experiments driver, produced by running the
REFERENCE's own ``maxwelldd.experiments.run_table`` (experiments.py:391-467).

    python tests/golden/make_golden_experiments.py             # ~1 minute, writes experiments.json
    python tests/golden/make_golden_experiments.py --presets   # whole presets -> experiments_presets.json (~5 min)

Needs /root/reference (read-only) in this container; the JSON is committed so
the GPU box can compare the device path's tables against it.
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")

from maxwelldd.experiments import config_from_preset, run_table  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

TINY = {"k_list": "2", "fine_list": "4", "sub_list": "2", "coarse_list": "2", "overlap_layers": "1",
        "preconditioners": "as2,as1", "times": "false", "seed": "5"}

# name -> (preset, overrides); the shapes follow the reference's own test_experiments.py cases,
# plus one row per preconditioner family/correction and the table3/table4 settings
CASES = {
    "tiny": (None, dict(TINY)),
    "tiny_seed6": (None, {**TINY, "seed": "6"}),
    "single_subdomain": (None, {"k_list": "2", "fine_list": "2", "sub_list": "1", "coarse_rule": "none",
                                "overlap_layers": "1", "preconditioners": "as1", "times": "false"}),
    "heterogeneous": (None, {"k_list": "2", "fine_list": "4", "sub_list": "2", "coarse_list": "2",
                             "overlap_layers": "1", "preconditioners": "imphras,impras1",
                             "heterogeneity": "inclusion", "incl_box": "0,1,0,1,0.25,0.75",
                             "incl_sigma_over_k": "0.0", "bg_sigma_over_k": "1.0", "xi_prob": "zero",
                             "xi_prec": "zero", "times": "false"}),
    "maxit2": (None, {**TINY, "preconditioners": "as1", "gmres_maxit": "2", "xi_prob": "zero",
                      "xi_prec": "k2"}),
    "table6_small": ("table6", {"k_list": "3,4", "fine_list": "6,8", "sub_list": "2,2", "coarse_list": "2,2",
                                "times": "false"}),
    "table3_small": ("table3", {"k_list": "4", "fine_list": "8", "sub_list": "2", "coarse_list": "2",
                                "times": "false"}),
    "table4_small": ("table4", {"k_list": "4", "fine_list": "8", "sub_list": "2", "coarse_list": "2",
                                "times": "false"}),
    "impedance_all": (None, {"k_list": "3", "fine_list": "6", "sub_list": "2", "coarse_list": "3",
                             "overlap_layers": "1",
                             "preconditioners": "impras1,impras2,imphras,impadef1,as-h,as-adef1",
                             "times": "false", "seed": "11"}),
    # global impedance boundary (bc = impedance keeps every edge), left-preconditioned weighted
    # GMRES, the alpha/gpw geometry rules, and the hybrid correction built on A_prec
    "impedance_bc": (None, {"bc": "impedance", "k_list": "3,4", "fine_list": "6,8", "sub_list": "2,2",
                            "coarse_list": "3,2", "overlap_layers": "1",
                            "preconditioners": "as2,ras1,impras2,imphras,hras", "times": "false"}),
    "weighted_left": ("table4", {"k_list": "3,4", "gmres_side": "left", "times": "false"}),
    "alpha_rules": (None, {"k_list": "3,5", "fine_rule": "gpw", "fine_g": "12", "sub_rule": "alpha",
                           "sub_c": "0.5", "coarse_rule": "gpw", "coarse_g": "4",
                           "preconditioners": "as2,adef1,as-h", "times": "false", "initial_guess": "zero"}),
    "hybrid_prec_matrix": (None, {"k_list": "4", "fine_list": "8", "sub_list": "2", "coarse_list": "2",
                                  "hybrid_matrix": "prec", "xi_prob": "k", "xi_prec": "k2",
                                  "preconditioners": "hras,imphras,as-h", "times": "false"}),
}


# the paper-table presets (reference experiments.py:184-219), whole wavenumber lists,
# times off; a few minutes of CPU in total (run one process at a time: concurrent
# runs oversubscribe the BLAS threads and crawl)
PRESET_TABLES = ("table1", "table2", "table3", "table4", "table6", "medimax-cube")


def presets(names):
    """tests/golden/experiments_presets.json from the reference's own run_table."""
    out = {}
    for name in names:
        overrides = {"times": "false"}
        _, csv_text = run_table(config_from_preset(name, None, overrides))
        out[name] = {"preset": name, "overrides": overrides, "csv": csv_text}
        print(name, csv_text.count("\n") - 1, "rows", flush=True)
    with open(os.path.join(HERE, "experiments_presets.json"), "w", encoding="utf-8") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--presets":
        presets(sys.argv[2:] or PRESET_TABLES)
        return
    out = {}
    for name, (preset, overrides) in CASES.items():
        cfg = config_from_preset(preset, None, overrides)
        _, csv_text = run_table(cfg)
        out[name] = {"preset": preset, "overrides": overrides, "csv": csv_text}
        print(name, csv_text.count("\n") - 1, "rows")
    with open(os.path.join(HERE, "experiments.json"), "w", encoding="utf-8") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
