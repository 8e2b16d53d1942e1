"""Experiments driver and CLI, modelled on the reference's
tests/test_experiments.py.  Host-only checks run without a GPU; the table
parity cases (``-m gpu``) compare the device path's CSV against tables the
reference's own run_table produced (tests/golden/experiments.json,
tests/golden/make_golden_experiments.py)."""

import json
import os

import pytest

from conftest import GOLDEN
from paper_1711_03789_b200.experiments import (
    CSV_HEADER,
    PRECONDITIONERS,
    PRESETS,
    ConfigError,
    RunRecord,
    config_from_preset,
    parse_config_file,
    resolve_geometry,
    run_table,
)

TINY = {"k_list": "2", "fine_list": "4", "sub_list": "2", "coarse_list": "2", "overlap_layers": "1",
        "preconditioners": "as2,as1", "times": "false", "seed": "5"}


def _golden():
    with open(os.path.join(GOLDEN, "experiments.json"), encoding="utf-8") as fh:
        return json.load(fh)


# ----------------------------------------------------------------- host-only
def test_unknown_key_rejected():
    with pytest.raises(ConfigError, match="unknown configuration key"):
        config_from_preset(overrides={"grid_pionts": "3"})


def test_unknown_preset_rejected():
    with pytest.raises(ConfigError, match="unknown preset"):
        config_from_preset("table99")


def test_unknown_preconditioner_rejected():
    with pytest.raises(ConfigError, match="unknown preconditioner"):
        config_from_preset(overrides={"preconditioners": "qas2"})


@pytest.mark.parametrize("key,val", [("bc", "neumann"), ("fine_rule", "x"), ("coarse_rule", "x"),
                                     ("sub_rule", "x"), ("heterogeneity", "x"), ("incl_box", "0,1"),
                                     ("times", "maybe")])
def test_bad_values_rejected(key, val):
    with pytest.raises(ConfigError):
        config_from_preset(overrides={key: val})


def test_presets_and_labels():
    for name in ("table1", "table2", "table3", "table4", "table6", "medimax-cube"):
        assert name in PRESETS
        config_from_preset(name)
    assert len(PRECONDITIONERS) == 12
    assert config_from_preset("table6").preconditioners == ["as2", "ras1", "ras2", "hras", "adef1"]
    assert config_from_preset("abs-error").k_list == [3.0, 4.0, 5.0, 6.0, 7.0, 8.0]


def test_layering_preset_file_overrides(tmp_path):
    path = tmp_path / "run.cfg"
    path.write_text("# comment\nk_list = 2,3\nseed = 9\n\noverlap_layers = 1  # trailing\n")
    raw = parse_config_file(str(path))
    assert raw == {"k_list": "2,3", "seed": "9", "overlap_layers": "1"}
    cfg = config_from_preset("table3", raw, {"seed": "4"})
    assert cfg.k_list == [2.0, 3.0]
    assert cfg.seed == 4 and cfg.overlap_layers == 1 and cfg.xi_prob == "k"
    with pytest.raises(AttributeError):
        cfg.not_a_key


def test_config_file_rejects_garbage(tmp_path):
    path = tmp_path / "bad.cfg"
    path.write_text("this is not a key value line\n")
    with pytest.raises(ConfigError, match="expected 'key = value'"):
        parse_config_file(str(path))


def test_geometry_snapping():
    cfg = config_from_preset(overrides={"k_list": "5", "fine_rule": "gpw", "fine_g": "8.4",
                                        "sub_list": "3", "coarse_list": "3"})
    geo = resolve_geometry(cfg, 5.0, 0)
    assert (geo.n, geo.p_axis, geo.n_coarse) == (6, 3, 3)  # 8.4*5/(2 pi) = 6.68 -> 6


def test_geometry_alpha_rules():
    cfg = config_from_preset(overrides={"k_list": "4", "fine_rule": "pow32", "fine_c": "1.0",
                                        "sub_rule": "alpha", "sub_alpha": "1.0", "sub_c": "0.5",
                                        "coarse_rule": "alpha", "coarse_alpha": "1.0", "coarse_c": "0.5"})
    geo = resolve_geometry(cfg, 4.0, 0)
    assert (geo.p_axis, geo.n_coarse, geo.n) == (2, 2, 8)


def test_geometry_lcm_and_short_lists():
    cfg = config_from_preset(overrides={"k_list": "4,5", "fine_list": "11", "sub_list": "2,2",
                                        "coarse_list": "3,3"})
    assert resolve_geometry(cfg, 4.0, 0).n == 12  # nearest multiple of lcm(2, 3) = 6
    with pytest.raises(ConfigError, match="fine_list list is shorter"):
        resolve_geometry(cfg, 5.0, 1)


def test_two_level_requires_coarse():
    cfg = config_from_preset(overrides={**TINY, "coarse_rule": "none", "preconditioners": "as2"})
    with pytest.raises(ConfigError, match="coarse"):
        run_table(cfg)  # raised by the geometry rule, before any device work


def test_csv_row_format():
    rec = RunRecord(k=2.0, n=316, n_sub=8, n_cs=26, xi_prob=4.0, xi_prec=4.0, preconditioner="as2",
                    iterations=19, converged=True, setup_time_s=1.5, gmres_time_s=0.25,
                    final_relative_residual=5.300782e-07, seed=5, h=0.4330127018922193,
                    h_coarse=0.8660254037844386, h_sub=0.8660254037844386, layers=1)
    row = "2,316,8,26,4,4,as2,19,1,0.000000,0.000000,5.300782e-07,5,0.4330127019,0.8660254038,0.8660254038,1"
    assert rec.csv_row(times=False) == row
    assert rec.csv_row().split(",")[9:11] == ["1.500000", "0.250000"]
    assert _golden()["tiny"]["csv"].split("\n")[1] == row
    assert _golden()["tiny"]["csv"].split("\n")[0] == CSV_HEADER


def test_cli_errors(capsys):
    from paper_1711_03789_b200.cli import main

    assert main(["run", "--set", "bogus_key=1"]) == 2
    assert "unknown configuration key" in capsys.readouterr().err
    assert main(["run", "--set", "novalue"]) == 2
    assert "--set expects key=value" in capsys.readouterr().err
    assert main(["fov", "--identity"]) == 2
    assert "outside the accelerated path" in capsys.readouterr().err


def test_cli_mesh_info(capsys):
    from paper_1711_03789_b200.cli import main

    assert main(["mesh-info", "--n", "1"]) == 0
    assert "vertices=8 tets=6 edges=19" in capsys.readouterr().out


# ---------------------------------------------------------- device parity
def _rows(csv_text):
    return [line.split(",") for line in csv_text.strip().split("\n")[1:]]


def _assert_tables_match(ours, ref):
    a, b = _rows(ours), _rows(ref)
    assert len(a) == len(b)
    for ra, rb in zip(a, b):
        # geometry, shifts, label, seed, mesh sizes: identical bytes
        for i in (0, 1, 2, 3, 4, 5, 6, 12, 13, 14, 15, 16):
            assert ra[i] == rb[i], (i, ra, rb)
        assert abs(int(ra[7]) - int(rb[7])) <= 1, (ra, rb)  # iterations within +-1 (north_star)
        assert ra[8] == rb[8], (ra, rb)
        if ra[7] == rb[7]:
            fa, fb = float(ra[11]), float(rb[11])
            # the final |r|/|b| is not a parity bar (iterations +-1 and the solution are):
            # in slowly converging rows (table2, minimal overlap) the last residual moves
            # by ~1% with rounding-level changes in the preconditioner (the reference's
            # partial-pivoting dense LU vs the unpivoted multifrontal factors)
            assert abs(fa - fb) <= 2e-2 * abs(fb) + 1e-11, (ra, rb)


@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(_golden()))
def test_run_table_matches_reference(case):
    g = _golden()[case]
    cfg = config_from_preset(g["preset"], None, g["overrides"])
    records, csv_text = run_table(cfg)
    assert csv_text.startswith(CSV_HEADER + "\n")
    _assert_tables_match(csv_text, g["csv"])
    assert len(records) == len(_rows(g["csv"]))


@pytest.mark.gpu
def test_run_table_deterministic_and_file(tmp_path):
    cfg = config_from_preset(overrides=dict(TINY))
    _, first = run_table(cfg)
    _, again = run_table(cfg)
    assert first == again  # byte-identical rerun
    out = tmp_path / "rows.csv"
    run_table(config_from_preset(overrides={**TINY, "out": str(out)}))
    data = out.read_bytes()
    assert b"\r" not in data and data.decode("utf-8") == first
    _, seed6 = run_table(config_from_preset(overrides={**TINY, "seed": "6"}))
    assert seed6 != first


@pytest.mark.gpu
def test_sizing_refusal():
    with pytest.raises(ConfigError, match="infeasible"):
        run_table(config_from_preset(overrides={**TINY, "lu_cap": "10"}))


@pytest.mark.gpu
def test_cli_run(tmp_path, capsys):
    from paper_1711_03789_b200.cli import main

    cfgfile = tmp_path / "exp.cfg"
    cfgfile.write_text("k_list = 2\nfine_list = 4\nsub_list = 2\ncoarse_list = 2\n"
                       "overlap_layers = 1\npreconditioners = as2\ntimes = false\n")
    out = tmp_path / "exp.csv"
    rc = main(["run", "--config", str(cfgfile), "--out", str(out), "--seed", "5",
               "--set", "preconditioners=as1"])
    assert rc == 0
    text = out.read_text()
    assert text.startswith(CSV_HEADER) and ",as1," in text and ",as2," not in text
    _assert_tables_match(text, "\n".join(_golden()["tiny"]["csv"].split("\n")[i] for i in (0, 2)))
    assert "iters=" in capsys.readouterr().out


def _preset_tables():
    path = os.path.join(GOLDEN, "experiments_presets.json")
    if not os.path.exists(path):
        return {}
    with open(path, encoding="utf-8") as fh:
        return json.load(fh)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(_preset_tables()))
def test_paper_preset_matches_reference(name):
    """A whole paper-table preset (reference experiments.py:184-219: every
    wavenumber and preconditioner of the table) through the device path against
    the reference's own run_table output."""
    g = _preset_tables()[name]
    _, ours = run_table(config_from_preset(g["preset"], None, g["overrides"]))
    _assert_tables_match(ours, g["csv"])
