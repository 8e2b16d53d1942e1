"""Command line for the device path (reference ``maxwelldd.cli``,
/root/reference/pkg/src/maxwelldd/cli.py:26-183).

Subcommands on the hot path:
  run         paper-table sweep from a preset and/or key-value file (cli.py:26-64)
  mesh-info   entity counts for a cube mesh (cli.py:67-71)

The reference's analysis subcommands (coercivity, fov, abs-error) study the
operator's numerical range with dense eigen-solvers; they are outside the
accelerated path and exit with status 2 and a message.
Exit status 2 on configuration errors, as in the reference (cli.py:174-180).

    python -m paper_1711_03789_b200.cli run --preset table1 --set lu_cap=0
"""

from __future__ import annotations

import argparse
import sys

from .experiments import ConfigError, config_from_preset, parse_config_file, run_table
from .mesh import build_cube_mesh

__all__ = ["main", "build_parser"]


def _overrides(args) -> dict:
    out = {}
    for item in args.set or []:
        key, sep, val = item.partition("=")
        if not sep:
            raise ConfigError(f"--set expects key=value, got {item!r}")
        out[key.strip()] = val.strip()
    if args.out:
        out["out"] = args.out
    if args.seed is not None:
        out["seed"] = str(args.seed)
    return out


def _cmd_run(args) -> int:
    if args.preset == "abs-error":
        raise ConfigError("preset 'abs-error' is an analysis sweep outside the accelerated path")
    file_raw = parse_config_file(args.config) if args.config else None
    cfg = config_from_preset(args.preset, file_raw, _overrides(args))
    records, csv_text = run_table(cfg)
    for rec in records:
        print(f"k={rec.k:g} {rec.preconditioner:>9s} n={rec.n} N={rec.n_sub} "
              f"ncs={rec.n_cs} iters={rec.iterations} [{'ok' if rec.converged else 'MAXIT'}]")
    if cfg.out:
        print(f"wrote {cfg.out}")
    elif not args.out:
        sys.stdout.write(csv_text)
    return 0


def _cmd_mesh_info(args) -> int:
    mesh = build_cube_mesh(args.n)
    print(f"vertices={mesh.n_vertices} tets={mesh.n_tets} edges={mesh.n_edges}")
    print(f"boundary_faces={mesh.boundary_faces.shape[0]} h={mesh.h:.6g}")
    return 0


_ANALYSIS = ("coercivity", "fov", "abs-error")


def _cmd_analysis(args) -> int:
    raise ConfigError(f"'{args.cmd}' is an operator-analysis command outside the accelerated path "
                      "(use the reference package)")


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_1711_03789_b200")
    sub = parser.add_subparsers(dest="cmd", required=True)

    run = sub.add_parser("run", help="run an experiment sweep on the GPU")
    run.add_argument("--config", help="key-value configuration file")
    run.add_argument("--preset", help="named preset (table1..table6, medimax-cube)")
    run.add_argument("--out", help="CSV output path")
    run.add_argument("--seed", type=int, help="seed override")
    run.add_argument("--set", action="append", metavar="KEY=VALUE", help="config override")
    run.set_defaults(func=_cmd_run)

    mesh = sub.add_parser("mesh-info", help="cube mesh entity counts")
    mesh.add_argument("--n", type=int, required=True)
    mesh.set_defaults(func=_cmd_mesh_info)

    for name in _ANALYSIS:
        sub.add_parser(name, help="(reference analysis command; not on the device path)").set_defaults(
            func=_cmd_analysis)
    return parser


def main(argv=None) -> int:
    parser = build_parser()
    args, extra = parser.parse_known_args(argv)
    if extra and args.cmd not in _ANALYSIS:
        parser.error(f"unrecognized arguments: {' '.join(extra)}")
    try:
        return args.func(args)
    except ValueError as exc:  # ConfigError, FemError, MeshError, DecompositionError
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
