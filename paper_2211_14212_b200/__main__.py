"""``python -m paper_2211_14212_b200 {simulate,reconstruct,compare} ...`` -- the reference's
command-line front end (tools/ctkrylov_main.cpp) over pipeline.py: the same subcommands,
flags, override order and exit codes (0 ok; 1 numerical failure or other error; 2 usage,
parameter, geometry, dimension or degenerate-input error)."""
from __future__ import annotations

import argparse
import sys

from .api import CtkError, DegenerateInputError, DimensionError, GeometryError, NumericalError, ParameterError
from .config import RunConfig, apply_override, load_config


def _add_common(sub, with_projections: bool) -> None:
    """ctkrylov_main.cpp:20-30."""
    sub.add_argument("--config", default="", help="flat key = value config file")
    sub.add_argument("--output", default="", help="output directory")
    sub.add_argument("--precision", default="", choices=["", "single", "double"], help="working precision")
    sub.add_argument("--threads", type=int, default=-1, help="operator thread count (0 = library default)")
    sub.add_argument("--seed", type=int, default=-1, help="noise RNG seed (overrides config)")
    sub.add_argument("--set", action="append", default=[], dest="overrides",
                     help="extra key=value override (repeatable)")
    if with_projections:
        sub.add_argument("projections", nargs="?", default="", help="projection data file (raw + .hdr)")


def build_config(a) -> RunConfig:
    """ctkrylov_main.cpp:32-47: config file, then flags, then --set overrides in order."""
    cfg = load_config(a.config) if a.config else RunConfig()
    if a.output:
        cfg.output_dir = a.output
    if a.precision:
        cfg.precision = a.precision
    if getattr(a, "projections", ""):
        cfg.projections = a.projections
    if a.threads >= 0:
        cfg.threads = a.threads
    if a.seed >= 0:
        cfg.seed = a.seed
    for kv in a.overrides:
        eq = kv.find("=")
        if eq < 0:
            raise ParameterError(f"--set expects key=value, got '{kv}'")
        apply_override(cfg, kv[:eq], kv[eq + 1:])
    return cfg


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="ctkrylov",
                                 description="Matrix-free Krylov reconstruction pipeline for simulated CT data")
    subs = ap.add_subparsers(dest="cmd", required=True)
    _add_common(subs.add_parser("simulate", help="generate phantom and measurements"), False)
    _add_common(subs.add_parser("reconstruct", help="run one solver on projection data"), True)
    _add_common(subs.add_parser("compare", help="run several solvers on identical data"), True)
    a = ap.parse_args(argv)  # usage errors exit 2
    from . import pipeline

    try:
        run = {"simulate": pipeline.run_simulate, "reconstruct": pipeline.run_reconstruct,
               "compare": pipeline.run_compare}[a.cmd]
        run(build_config(a))
        return 0
    except NumericalError as e:
        print(f"numerical failure: {e} (iteration {e.iteration})", file=sys.stderr)
        return 1
    except (ParameterError, GeometryError, DimensionError, DegenerateInputError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except (CtkError, Exception) as e:  # noqa: B014 -- everything else, like std::exception
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
