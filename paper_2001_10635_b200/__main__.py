"""Command-line front end (the reference's ``ivreach run`` / ``ivreach config``):

    python -m paper_2001_10635_b200 run CONFIG [--mode exact|fast] [--workers N]
    python -m paper_2001_10635_b200 config CONFIG     # resolved config, serialize_config

``run`` parses the reference's .cfg format, integrates on the GPU and writes
``<output>.json|csv`` and ``<output>.report.json`` in the reference's formats.
"""
from __future__ import annotations

import argparse
import sys


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2001_10635_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run", help="run a reachability config on the GPU")
    r.add_argument("config")
    r.add_argument("--mode", choices=["exact", "fast"], default="exact")
    r.add_argument("--workers", type=int, default=None, help="override the config's workers (shard lanes)")
    c = sub.add_parser("config", help="print the fully resolved config")
    c.add_argument("config")
    args = ap.parse_args(argv)

    from . import config as CF
    from .reach import set_default_mode

    try:
        cfg = CF.parse_config_file(args.config)
        if args.cmd == "config":
            sys.stdout.write(CF.serialize_config(cfg))
            return 0
        if args.workers is not None:
            cfg.workers = args.workers
        set_default_mode(args.mode)
        out = CF.run_config(cfg)
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except RuntimeError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    rep = out.tube.report
    print(f"{rep.method}: n={rep.n} steps={rep.steps} boxes={len(out.tube.entries)} "
          f"integration {rep.phases.integration_s:.6f} s -> {out.tube_path}, {out.report_path}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
