"""python -m paper_2108_12574_b200 golden <suite ...|all> [--goldens PATH]

The reference CLI's golden subcommand (cli.py:358-361, 363-390) on the
device path; the experiment tables (spectrum / solve sweeps) are outside the
hot path."""

import argparse
import sys

from .golden import EXIT_CONFIG, EXIT_NUMERICAL, EXIT_OK, ConfigError, run_golden
from .linalg import NotPositiveDefinite


def main(argv=None) -> int:
    parser = argparse.ArgumentParser(prog="python -m paper_2108_12574_b200")
    sub = parser.add_subparsers(dest="subcommand", required=True)
    g = sub.add_parser("golden")
    g.add_argument("suites", nargs="*", help="suite names, or 'all'")
    g.add_argument("--goldens", default=None, help="goldens.json path (default: the packaged data/goldens.json)")
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return EXIT_CONFIG if exc.code not in (0, None) else EXIT_OK
    try:
        return run_golden(args.suites, args.goldens)
    except ConfigError as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    except (NotPositiveDefinite, FloatingPointError, RuntimeError) as exc:
        print(f"numerical failure: {exc}", file=sys.stderr)
        return EXIT_NUMERICAL


if __name__ == "__main__":
    sys.exit(main())
