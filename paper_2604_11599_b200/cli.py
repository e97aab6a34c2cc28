"""`qasm2cudaq` command line with a backend switch:

    python -m paper_2604_11599_b200.cli [--backend b200|cpu] run prog.qasm --shots 100000
    python -m paper_2604_11599_b200.cli --backend b200 validate --suite all

Every other argument is the reference CLI's own (`qasm2cudaq/cli.py:14-57`); after the
switch the reference's `cli.main` runs unchanged, its `sim.sample` / `sim.statevector` /
`sim.expval_pauli` calls (cli.py:97-112) and the validation suites (cli.py:115-128)
executing on the device.
"""

from __future__ import annotations

import argparse
import sys


def main(argv: list[str] | None = None) -> int:
    ap = argparse.ArgumentParser(add_help=False)
    ap.add_argument("--backend", choices=("b200", "cpu"), default="b200")
    ns, rest = ap.parse_known_args(sys.argv[1:] if argv is None else argv)
    from . import backend

    backend.install(ns.backend)
    from qasm2cudaq import cli

    return cli.main(rest)


if __name__ == "__main__":
    sys.exit(main())
