"""pytest plugin: run a qasm2cudaq test suite against the B200 backend, unmodified.

    pytest -p paper_2604_11599_b200.pytest_backend <qasm2cudaq's tests/>

Installs the backend switch (`backend.install`, QSB_BACKEND=b200 by default, =cpu for
the reference simulator) when the plugin is imported -- before the suite's conftest
imports `qasm2cudaq` -- so every `qasm2cudaq.sim` reference in the tests and in the
suites they drive (`suites.py`) is the device simulator.
"""

from __future__ import annotations

import os

from . import backend

backend.install(os.environ.get("QSB_BACKEND", "b200"))


def pytest_report_header(config):
    return f"qasm2cudaq.sim backend: {backend.current()}"


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    terminalreporter.write_line(f"qasm2cudaq.sim backend: {backend.current()}")
