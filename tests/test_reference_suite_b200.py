"""the reference's OWN test suite (pkg/tests: test_sim.py,
test_acceptance.py, test_harness.py, ... -- unmodified, staged into baseline/_ref/ref_tests
by tests/ref_suite/stage_reference_tests.py) run with `qasm2cudaq.sim` switched to the
B200 backend (`-p paper_2604_11599_b200.pytest_backend`), plus the CLI switch.

The CPU tests check the switch itself (no device call); the GPU test runs the suite."""

import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "ref_tests")


def _ref_path():
    if os.path.isdir(os.path.join(REF, "qasm2cudaq")):
        return REF
    if os.path.isdir("/root/reference/pkg/src/qasm2cudaq"):
        return "/root/reference/pkg/src"
    pytest.skip("the reference package is not installed (baseline/_ref)")


def _run(code: str) -> str:
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([_ref_path(), REPO]), PYTHONDONTWRITEBYTECODE="1")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    return r.stdout


def test_switch_routes_every_reference_binding():
    out = _run(
        "import sys, qasm2cudaq, qasm2cudaq.suites, qasm2cudaq.cli\n"
        "from paper_2604_11599_b200 import backend, sim as dev\n"
        "ref = sys.modules['qasm2cudaq.sim']\n"
        "backend.install('b200', warm=False)\n"
        "import qasm2cudaq.sim as s1\n"
        "from qasm2cudaq import sim as s2, sample, StateVector\n"
        "assert s1 is dev and s2 is dev and qasm2cudaq.suites.sim is dev and qasm2cudaq.cli.sim is dev\n"
        "assert sample is dev.sample and StateVector is dev.StateVector\n"
        "from qasm2cudaq.errors import DegenerateNorm\n"
        "assert dev.DegenerateNorm is DegenerateNorm\n"
        "assert backend.current() == 'b200'\n"
        "backend.install('cpu')\n"
        "assert sys.modules['qasm2cudaq.sim'] is ref and qasm2cudaq.suites.sim is ref and qasm2cudaq.sample is ref.sample\n"
        "print('ok')\n")
    assert out.strip() == "ok"


def test_cli_switch_cpu_matches_reference_cli(tmp_path):
    prog = tmp_path / "p.qasm"
    prog.write_text('OPENQASM 3.0;\ninclude "stdgates.inc";\nqubit q;\nbit c;\nh q;\nc = measure q;\n')
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([_ref_path(), REPO]))
    args = ["run", str(prog), "--shots", "500", "--seed", "7"]
    a = subprocess.run([sys.executable, "-m", "paper_2604_11599_b200.cli", "--backend", "cpu"] + args,
                       capture_output=True, text=True, env=env, timeout=300, check=True).stdout
    b = subprocess.run([sys.executable, "-m", "qasm2cudaq.cli"] + args, capture_output=True, text=True, env=env,
                       timeout=300, check=True).stdout
    assert a == b and a.strip()


@pytest.mark.gpu
def test_cli_switch_b200_histogram_identical(tmp_path):
    """`--backend b200 run` prints exactly the reference CLI's histogram (static and
    trajectory paths)."""
    prog = tmp_path / "p.qasm"
    prog.write_text('OPENQASM 3.0;\ninclude "stdgates.inc";\nqubit[2] q;\nbit[2] c;\nh q[0];\ncx q[0], q[1];\n'
                    'c[0] = measure q[0];\nif (c[0] == 1) { x q[1]; }\nc[1] = measure q[1];\n')
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([_ref_path(), REPO]))
    args = ["run", str(prog), "--shots", "4000", "--seed", "42"]
    a = subprocess.run([sys.executable, "-m", "paper_2604_11599_b200.cli", "--backend", "b200"] + args,
                       capture_output=True, text=True, env=env, timeout=300, check=True).stdout
    b = subprocess.run([sys.executable, "-m", "qasm2cudaq.cli"] + args, capture_output=True, text=True, env=env,
                       timeout=300, check=True).stdout
    assert a == b and a.strip()


@pytest.mark.gpu
@pytest.mark.timeout(3600)
def test_reference_test_suite_on_b200(tmp_path):
    """Every test of the reference's own suite passes with the device simulator."""
    if not os.path.isdir(REF_TESTS):
        pytest.skip("reference tests not staged (tests/ref_suite/stage_reference_tests.py)")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([_ref_path(), REPO]), PYTHONDONTWRITEBYTECODE="1",
               HYPOTHESIS_STORAGE_DIRECTORY=str(tmp_path / "hyp"), QSB_BACKEND="b200")
    log = os.path.join(REPO, "gpurun_out", "reference_suite_b200.log")
    os.makedirs(os.path.dirname(log), exist_ok=True)
    r = subprocess.run([sys.executable, "-m", "pytest", "-p", "paper_2604_11599_b200.pytest_backend", REF_TESTS,
                        "-q", "-p", "no:cacheprovider", "--rootdir", str(tmp_path), "-rfE"],
                       capture_output=True, text=True, env=env, timeout=3500, cwd=str(tmp_path))
    with open(log, "w") as f:
        f.write(r.stdout + r.stderr)
    assert "qasm2cudaq.sim backend: b200" in r.stdout
    assert r.returncode == 0, r.stdout[-5000:]
