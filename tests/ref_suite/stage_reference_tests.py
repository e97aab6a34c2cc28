"""Stage the reference's own test suite next to the reference install.

    python tests/ref_suite/stage_reference_tests.py

Copies /root/reference/pkg/tests (read-only, unmodified) to baseline/_ref/ref_tests, the
git-ignored directory that holds the `pip install --target` copy of the reference and
travels to the GPU box with the snapshot.  `tests/test_reference_suite_b200.py` runs it
there with `-p paper_2604_11599_b200.pytest_backend`, i.e. the reference's tests against
the device simulator.  Nothing of it enters the repository's history.
"""

import os
import shutil
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
SRC = os.environ.get("QASM2CUDAQ_TESTS", "/root/reference/pkg/tests")
DST = os.path.join(REPO, "baseline", "_ref", "ref_tests")


def main() -> int:
    if not os.path.isdir(SRC):
        print(f"{SRC} absent: nothing to stage")
        return 0
    if os.path.isdir(DST):
        shutil.rmtree(DST)
    shutil.copytree(SRC, DST, ignore=shutil.ignore_patterns("__pycache__", ".hypothesis", "*.pyc"))
    print(f"staged {SRC} -> {DST}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
