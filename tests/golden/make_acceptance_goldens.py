"""Record every simulator call the reference's acceptance suites make, with the
reference's own results, so the GPU backend can replay them.

Run in the build container (where `/root/reference` exists):

    python tests/golden/make_acceptance_goldens.py

The reference's suites (`suites.py`: conditional reset, teleportation, Clifford
differential, compile-once VQE, algorithms -- the programs behind acceptance
criteria 1-5 and 7 of `tests/test_acceptance.py`) run unchanged, on the reference CPU
simulator, with `qasm2cudaq.sim.sample / statevector / expval_pauli` wrapped (in this
process only) by recorders.  Each call is stored as the lowered Kernel IR (mirror
JSON), its bound values and arguments, and the reference result: histograms exactly,
states up to 10 qubits as amplitudes (larger ones as norm and |<0|psi>|^2),
expectation values as floats (repr, exact).  `tests/test_acceptance_replay.py`
replays the calls through the B200 backend.  Nothing is written into the reference.
"""

from __future__ import annotations

import json
import os
import sys

sys.dont_write_bytecode = True
REF = os.environ.get("QASM2CUDAQ_REF", "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
from qasm2cudaq import sim as rsim  # noqa: E402
from qasm2cudaq import suites as rsuites  # noqa: E402

from paper_2604_11599_b200 import ir  # noqa: E402

MAX_STATE_QUBITS = 10


def cvec(a) -> dict:
    a = np.asarray(a, dtype=np.complex128)
    return {"re": [float(x) for x in a.real], "im": [float(x) for x in a.imag]}


class Recorder:
    def __init__(self):
        self.calls: list[dict] = []
        self.kernels: dict[int, int] = {}  # id(kernel) -> index in self.kernel_json
        self.kernel_json: list[dict] = []
        self.alive: list = []  # keeps recorded kernels / states alive: ids must not be reused
        self.state_ids: dict[int, int] = {}  # id(StateVector) -> call index
        self.suite = ""
        self._sample, self._statevector, self._expval = rsim.sample, rsim.statevector, rsim.expval_pauli

    def kernel_index(self, kernel) -> int:
        idx = self.kernels.get(id(kernel))
        if idx is None:
            idx = len(self.kernel_json)
            self.kernels[id(kernel)] = idx
            self.kernel_json.append(ir.kernel_to_json(kernel))
            self.alive.append(kernel)
        return idx

    def sample(self, bound, shots, seed, workers=1):
        hist = self._sample(bound, shots, seed, workers)
        self.calls.append({"suite": self.suite, "call": "sample", "kernel": self.kernel_index(bound.kernel),
                           "values": [float(v) for v in bound.values], "shots": shots, "seed": seed,
                           "workers": workers, "counts": dict(hist.counts)})
        return hist

    def statevector(self, bound):
        st = self._statevector(bound)
        rec = {"suite": self.suite, "call": "statevector", "kernel": self.kernel_index(bound.kernel),
               "values": [float(v) for v in bound.values], "n": st.n}
        amps = np.asarray(st.amps)
        if st.n <= MAX_STATE_QUBITS:
            rec["state"] = cvec(amps)
        else:
            rec["norm"] = float(np.linalg.norm(amps))
            rec["p0"] = float(abs(amps[0]) ** 2)
        self.state_ids[id(st)] = len(self.calls)
        self.alive.append(st)
        self.calls.append(rec)
        return st

    def expval(self, state, pauli):
        val = self._expval(state, pauli)
        self.calls.append({"suite": self.suite, "call": "expval_pauli", "state_call": self.state_ids.get(id(state)),
                           "pauli": pauli, "value": float(val)})
        return val


def main():
    rec = Recorder()
    rsim.sample, rsim.statevector, rsim.expval_pauli = rec.sample, rec.statevector, rec.expval
    reports = {}
    try:
        for name, fn in [
            ("conditional_reset", lambda: rsuites.suite_conditional_reset(shots=1000, seed=1234)),
            ("teleport", lambda: rsuites.suite_teleport(shots=1000, seed=1234)),
            ("clifford", lambda: rsuites.suite_clifford_differential(case_count=16, seed=1234, uncompute_cases=4,
                                                                    smoke_cases=1)),
            ("vqe", lambda: rsuites.suite_vqe(iterations=8, seed=1234)),
            ("algorithms", lambda: rsuites.suite_algorithms(seed=1234, bv_cases=6)),
        ]:
            rec.suite = name
            rep = fn()
            reports[name] = {"passed": bool(rep.passed), "cases": [[c.name, bool(c.passed)] for c in rep.cases]}
    finally:
        rsim.sample, rsim.statevector, rsim.expval_pauli = rec._sample, rec._statevector, rec._expval
    out = {"kernels": rec.kernel_json, "calls": rec.calls, "reports": reports}
    path = os.path.join(HERE, "acceptance.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(f"wrote acceptance.json: {len(rec.calls)} calls, {len(rec.kernel_json)} kernels, "
          f"{os.path.getsize(path) / 1024:.1f} KiB; suites passed: {[k for k, v in reports.items() if v['passed']]}")


if __name__ == "__main__":
    main()
