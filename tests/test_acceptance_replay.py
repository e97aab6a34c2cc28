"""Replay of every simulator call the reference's acceptance suites make
(`suites.py`: conditional reset, teleportation, Clifford differential, compile-once
VQE, algorithms -- acceptance criteria 1-5), recorded with the reference's results by
`tests/golden/make_acceptance_goldens.py`.

GPU: every call through the B200 backend -- histograms bit-exact, states within 1e-10,
expectation values within 1e-10.  CPU: the oracle reproduces the recorded states and a
sample of the histograms exactly (pins the fixture)."""

import numpy as np
import pytest

from oracle import sim_port as P
from paper_2604_11599_b200 import ir, sim


def _load(golden):
    g = golden("acceptance.json")
    kernels = [ir.kernel_from_json(k) for k in g["kernels"]]
    return g, kernels


def _state(rec):
    return np.array(rec["state"]["re"]) + 1j * np.array(rec["state"]["im"])


def test_reference_suites_passed_when_recorded(golden):
    g, _ = _load(golden)
    assert set(g["reports"]) == {"conditional_reset", "teleport", "clifford", "vqe", "algorithms"}
    assert all(r["passed"] for r in g["reports"].values())


def test_oracle_reproduces_recorded_calls(golden):
    g, kernels = _load(golden)
    checked_states = checked_hists = 0
    for rec in g["calls"]:
        b = ir.bind(kernels[rec["kernel"]], rec["values"]) if "kernel" in rec else None
        if rec["call"] == "statevector" and "state" in rec and rec["n"] <= 8:
            np.testing.assert_array_equal(P.final_state(b).amps, _state(rec))
            checked_states += 1
        elif rec["call"] == "sample" and rec["shots"] <= 1000 and checked_hists < 3:
            assert P.sample_counts(b, rec["shots"], rec["seed"]) == rec["counts"]
            checked_hists += 1
    assert checked_states > 5 and checked_hists == 3


@pytest.mark.gpu
@pytest.mark.parametrize("suite", ["conditional_reset", "teleport", "clifford", "vqe", "algorithms"])
def test_acceptance_calls_on_device(golden, suite):
    g, kernels = _load(golden)
    states = {}
    n_calls = 0
    for i, rec in enumerate(g["calls"]):
        if rec["suite"] != suite:
            continue
        n_calls += 1
        if rec["call"] == "sample":
            b = ir.bind(kernels[rec["kernel"]], rec["values"])
            got = sim.sample(b, rec["shots"], rec["seed"], workers=rec["workers"]).counts
            assert got == rec["counts"], i
        elif rec["call"] == "statevector":
            st = sim.statevector(ir.bind(kernels[rec["kernel"]], rec["values"]))
            states[i] = st
            a = st.amps
            if "state" in rec:
                assert np.max(np.abs(a - _state(rec))) <= 1e-10, i
            else:
                assert abs(np.linalg.norm(a) - rec["norm"]) <= 1e-10, i
                assert abs(abs(a[0]) ** 2 - rec["p0"]) <= 1e-10, i
        else:
            st = states[rec["state_call"]]
            assert abs(sim.expval_pauli(st, rec["pauli"]) - rec["value"]) <= 1e-10, i
    assert n_calls > 0
