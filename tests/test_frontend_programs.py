"""OpenQASM 3 programs lowered by the reference's own frontend -- bounded `for` loops
(unrolled statically by sema.py:640-660) with mid-circuit measurement, feedforward,
resets, nested if/else and register predicates inside -- replayed against the
reference simulator's recorded results (tests/golden/make_frontend_goldens.py).

CPU: the oracle reproduces the recorded histograms, keys, traces and states exactly.
GPU: the device reproduces histograms and per-shot keys / traces bit-exactly and final
states within 1e-10, through both engines.
"""

import contextlib

import numpy as np
import pytest

from oracle import sim_port as P
from paper_2604_11599_b200 import _lib, ir, sim


def cvec(d):
    return np.array(d["re"]) + 1j * np.array(d["im"])


def test_frontend_programs_oracle(golden):
    cases = golden("frontend.json")
    assert len(cases) >= 4
    for name, case in cases.items():
        b = ir.bind(ir.kernel_from_json(case["kernel"]), [])
        assert P.is_dynamic(b.kernel), name
        assert P.sample_counts(b, 1024, 1234) == case["hist_1024_seed1234"], name
        for rec in case["shots"]:
            trace = []
            store, st = P.trajectory(b, P.PortRng.for_shot(1234, rec["shot"]), trace)
            assert store.key() == rec["key"], (name, rec["shot"])
            assert [[t[2], t[1]] for t in trace] == rec["trace"]
            np.testing.assert_array_equal(st.amps, cvec(rec["state"]))


@contextlib.contextmanager
def _engine(which):
    ctx = _lib.context()
    ctx.set_option("engine", {"resident": 0, "stream": 1}[which])
    try:
        yield
    finally:
        ctx.set_option("engine", -1)


@pytest.mark.gpu
@pytest.mark.parametrize("eng", ["resident", "stream"])
def test_frontend_programs_device(golden, eng):
    with _engine(eng):
        for name, case in golden("frontend.json").items():
            b = ir.bind(ir.kernel_from_json(case["kernel"]), [])
            assert sim.sample(b, 1024, 1234).counts == case["hist_1024_seed1234"], (name, eng)
            for rec in case["shots"]:
                trace = []
                store, st = sim.run_trajectory(b, sim.RngStream.for_shot(1234, rec["shot"]), trace)
                assert store.key() == rec["key"], (name, rec["shot"])
                assert [[t[2], t[1]] for t in trace] == rec["trace"]
                err = np.max(np.abs(st.amps - cvec(rec["state"])))
                assert err <= 1e-10, (name, rec["shot"], err)
