"""Pin the CPU oracle (oracle/sim_port.py) to the REAL reference's outputs.

The fixtures were produced by tests/golden/make_goldens.py running
/root/reference/pkg/src/qasm2cudaq/sim.py.  Everything here is exact equality:
RNG words, uniforms, histograms, per-shot keys, executed-branch traces and
amplitudes (the port follows the reference's numpy call sequence, so rounding
is identical).
"""

import numpy as np
import pytest

from oracle import sim_port as P
from paper_2604_11599_b200 import ir


def cvec(d):
    return np.array(d["re"]) + 1j * np.array(d["im"])


def test_rng_known_answers(golden):
    g = golden("rng.json")
    r = P.PortRng(42)
    assert [str(x) for x in r.s] == g["seed42_state"]
    assert [str(r.next_u64()) for _ in range(8)] == g["seed42_words"]
    for case in g["for_shot"]:
        r = P.PortRng.for_shot(case["seed"], case["shot"])
        assert [str(x) for x in r.s] == case["state"]
        assert [r.uniform() for _ in range(6)] == case["uniforms"]


def _check_record(bound, rec, seed):
    if "error" in rec:
        with pytest.raises(P.DegenerateBranch):
            P.trajectory(bound, P.PredrawnStream(rec["uniforms"]) if seed is None else P.PortRng.for_shot(seed, rec["shot"]))
        return
    rng = P.PredrawnStream(rec["uniforms"] + [0.5]) if seed is None else P.PortRng.for_shot(seed, rec["shot"])
    trace = []
    store, st = P.trajectory(bound, rng, trace)
    assert store.key() == rec["key"]
    assert [[t[2], t[1]] for t in trace] == rec["trace"]
    if "state" in rec:
        np.testing.assert_array_equal(st.amps, cvec(rec["state"]))


def test_ff_suite(golden):
    for name, case in golden("ff_suite.json").items():
        k = ir.kernel_from_json(case["kernel"])
        b = ir.bind(k, [])
        assert P.sample_counts(b, 1024, 1234) == case["hist_1024_seed1234"], name
        for rec in case["shots"]:
            _check_record(b, rec, 1234)


def test_static_states_and_expval(golden):
    for case in golden("static.json"):
        k = ir.kernel_from_json(case["kernel"])
        st = P.final_state(ir.bind(k, case["values"]))
        np.testing.assert_array_equal(st.amps, cvec(case["state"]))
        assert st.norm() == case["norm"]
        for word, val in case["expval"]:
            assert P.pauli_expectation(st, word) == val


def test_static_sampling(golden):
    for case in golden("static_sampling.json"):
        b = ir.bind(ir.kernel_from_json(case["kernel"]), [])
        assert not P.is_dynamic(b.kernel)
        assert P.sample_counts(b, case["shots"], case["seed"]) == case["counts"]


def test_dynamic(golden):
    for case in golden("dynamic.json"):
        b = ir.bind(ir.kernel_from_json(case["kernel"]), [])
        assert P.is_dynamic(b.kernel) == case["needs_trajectories"]
        if case["counts_512"] is not None:
            assert P.sample_counts(b, 512, case["seed"]) == case["counts_512"]
        for rec in case["shots"]:
            _check_record(b, rec, case["seed"])


def test_predrawn_streams(golden):
    for case in golden("predrawn.json"):
        b = ir.bind(ir.kernel_from_json(case["kernel"]), [])
        rec = dict(case["record"])
        rec["uniforms"] = case["values"]
        if "error" in case["record"]:
            with pytest.raises(P.DegenerateBranch):
                P.trajectory(b, P.PredrawnStream(case["values"]))
            continue
        _check_record(b, rec, None)


def test_twins(golden):
    t = golden("twins.json")
    b = ir.bind(ir.kernel_from_json(t["dyn8"]["kernel"]), [])
    assert P.sample_counts(b, 1024, 1234) == t["dyn8"]["counts_1024"]
    for rec in t["dyn8"]["shots"][:16]:
        _check_record(b, rec, 1234)
    b = ir.bind(ir.kernel_from_json(t["rdc10"]["kernel"]), [])
    for rec in t["rdc10"]["shots"]:
        _check_record(b, rec, 1234)
    v = t["vqe6"]
    k = ir.kernel_from_json(v["kernel"])
    ham = [(c, w) for c, w in v["hamiltonian"]]
    for pt, e, per in zip(v["points"], v["energies"], v["per_term"]):
        st = P.final_state(ir.bind(k, pt))
        assert [P.pauli_expectation(st, w) for _, w in ham] == per
        assert P.observe(ir.bind(k, pt), ham) == e
