"""GPU parity: the B200 backend through the C ABI vs the reference (golden
fixtures recorded from /root/reference by tests/golden/make_goldens.py) and vs
the CPU oracle (oracle/sim_port.py, itself pinned bit-exact to the reference).

Tolerances (north_star / SURVEY.md §4):
  amplitudes, expectation values : 1e-10 (complex128), 1e-5 (complex64)
  histograms, per-shot keys, branch traces, RNG words : bit-exact (complex128)
"""

import contextlib
import math
import random

import numpy as np
import pytest

from oracle import sim_port as P
from paper_2604_11599_b200 import _lib, ir, sim, workloads
from paper_2604_11599_b200.errors import BadPauliString, DegenerateNorm, DynamicCircuit, SimError

pytestmark = pytest.mark.gpu

TOL = {"c128": 1e-10, "c64": 1e-5}


def cvec(d):
    return np.array(d["re"]) + 1j * np.array(d["im"])


@contextlib.contextmanager
def engine(which):
    """which: 'auto' | 'resident' | 'stream'"""
    ctx = _lib.context()
    ctx.set_option("engine", {"auto": -1, "resident": 0, "stream": 1}[which])
    try:
        yield
    finally:
        ctx.set_option("engine", -1)


@contextlib.contextmanager
def option(key, value, reset):
    ctx = _lib.context()
    ctx.set_option(key, value)
    try:
        yield
    finally:
        ctx.set_option(key, reset)


def assert_state(got, want, tol):
    err = np.max(np.abs(np.asarray(got) - np.asarray(want))) if len(want) else 0.0
    assert err <= tol, f"max |err| {err:.3e} > {tol}"


# ---------------------------------------------------------------------------


def test_device_rng_known_answers(golden):
    ctx = _lib.context()
    for case in golden("rng.json")["for_shot"]:
        out = np.zeros(6)
        _lib.check(ctx.lib.qsb_debug_rng(ctx.handle, case["seed"] & ((1 << 64) - 1), case["shot"], 6, _lib.ptr(out)))
        assert list(out) == case["uniforms"]


@pytest.mark.parametrize("eng", ["resident", "stream"])
def test_ff_suite_histograms_bit_exact(golden, eng):
    with engine(eng):
        for name, case in golden("ff_suite.json").items():
            b = ir.bind(ir.kernel_from_json(case["kernel"]), [])
            assert sim.sample(b, 1024, 1234).counts == case["hist_1024_seed1234"], name


@pytest.mark.parametrize("eng", ["resident", "stream"])
def test_ff_suite_trajectories(golden, eng):
    with engine(eng):
        for name, case in golden("ff_suite.json").items():
            b = ir.bind(ir.kernel_from_json(case["kernel"]), [])
            for rec in case["shots"][:32]:
                rng = sim.RngStream.for_shot(1234, rec["shot"])
                trace = []
                store, st = sim.run_trajectory(b, rng, trace)
                assert store.key() == rec["key"], (name, rec["shot"])
                assert [[t[2], t[1]] for t in trace] == rec["trace"]
                assert_state(st.amps, cvec(rec["state"]), 1e-10)
                # rng advanced by exactly the uniforms consumed
                ref = sim.RngStream.for_shot(1234, rec["shot"])
                for _ in rec["uniforms"]:
                    ref.uniform()
                assert (rng.s0, rng.s1, rng.s2, rng.s3) == (ref.s0, ref.s1, ref.s2, ref.s3)


@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("eng", ["auto", "stream"])
def test_static_statevectors_and_expval(golden, prec, eng):
    with engine(eng):
        for case in golden("static.json"):
            k = ir.kernel_from_json(case["kernel"])
            st = sim.statevector(ir.bind(k, case["values"]), precision=prec)
            assert_state(st.amps, cvec(case["state"]), TOL[prec])
            assert abs(st.norm() - case["norm"]) <= TOL[prec]
            for word, val in case["expval"]:
                assert abs(sim.expval_pauli(st, word) - val) <= 4 * TOL[prec], word


def test_static_sampling_bit_exact(golden):
    for case in golden("static_sampling.json"):
        b = ir.bind(ir.kernel_from_json(case["kernel"]), [])
        assert sim.sample(b, case["shots"], case["seed"]).counts == case["counts"]


@pytest.mark.parametrize("eng", ["resident", "stream"])
def test_dynamic_random_circuits(golden, eng):
    with engine(eng):
        for case in golden("dynamic.json"):
            b = ir.bind(ir.kernel_from_json(case["kernel"]), [])
            if case["counts_512"] is not None:
                assert sim.sample(b, 512, case["seed"]).counts == case["counts_512"]
            for rec in case["shots"]:
                rng = sim.RngStream.for_shot(case["seed"], rec["shot"])
                if "error" in rec:
                    with pytest.raises(DegenerateNorm):
                        sim.run_trajectory(b, rng)
                    continue
                trace = []
                store, st = sim.run_trajectory(b, rng, trace)
                assert store.key() == rec["key"]
                assert [[t[2], t[1]] for t in trace] == rec["trace"]
                if "state" in rec:
                    assert_state(st.amps, cvec(rec["state"]), 1e-10)


@pytest.mark.parametrize("eng", ["resident", "stream"])
def test_predrawn_streams(golden, eng):
    with engine(eng):
        for case in golden("predrawn.json"):
            b = ir.bind(ir.kernel_from_json(case["kernel"]), [])
            vals = np.array([case["values"]])
            if "error" in case["record"]:
                with pytest.raises(DegenerateNorm):
                    sim.sample_words(b, 1, 0, predrawn=vals)
                continue
            words, tape = sim.sample_words(b, 1, 0, predrawn=vals)
            assert tape.keys(words) == [case["record"]["key"]]
            # the per-op path with an arbitrary uniform() object
            store, st = sim.run_trajectory(b, P.PredrawnStream(case["values"]))
            assert store.key() == case["record"]["key"]
            assert_state(st.amps, cvec(case["record"]["state"]), 1e-10)


@pytest.mark.parametrize("eng", ["resident", "stream"])
def test_twins(golden, eng):
    t = golden("twins.json")
    with engine(eng):
        b = ir.bind(ir.kernel_from_json(t["dyn8"]["kernel"]), [])
        assert sim.sample(b, 1024, 1234).counts == t["dyn8"]["counts_1024"]
        for rec in t["dyn8"]["shots"][:8]:
            store, st = sim.run_trajectory(b, sim.RngStream.for_shot(1234, rec["shot"]))
            assert store.key() == rec["key"]
            if "state" in rec:
                assert_state(st.amps, cvec(rec["state"]), 1e-10)
        b = ir.bind(ir.kernel_from_json(t["rdc10"]["kernel"]), [])
        for rec in t["rdc10"]["shots"]:
            store, st = sim.run_trajectory(b, sim.RngStream.for_shot(1234, rec["shot"]))
            assert store.key() == rec["key"]
            if "state" in rec:
                assert_state(st.amps, cvec(rec["state"]), 1e-10)


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_vqe_observe(golden, prec):
    v = golden("twins.json")["vqe6"]
    k = ir.kernel_from_json(v["kernel"])
    ham = [(c, w) for c, w in v["hamiltonian"]]
    e, terms = sim.observe(k, ham, v["points"], precision=prec, return_terms=True)
    scale = sum(abs(c) for c, _ in ham)
    assert np.max(np.abs(e - np.array(v["energies"]))) <= TOL[prec] * scale
    assert np.max(np.abs(terms - np.array(v["per_term"]))) <= 4 * TOL[prec]


def test_dyn20_first_shots_bit_exact(golden):
    """The headline workload (cfg 2) itself: per-shot keys of the first shots vs the
    reference, and the consumed-uniform count."""
    _, k = workloads.dyn_circuit()
    b = ir.bind(k, [])
    recs = golden("twins.json")["dyn20"]["shots"]
    words, tape = sim.sample_words(b, len(recs), 1234)
    assert tape.keys(words) == [r["key"] for r in recs]
    for rec in recs:
        rng = sim.RngStream.for_shot(1234, rec["shot"])
        trace = []
        store, st = sim.run_trajectory(b, rng, trace)
        assert store.key() == rec["key"]
        assert [[t[2], t[1]] for t in trace] == rec["trace"]
        assert abs(st.norm() - 1.0) < 1e-10


def test_rdc_state_vs_oracle_c128_and_c64():
    """Down-scaled RDC (cfg 4 twin): final state of one trajectory, streaming engine."""
    _, k = workloads.rdc_circuit(n=16, depth=40, every=20, seed=30200)
    b = ir.bind(k, [])
    rs, ref = P.trajectory(b, P.PortRng.for_shot(1234, 0))
    for prec in ("c128", "c64"):
        store, st = sim.run_trajectory(b, sim.RngStream.for_shot(1234, 0), precision=prec)
        assert store.key() == rs.key()
        assert_state(st.amps, ref.amps, TOL[prec])


def test_batch_and_run_invariance():
    """Histograms do not depend on the device batch size and repeat bit-identically."""
    _, k = workloads.dyn_circuit(n=14, layers=10, every=5, nmeas=3, seed=11)
    b = ir.bind(k, [])
    base = sim.sample(b, 600, 77).counts
    with option("batch", 64, 0):
        assert sim.sample(b, 600, 77).counts == base
    assert sim.sample(b, 600, 77).counts == base
    ref = P.sample_counts(b, 60, 77)
    assert sim.sample(b, 60, 77).counts == ref


def test_tile_sizes_agree():
    _, k = workloads.dyn_circuit(n=15, layers=10, every=5, nmeas=3, seed=12)
    b = ir.bind(k, [])
    want = P.trajectory_keys(b, 5, 0, 12)
    for tq in (6, 9, 12):
        with option("tile_qubits", tq, 0):
            words, tape = sim.sample_words(b, 12, 5)
            assert tape.keys(words) == want, tq


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_jit_kernels_bit_identical_to_generic(prec):
    """The NVRTC-specialised pass kernels and the generic register-blocked kernel run
    the same arithmetic: final states must agree bit for bit, and both match the
    oracle.  Covers controls on register / thread / out-of-tile qubits, negative
    controls, swaps, ParamRef angles and diagonal gates outside the tile."""
    k = workloads.random_static(15, 400, seed=77, nparams=4, max_controls=2)
    vals = [0.3, -1.1, 2.2, 0.7]
    b = ir.bind(k, vals)
    with option("fuse", 0, 1):  # gate fusion changes the arithmetic (tested below)
        with option("jit", 0, 1):
            generic = sim.statevector(b, precision=prec).amps
        jit = sim.statevector(b, precision=prec).amps
        assert sim.last_stats()["jit_passes"] > 0
        np.testing.assert_array_equal(jit, generic)
        assert_state(jit, P.final_state(b).amps, TOL[prec])
        _, kd = workloads.dyn_circuit(n=16, layers=10, every=5, nmeas=3, seed=21)
        bd = ir.bind(kd, [])
        with option("jit", 0, 1):
            w0, tape = sim.sample_words(bd, 64, 9, precision=prec)
        w1, _ = sim.sample_words(bd, 64, 9, precision=prec)
        np.testing.assert_array_equal(w0, w1)
        if prec == "c128":
            assert tape.keys(w1) == P.trajectory_keys(bd, 9, 0, 64)


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_fused_blocks_match_oracle(prec):
    """Register-phase gate fusion (dense 2x2 / 4x4 products of literal gates, NVRTC
    kernels): the fused kernels run fewer FP operations than the unfused ones and
    agree with the oracle within the precision's tolerance; c128 trajectories of a
    u-brick dynamic circuit stay bit-exact."""
    _, kd = workloads.dyn_circuit(n=16, layers=10, every=5, nmeas=3, seed=21)
    bd = ir.bind(kd, [])
    # the gates before the first measurement round: a static u-brick
    first = []
    for op in kd.body:
        if not isinstance(op, ir.Gate):
            break
        first.append(op)
    bs = ir.bind(ir.Kernel(kd.qubit_count, kd.qubit_layout, [], [], first), [])
    ref = P.final_state(bs).amps
    stats = {}
    for fuse in (0, 1):
        with option("fuse", fuse, 1):
            st = sim.statevector(bs, precision=prec)
            stats[fuse] = sim.last_stats()
            assert stats[fuse]["jit_passes"] > 0
            assert_state(st.amps, ref, TOL[prec])
    assert stats[1]["pass_flops"] < 0.9 * stats[0]["pass_flops"], (stats[0]["pass_flops"], stats[1]["pass_flops"])
    words, tape = sim.sample_words(bd, 64, 9, precision=prec)
    if prec == "c128":
        assert tape.keys(words) == P.trajectory_keys(bd, 9, 0, 64)
    k = workloads.random_static(15, 400, seed=77, nparams=4, max_controls=2)
    b = ir.bind(k, [0.3, -1.1, 2.2, 0.7])
    assert_state(sim.statevector(b, precision=prec).amps, P.final_state(b).amps, TOL[prec])


@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("jit", [0, 1])
def test_register_blocking(prec, jit):
    """8, 16 or 32 amplitudes per thread regroup the gates into different phases, which
    reorders commuting gates on disjoint qubits (a last-ulp effect, like any
    reordering of (A x I)(I x B)): both blockings must match the oracle within the
    precision's tolerance, and c128 trajectories must stay bit-exact."""
    k = workloads.random_static(15, 300, seed=5, nparams=2, max_controls=2)
    b = ir.bind(k, [0.4, -0.9])
    _, kd = workloads.dyn_circuit(n=15, layers=10, every=5, nmeas=3, seed=23)
    bd = ir.bind(kd, [])
    want = P.final_state(b).amps
    with option("jit", jit, 1):
        for rb in (4, 3, 5):
            with option("reg_bits", rb, 4):
                assert_state(sim.statevector(b, precision=prec).amps, want, TOL[prec])
                words, tape = sim.sample_words(bd, 48, 3, precision=prec)
                if prec == "c128":
                    assert tape.keys(words) == P.trajectory_keys(bd, 3, 0, 48), rb


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_history_dedup_bit_identical(prec):
    """Trajectories with equal outcome histories share one state buffer; per-shot keys
    (and therefore histograms) must not change, and the first segment of DYN-like
    circuits must run on a single state (fewer physical bytes than logical)."""
    _, k = workloads.dyn_circuit(n=14, layers=10, every=5, nmeas=3, seed=31)
    b = ir.bind(k, [])
    with option("dedup", 0, 1):
        w0, tape = sim.sample_words(b, 300, 5, precision=prec)
        logical = sim.last_stats()["pass_bytes"]
    w1, _ = sim.sample_words(b, 300, 5, precision=prec)
    physical = sim.last_stats()["pass_bytes"]
    np.testing.assert_array_equal(w0, w1)
    assert physical < logical
    if prec == "c128":
        assert tape.keys(w1[:40]) == P.trajectory_keys(b, 5, 0, 40)


def test_per_op_api_matches_reference_semantics():
    from paper_2604_11599_b200.ir import Gate

    st = sim.StateVector.zero(2)
    sim.apply_gate(st, Gate("x", (), (0,), ()))
    sim.apply_gate(st, Gate("x", (), (1,), ((0, 1),)))
    np.testing.assert_allclose(st.amps, [0, 0, 0, 1], atol=1e-15)
    st = sim.StateVector.zero(1)
    sim.apply_gate(st, Gate("h", (), (0,), ()))
    assert abs(sim.expval_pauli(st, "X") - 1.0) < 1e-12
    outs = {sim.measure(sim.apply_gate(sim.StateVector.zero(1), Gate("h", (), (0,), ())), 0,
                        sim.RngStream.for_shot(3, s)) for s in range(40)}
    assert outs == {0, 1}
    st = sim.StateVector.zero(1)
    sim.apply_gate(st, Gate("x", (), (0,), ()))
    sim.reset(st, 0, sim.RngStream(0))
    np.testing.assert_allclose(st.amps, [1, 0], atol=1e-15)
    # reading .amps hands out a read-only snapshot and costs no re-upload
    st = sim.StateVector.zero(1)
    a = st.amps
    with pytest.raises(ValueError):
        a[:] = [0, 1]
    sim.apply_gate(st, Gate("h", (), (0,), ()))
    assert st.uploads == 0
    # explicit host edits are honoured by the next device op: in place after flipping
    # the snapshot writeable, or by assignment
    st = sim.StateVector.zero(1)
    a = st.amps
    a.flags.writeable = True
    a[:] = [0, 1]
    sim.apply_gate(st, Gate("x", (), (0,), ()))
    np.testing.assert_allclose(st.amps, [1, 0], atol=1e-15)
    assert st.uploads == 1
    st.amps = np.array([0, 1j])
    sim.apply_gate(st, Gate("x", (), (0,), ()))
    np.testing.assert_allclose(st.amps, [1j, 0], atol=1e-15)
    with pytest.raises(BadPauliString):
        sim.expval_pauli(st, "ZZ")
    with pytest.raises(BadPauliString):
        sim.expval_pauli(st, "Q")


def test_errors():
    _, k = workloads.ff_teleport()
    b = ir.bind(k, [])
    with pytest.raises(SimError):
        sim.sample(b, 0, 1)
    with pytest.raises(DynamicCircuit):
        sim.statevector(b)
    deg = ir.Kernel(1, [("q", 1)], [], [("c", 1)], [ir.Gate("rx", (2e-9,), (0,), ()), ir.Measure(0, ("c", 0))])
    with pytest.raises(DegenerateNorm):
        sim.sample_words(ir.bind(deg, []), 1, 0, predrawn=np.array([[0.0]]))


def test_empty_and_no_bits():
    k = ir.Kernel(1, [("q", 1)], [], [], [ir.Gate("h", (), (0,), ())])
    assert sim.sample(ir.bind(k, []), 50, 1).counts == {"": 50}
    k0 = ir.Kernel(0, [], [], [], [])
    st = sim.statevector(ir.bind(k0, []))
    np.testing.assert_allclose(st.amps, [1.0])


def test_qft_matches_dft():
    n = 12
    body = [ir.Gate("x", (), (0,), ())]
    for j in reversed(range(n)):
        body.append(ir.Gate("h", (), (j,), ()))
        for q in reversed(range(j)):
            body.append(ir.Gate("p", (math.pi / (1 << (j - q)),), (j,), ((q, 1),)))
    for i in range(n // 2):
        body.append(ir.Gate("swap", (), (i, n - 1 - i), ()))
    k = ir.Kernel(n, [("q", n)], [], [], body)
    for eng in ("auto", "stream"):
        with engine(eng):
            st = sim.statevector(ir.bind(k, []))
            j = np.arange(1 << n)
            want = np.exp(2j * math.pi * j / (1 << n)) / math.sqrt(1 << n)
            fid = abs(np.vdot(st.amps, want)) ** 2
            assert fid > 1 - 1e-10


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_device_histogram_matches_per_shot_words(golden, prec):
    """qsb_sample_counts (sort + run-length encode in HBM) == the histogram of the
    per-shot words, for the trajectory path, the static path and a bitless kernel."""
    _, kd = workloads.dyn_circuit(n=14, layers=10, every=5, nmeas=3, seed=41)
    cases = [ir.bind(kd, [])]
    cases += [ir.bind(ir.kernel_from_json(c["kernel"]), []) for c in golden("static_sampling.json")]
    cases.append(ir.bind(ir.Kernel(2, [("q", 2)], [], [], [ir.Gate("h", (), (0,), ())]), []))
    for b in cases:
        words, tape = sim.sample_words(b, 700, 99, shot_begin=5, precision=prec)
        uniq, counts = sim.sample_counts(b, 700, 99, shot_begin=5, precision=prec)
        w, c = np.unique(words[:, 0], return_counts=True)
        np.testing.assert_array_equal(uniq[:, 0], w)
        np.testing.assert_array_equal(counts, c)
        assert counts.sum() == 700
        w0, _ = sim.sample_words(b, 700, 99, precision=prec)
        assert sim.sample(b, 700, 99, precision=prec).counts == sim.histogram_from_words(tape, w0, 700).counts
    # sample() goes through the device histogram and still matches the reference goldens
    for name, case in golden("ff_suite.json").items():
        b = ir.bind(ir.kernel_from_json(case["kernel"]), [])
        if prec == "c128":
            assert sim.sample(b, 1024, 1234).counts == case["hist_1024_seed1234"], name


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_observe_register_mapped_reducer(prec):
    """Full 12-qubit tiles take the register-mapped Pauli kernel: X supports up to 5
    letters (> 4 forces extra mappings / groups), Y phases, out-of-tile Z signs and
    diagonal terms, per term against the oracle's expval_pauli."""
    n = 15
    k = workloads.random_static(n, 200, seed=61, nparams=3, max_controls=1)
    vals = [0.2, -1.3, 0.8]
    ham = workloads.vqe_hamiltonian(n=n, terms=70, seed=5)
    ham += [(0.5, "X" * 5 + "I" * (n - 5)), (-0.25, "I" * 3 + "YZXZY" + "I" * (n - 8)),
            (0.75, "Z" * n), (0.1, "I" * n), (0.3, "Y" + "I" * (n - 2) + "X")]
    e, terms = sim.observe(k, ham, [vals], precision=prec, return_terms=True)
    st = P.final_state(ir.bind(k, vals))
    want = np.array([P.pauli_expectation(st, w) for _, w in ham])
    assert np.max(np.abs(terms[0] - want)) <= 4 * TOL[prec]
    assert abs(e[0] - sum(c * v for (c, _), v in zip(ham, want))) <= TOL[prec] * sum(abs(c) for c, _ in ham)


def _local_brick(n, layers, seed):
    """Dense neighbour-local circuit for the fusion planner: every layer puts a random
    single-qubit gate (any base, random adjoint) on each qubit, then random controlled
    gates (positive or negative control) on neighbouring pairs."""
    rng = random.Random(seed)
    body = []
    one = ("x", "y", "z", "h", "s", "t", "sx", "rx", "ry", "rz", "p", "u")
    arity = {"rx": 1, "ry": 1, "rz": 1, "p": 1, "u": 3}
    for layer in range(layers):
        for q in range(n):
            b = rng.choice(one)
            angles = tuple(rng.uniform(-math.pi, math.pi) for _ in range(arity.get(b, 0)))
            body.append(ir.Gate(b, angles, (q,), (), rng.random() < 0.3))
        for q in range(layer % 2, n - 1, 2):
            b = rng.choice(("x", "z", "y", "rz", "p", "u", "h"))
            angles = tuple(rng.uniform(-math.pi, math.pi) for _ in range(arity.get(b, 0)))
            c, t = (q, q + 1) if rng.random() < 0.5 else (q + 1, q)
            body.append(ir.Gate(b, angles, (t,), ((c, rng.choice((0, 1))),), rng.random() < 0.2))
    return ir.Kernel(n, [("q", n)], [], [], body)


@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_fusion_random_local_circuits(prec, seed):
    """Random neighbour-local circuits (all bases, adjoints, positive / negative
    controls, controlled non-Pauli gates) through the fused NVRTC kernels: states match
    the oracle within the precision's tolerance, with and without fusion, and fusion
    lowers the executed FP work."""
    k = _local_brick(14, 12, seed)
    b = ir.bind(k, [])
    want = P.final_state(b).amps
    flops = {}
    for fuse in (0, 1):
        with option("fuse", fuse, 1):
            got = sim.statevector(b, precision=prec).amps
            st = sim.last_stats()
            assert st["jit_passes"] > 0
            flops[fuse] = st["pass_flops"]
            assert_state(got, want, TOL[prec])
    assert flops[1] < flops[0], flops


@pytest.mark.gpu
def test_rdc30_full_size_properties():
    """BASELINE cfg 4 at full size (30 qubits, two measurement rounds): size-independent
    properties where the oracle cannot follow -- the final state stays normalised (1e-10
    complex128 / 1e-5 complex64), the measured register is identical in both precisions
    (no decision inside the tie band), and a static 28-qubit circuit followed by its exact
    inverse returns |0...0> (every <Z_k> = 1 within 1e-10)."""
    _, k = workloads.rdc_circuit(n=30, depth=40, every=20, seed=30200)
    b = ir.bind(k, [])
    keys = {}
    for prec, tol in (("c128", 1e-10), ("c64", 1e-5)):
        store, st = sim.run_trajectory(b, sim.RngStream.for_shot(1234, 0), precision=prec)
        assert abs(st.norm() - 1.0) <= tol, (prec, st.norm())
        keys[prec] = store.key()
        del st
    assert keys["c128"] == keys["c64"], keys
    fwd = [op for op in workloads.rdc_circuit(n=28, depth=12, every=100, seed=7)[1].body if isinstance(op, ir.Gate)]
    inv = [ir.Gate(g.base, g.angles, g.targets, g.controls, not g.adjoint) for g in reversed(fwd)]
    st = sim.statevector(ir.bind(ir.Kernel(28, [("q", 28)], [], [], fwd + inv), []))
    assert abs(st.norm() - 1.0) <= 1e-10
    for q in range(28):
        z = sim.expval_pauli(st, "".join("Z" if i == q else "I" for i in range(28)))
        assert z >= 1.0 - 1e-10, (q, z)


def test_compiled_tape_released_with_its_kernel():
    """the tape cache must not keep a kernel (and its device tape, plans and
    NVRTC modules) alive -- deleting the kernel drops its cache entry."""
    import gc
    import weakref

    k = workloads.random_static(6, 20, seed=3)
    sim.statevector(ir.bind(k, []))
    key = (id(k), sim._ctx().device)
    assert key in sim._tape_cache
    ref = weakref.ref(k)
    del k
    gc.collect()
    assert ref() is None
    assert key not in sim._tape_cache


def test_jit_async_generic_first_then_specialised_bit_identical():
    """Option jit_async: the first runs of a new tape use the generic kernel while NVRTC
    compiles in the background, later runs the specialised kernels -- fusion is off for
    such plans, so every run is bit-identical to the generic kernel (deterministic
    whichever kernel ran), and the specialised kernels do arrive."""
    import time

    _, k = workloads.dyn_circuit(n=15, layers=10, every=5, nmeas=3, seed=77)
    b = ir.bind(k, [])
    with option("jit", 0, 1):
        ref_words, ref_states = sim.sample_final_states(b, 32, 5, 2)
        ref_amps = [np.array(st.amps) for st in ref_states]
    ctx = _lib.context()
    ctx.set_option("jit_async", 1)
    try:
        _, k2 = workloads.dyn_circuit(n=15, layers=10, every=5, nmeas=3, seed=77)  # a fresh tape
        b2 = ir.bind(k2, [])
        seen = set()
        for _ in range(60):
            words, states = sim.sample_final_states(b2, 32, 5, 2)
            np.testing.assert_array_equal(words, ref_words)
            for st, ra in zip(states, ref_amps):
                np.testing.assert_array_equal(st.amps, ra)
            seen.add(sim.last_stats()["jit_passes"] > 0)
            if True in seen:
                break
            time.sleep(1.0)
        assert True in seen, "the background NVRTC kernels never arrived"
        words, states = sim.sample_final_states(b2, 32, 5, 2)
        np.testing.assert_array_equal(words, ref_words)
    finally:
        ctx.set_option("jit_async", 0)


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_observe_jit_reducer_bit_identical_to_generic(prec):
    """The NVRTC-specialised Pauli reducer (n >= 16, >= 8 terms) computes exactly the
    generic accumulating kernel's arithmetic (same products, same butterfly order with the
    signs folded into add / subtract, same accumulation): bit-identical energies and
    per-term values, and both match the oracle."""
    n = 17
    k = workloads.random_static(n, 120, seed=91, nparams=2, max_controls=1)
    ham = workloads.vqe_hamiltonian(n=n, terms=60, seed=9)
    ham += [(0.5, "XXXXX" + "I" * (n - 5)), (0.25, "Z" * n)]
    pts = [[0.3, -0.7], [1.1, 0.4]]
    out = {}
    for jit in (0, 1):
        with option("expval_jit", jit, 1):
            out[jit] = sim.observe(k, ham, pts, precision=prec, return_terms=True)
    np.testing.assert_array_equal(out[0][0], out[1][0])
    np.testing.assert_array_equal(out[0][1], out[1][1])
    st = P.final_state(ir.bind(k, pts[0]))
    want = np.array([P.pauli_expectation(st, w) for _, w in ham])
    assert np.max(np.abs(out[1][1][0] - want)) <= 4 * TOL[prec]
