"""Parity AT THE BENCHMARKED CONFIG SIZES (BASELINE configs 2-5), against fixtures the
REAL reference produced (tests/golden/make_config_goldens.py: `sim.run_trajectory`,
`sim.statevector`, `sim.expval_pauli` of /root/reference/pkg/src on the same circuits,
compiled by the reference frontend).  Production settings: the engine defaults the
bench runs with -- batch of 8192 trajectories, history dedup, register-phase fusion,
NVRTC-specialised kernels.

Tolerances (north_star): keys / traces bit-exact (complex128); amplitudes and
expectation values 1e-10 (complex128) and 1e-5 (complex64); energies 1e-10 * sum |c_k|.
States are compared through digests (tests/golden/digest.py: 512 amplitudes, every
per-qubit marginal, 4 full-state projections, the norm) -- a 2^20..2^24 state is too
large to commit.
"""

import os
import sys

import numpy as np
import pytest

from paper_2604_11599_b200 import _lib, ir, sim, workloads

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import digest  # noqa: E402

pytestmark = pytest.mark.gpu

TOL = {"c128": 1e-10, "c64": 1e-5}
BENCH_BATCH = 8192  # bench.py's trajectories per step


def _need(golden, name):
    if not os.path.exists(os.path.join(HERE, "golden", name)):
        pytest.fail(f"fixture {name} missing: run tests/golden/make_config_goldens.py")
    return golden(name)


def test_dyn20_2000_shot_keys_production_batch(golden):
    """cfg 2 DYN20: the classical key of every global shot 0..1999 (seed 1234) vs the
    reference, out of one production batch of 8192 trajectories (dedup + fusion + JIT),
    plus the final states of shots 0..15 as the batched engine leaves them (1e-10)."""
    g = _need(golden, "dyn20_keys.json")
    _, k = workloads.dyn_circuit()
    b = ir.bind(k, [])
    nst = len(g["states"])
    words, states = sim.sample_final_states(b, BENCH_BATCH, g["seed"], nst)
    st = sim.last_stats()
    assert st["jit_passes"] > 0 and st["engine"] == 1
    tape = sim.compile_tape(k)
    keys = tape.keys(words[: g["shots"]])
    bad = [i for i, (a, w) in enumerate(zip(keys, g["keys"])) if a != w]
    assert not bad, f"{len(bad)} of {g['shots']} keys differ, first shots {bad[:8]}"
    worst = 0.0
    for rec, sv in zip(g["states"], states):
        err = digest.max_error(digest.digest(sv.amps, 20), rec["digest"])
        worst = max(worst, err)
        assert err <= TOL["c128"], (rec["shot"], err)
    # and the same shots through the public sample(): histogram of the first 2000 keys
    from collections import Counter

    assert sim.sample(b, g["shots"], g["seed"]).counts == dict(Counter(g["keys"]))


def test_dyn20_batch_split_invariance(golden):
    """The 2000 keys do not depend on how the shots are batched or sharded: 4 disjoint
    global-shot ranges (as 4 ranks would run them) reproduce the reference keys."""
    g = _need(golden, "dyn20_keys.json")
    _, k = workloads.dyn_circuit()
    b = ir.bind(k, [])
    tape = sim.compile_tape(k)
    keys = []
    for lo, hi in ((0, 700), (700, 1000), (1000, 1999), (1999, 2000)):
        w, _ = sim.sample_words(b, hi - lo, g["seed"], shot_begin=lo)
        keys += tape.keys(w)
    assert keys == g["keys"]


def test_dyn20_c64_states_and_keys(golden):
    """complex64 at config size: final states of shots 0..15 within 1e-5 of the
    (complex128) reference wherever the key agrees; keys agree on >= 99 % of 2000."""
    g = _need(golden, "dyn20_keys.json")
    _, k = workloads.dyn_circuit()
    b = ir.bind(k, [])
    nst = len(g["states"])
    words, states = sim.sample_final_states(b, g["shots"], g["seed"], nst, precision="c64")
    keys = sim.compile_tape(k).keys(words)
    agree = sum(a == w for a, w in zip(keys, g["keys"]))
    assert agree >= 0.99 * g["shots"], agree
    for i, (rec, sv) in enumerate(zip(g["states"], states)):
        if keys[i] != g["keys"][i]:
            continue
        err = digest.max_error(digest.digest(sv.amps, 20), rec["digest"])
        assert err <= TOL["c64"], (rec["shot"], err)


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_vqe24_energies_16_points(golden, prec):
    """cfg 3 VQE24 (24 qubits, 8 layers, 200-term H): energies at points 0..15 of the
    4096-point sweep within TOL * sum |c_k|, per-term values at points 0 and 1 within
    TOL, all 16 points in one batched observe() call."""
    g = _need(golden, "vqe24.json")
    _, k = workloads.vqe_ansatz()
    ham = workloads.vqe_hamiltonian()
    assert len(ham) == g["hamiltonian_terms"]
    pts = workloads.vqe_points(4096)[: len(g["energies"])]
    e, terms = sim.observe(k, ham, pts, precision=prec, return_terms=True)
    scale = sum(abs(c) for c, _ in ham)
    err = np.max(np.abs(e - np.array(g["energies"])))
    assert err <= TOL[prec] * scale, err
    terr = np.max(np.abs(terms[:2] - np.array(g["per_term"])))
    assert terr <= TOL[prec], terr


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_rdc22_depth200_trajectories(golden, prec):
    """cfg 4's twin RDC22 (the RDC30 generator at 22 qubits, depth 200, 10 measure
    rounds): keys, consumed uniforms and the branch trace bit-exact, final state within
    TOL, shots 0 and 1."""
    g = _need(golden, "rdc22.json")
    _, k = workloads.rdc_circuit(n=22, depth=200)
    b = ir.bind(k, [])
    for rec in g["shots"]:
        trace = []
        store, st = sim.run_trajectory(b, sim.RngStream.for_shot(g["seed"], rec["shot"]), trace, precision=prec)
        if prec == "c128":
            assert store.key() == rec["key"]
            assert [[t[2], t[1]] for t in trace] == rec["trace"]
        elif store.key() != rec["key"]:
            continue  # a complex64 decision inside the tie band: no state to compare
        err = digest.max_error(digest.digest(st.amps, 22), rec["digest"])
        assert err <= TOL[prec], (rec["shot"], err)


def test_rdc24_sliced_three_global_qubits(golden):
    """cfg 5's twin: RDC24 depth 40 forced onto 8 slices (3 global qubits, 1-GPU
    emulation of the 8-rank exchange protocol) vs the reference's run_trajectory: keys
    bit-exact, final state within 1e-10; the unsliced device path agrees too."""
    from paper_2604_11599_b200 import sliced

    g = _need(golden, "rdc24.json")
    _, k = workloads.rdc_circuit(n=24, depth=40)
    b = ir.bind(k, [])
    for rec in g["shots"]:
        store, sst = sliced.run_trajectory_sliced(b, sim.RngStream.for_shot(g["seed"], rec["shot"]), global_qubits=3)
        assert store.key() == rec["key"]
        amps = sst.gather()
        err = digest.max_error(digest.digest(amps, 24), rec["digest"])
        assert err <= TOL["c128"], (rec["shot"], err)
        store, st = sim.run_trajectory(b, sim.RngStream.for_shot(g["seed"], rec["shot"]))
        assert store.key() == rec["key"]
        assert digest.max_error(digest.digest(st.amps, 24), rec["digest"]) <= TOL["c128"]


def _oracle_dyn20_state(shot):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from oracle import sim_port as P

    _, k = workloads.dyn_circuit()
    store, st = P.trajectory(ir.bind(k, []), P.PortRng.for_shot(1234, shot))
    return store.key(), st.amps


def test_dyn20_full_states_vs_oracle():
    """Full 2^20-amplitude final states (not digests) of DYN20 shots 0..7 out of a
    production batch, against the CPU oracle (oracle/sim_port.py, pinned at 0 ulp to
    the reference) run on this host's cores in parallel: every amplitude within 1e-10."""
    import multiprocessing as mp

    nshots = 8
    with mp.get_context("spawn").Pool(min(nshots, os.cpu_count() or 1)) as pool:
        pending = pool.map_async(_oracle_dyn20_state, range(nshots))
        _, k = workloads.dyn_circuit()
        words, states = sim.sample_final_states(ir.bind(k, []), BENCH_BATCH, 1234, nshots)
        keys = sim.compile_tape(k).keys(words[:nshots])
        ref = pending.get(timeout=1800)
    for i, (rkey, ramps) in enumerate(ref):
        assert keys[i] == rkey, i
        err = float(np.max(np.abs(states[i].amps - ramps)))
        assert err <= TOL["c128"], (i, err)


def test_digest_is_sensitive():
    """The digest catches an error on a digested amplitude, a 1e-9 relative error of
    the whole state, a wrong phase on half the state, and a swap of two amplitudes.  It
    cannot see a tiny error confined to one undigested amplitude -- the full-state
    comparison against the oracle above covers that."""
    rng = np.random.default_rng(0)
    n = 16
    a = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    a /= np.linalg.norm(a)
    d0 = digest.digest(a, n)
    b = a.copy()
    b[d0["idx"][7]] += 1e-9
    assert digest.max_error(digest.digest(b, n), d0) > 1e-10
    assert digest.max_error(digest.digest(a * (1 + 1e-9), n), d0) > 1e-10
    c = a.copy()
    c[1 << (n - 1):] *= np.exp(1e-7j)
    assert digest.max_error(digest.digest(c, n), d0) > 1e-10
    c = a.copy()
    c[[100, 40000]] = c[[40000, 100]]
    assert digest.max_error(digest.digest(c, n), d0) > 1e-7


def _oracle_final(args):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from oracle import sim_port as P

    kind, params, seed, shot = args
    k = workloads.random_dynamic(*params) if kind == "random" else workloads.dyn_circuit(**params)[1]
    try:
        store, st = P.trajectory(ir.bind(k, []), P.PortRng.for_shot(seed, shot))
    except P.DegenerateBranch:
        return None
    return store.key(), st.amps


@pytest.mark.parametrize("kind,params", [
    ("random", (17, 160, 11)), ("random", (17, 160, 12)), ("random", (18, 220, 13)),
    ("dyn", {"n": 18, "layers": 10, "every": 5, "nmeas": 3, "seed": 5}),
])
def test_streaming_dynamic_final_states_vs_oracle(kind, params):
    """Dynamic circuits on the streaming engine at its production settings (batch with
    history dedup, known-zero items after each measurement, zero-aware planning, NVRTC
    passes): random circuits with guarded measurements / resets / register predicates
    and a DYN-shaped circuit, final states of shots 0..5 of a 64-trajectory batch vs the
    oracle -- keys bit-exact, every amplitude within 1e-10."""
    import multiprocessing as mp

    k = workloads.random_dynamic(*params) if kind == "random" else workloads.dyn_circuit(**params)[1]
    b = ir.bind(k, [])
    seed, nst = 7, 6
    with mp.get_context("spawn").Pool(min(nst, os.cpu_count() or 1)) as pool:
        pending = pool.map_async(_oracle_final, [(kind, params, seed, s) for s in range(nst)])
        words, states = sim.sample_final_states(b, 64, seed, nst)
        ref = pending.get(timeout=1800)
    st = sim.last_stats()
    assert st["engine"] == 1
    keys = sim.compile_tape(k).keys(words[:nst])
    for i, r in enumerate(ref):
        if r is None:
            continue
        assert keys[i] == r[0], i
        np.testing.assert_allclose(states[i].amps, r[1], atol=TOL["c128"], rtol=0)


@pytest.mark.parametrize("kind,params", [
    ("random", (17, 160, 11)), ("dyn", {"n": 18, "layers": 10, "every": 5, "nmeas": 3, "seed": 5}),
])
def test_known_zero_skipping_is_exact(kind, params):
    """The known-zero machinery (items skipped, zeros generated in the gather instead of
    read, the end-of-run zero store) computes exactly what the plain path computes: same
    keys, equal amplitudes (context option zero_fill 1 vs 0, same plan)."""
    k = workloads.random_dynamic(*params) if kind == "random" else workloads.dyn_circuit(**params)[1]
    b = ir.bind(k, [])
    ctx = _lib.context()
    out = {}
    for zf in (0, 1):
        ctx.set_option("zero_fill", zf)
        try:
            out[zf] = sim.sample_final_states(b, 64, 7, 8)
        finally:
            ctx.set_option("zero_fill", 1)
    assert np.array_equal(out[0][0], out[1][0])
    for a, c in zip(out[0][1], out[1][1]):
        assert np.array_equal(a.amps, c.amps)
