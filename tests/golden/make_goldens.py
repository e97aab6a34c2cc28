"""Generate the parity fixtures by running the REAL reference simulator.

Run in the build container (where `/root/reference` exists):

    python tests/golden/make_goldens.py

It imports `qasm2cudaq` from `/root/reference/pkg/src` (read-only; bytecode writing
is disabled so nothing lands in the reference tree), runs `sim.sample`,
`sim.run_trajectory`, `sim.statevector`, `sim.expval_pauli` and `RngStream` on the
workloads of `paper_2604_11599_b200.workloads`, and writes small JSON fixtures
next to this script.  The fixtures travel to the GPU box; the reference does not.
Floats are written with `repr` (exact round trip).
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time

sys.dont_write_bytecode = True
REF = os.environ.get("QASM2CUDAQ_REF", "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
from qasm2cudaq import kir as rkir  # noqa: E402
from qasm2cudaq import sema as rsema  # noqa: E402
from qasm2cudaq import sim as rsim  # noqa: E402
from qasm2cudaq import suites as rsuites  # noqa: E402
from qasm2cudaq.errors import DegenerateNorm  # noqa: E402

from paper_2604_11599_b200 import ir, workloads  # noqa: E402


def to_ref(kernel_json: dict):
    """Mirror-IR JSON -> the reference's own kir dataclasses."""

    def ang(a):
        return rsema.ParamRef(a["slot"]) if isinstance(a, dict) else float(a)

    def op(d):
        k = d["op"]
        if k == "gate":
            return rkir.Gate(d["base"], tuple(ang(a) for a in d["angles"]), tuple(d["targets"]),
                             tuple((q, p) for q, p in d["controls"]), d["adjoint"])
        if k == "measure":
            return rkir.Measure(d["qubit"], (d["bit"][0], d["bit"][1]))
        if k == "reset":
            return rkir.Reset(d["qubit"])
        if k == "nop":
            return rkir.Nop(tuple(d["qubits"]))
        p = d["pred"]
        return rkir.CondBlock(rkir.Predicate(p["register"], p["index"], p["comparator"], p["rhs"]),
                              [op(o) for o in d["then"]], [op(o) for o in d["else"]])

    return rkir.Kernel(
        qubit_count=kernel_json["qubit_count"],
        qubit_layout=[tuple(x) for x in kernel_json["qubit_layout"]],
        param_layout=[rsema.ParamSpec(n, c, a, o) for n, c, a, o in kernel_json["param_layout"]],
        classical_layout=[tuple(x) for x in kernel_json["classical_layout"]],
        body=[op(o) for o in kernel_json["body"]],
    )


def ir_hash(kernel) -> str:
    return hashlib.sha256(json.dumps(ir.kernel_to_json(kernel), sort_keys=True).encode()).hexdigest()


def cvec(a) -> dict:
    a = np.asarray(a, dtype=np.complex128)
    return {"re": [float(x) for x in a.real], "im": [float(x) for x in a.imag]}


class LoggingRng:
    """Wraps a reference RNG (or a pre-drawn list) and records every uniform drawn."""

    def __init__(self, inner=None, values=None):
        self.inner, self.values, self.drawn = inner, values, []

    def uniform(self):
        u = self.inner.uniform() if self.inner is not None else self.values[len(self.drawn)]
        self.drawn.append(u)
        return u


def traj_record(bound, seed, shot, with_state=True, values=None):
    rng = LoggingRng(inner=None if values is not None else rsim.RngStream.for_shot(seed, shot), values=values)
    trace = []
    try:
        store, state = rsim.run_trajectory(bound, rng, trace)
    except DegenerateNorm as e:
        return {"shot": shot, "error": "DegenerateNorm", "msg": str(e), "uniforms": rng.drawn}
    rec = {
        "shot": shot,
        "key": store.key(),
        "uniforms": rng.drawn,
        "trace": [[t[2], {k: list(v) for k, v in t[1].items()}] for t in trace],
    }
    if with_state:
        rec["state"] = cvec(state.amps)
    return rec


def write(name, obj):
    path = os.path.join(HERE, name)
    with open(path, "w") as f:
        json.dump(obj, f, separators=(",", ":"))
    print(f"wrote {name}: {os.path.getsize(path) / 1024:.1f} KiB")


def main():
    t0 = time.time()
    # ---- RNG known answers (sim.py:26-72) ---------------------------------
    rng = rsim.RngStream(42)
    state = [rng.s0, rng.s1, rng.s2, rng.s3]
    words = [rng.next_u64() for _ in range(8)]
    pairs = [(1234, 0), (1234, 1), (42, 0), (7, 99999), (-1, 5), (-(1 << 63), 3), ((1 << 64) + 9, 0),
             (0, 0), (2604, 12345678901), (123, (1 << 40) + 7)]
    shots = []
    for seed, shot in pairs:
        r = rsim.RngStream.for_shot(seed, shot)
        shots.append({"seed": seed, "shot": shot, "state": [r.s0, r.s1, r.s2, r.s3],
                      "uniforms": [r.uniform() for _ in range(6)]})
    write("rng.json", {"seed42_state": [str(x) for x in state], "seed42_words": [str(w) for w in words],
                       "for_shot": [{**s, "state": [str(x) for x in s["state"]]} for s in shots]})

    # ---- workload IR identity with the reference frontend ----------------
    hashes = {}
    sources = dict(workloads.ff_suite())
    sources["dyn20"] = workloads.dyn_circuit()
    sources["dyn8"] = workloads.dyn_circuit(n=8, layers=10, every=5, nmeas=2, seed=8)
    sources["vqe24"] = workloads.vqe_ansatz()
    sources["vqe6"] = workloads.vqe_ansatz(6, 2)
    sources["rdc30"] = workloads.rdc_circuit()
    sources["rdc10"] = workloads.rdc_circuit(n=10, depth=40, every=20, seed=10)
    for name, (src, kern) in sources.items():
        ref_k = rsuites.compile_source(src)
        hashes[name] = {"reference": ir_hash(ref_k), "mirror": ir_hash(kern)}
        assert hashes[name]["reference"] == hashes[name]["mirror"], name
    write("workload_ir.json", hashes)

    # ---- cfg 1 feedforward suite ----------------------------------------
    ff = {}
    for name, (src, kern) in workloads.ff_suite().items():
        kj = ir.kernel_to_json(kern)
        bound = rkir.bind(to_ref(kj), [])
        hist = rsim.sample(bound, 1024, 1234)
        ff[name] = {
            "kernel": kj,
            "hist_1024_seed1234": hist.counts,
            "shots": [traj_record(bound, 1234, s) for s in range(64)],
        }
    write("ff_suite.json", ff)

    # ---- static circuits: statevector + expval + static sampling ----------
    static = []
    prng = np.random.default_rng(2026)
    for i, (n, g, npar) in enumerate([(1, 8, 0), (2, 20, 0), (2, 20, 2), (3, 40, 0), (3, 40, 3), (4, 60, 0),
                                      (5, 80, 4), (6, 100, 0), (7, 120, 5), (8, 150, 0), (9, 150, 6),
                                      (10, 200, 0), (11, 120, 0), (12, 120, 3)]):
        kern = workloads.random_static(n, g, seed=100 + i, nparams=npar)
        kj = ir.kernel_to_json(kern)
        values = [float(v) for v in prng.uniform(-math.pi, math.pi, npar)]
        bound = rkir.bind(to_ref(kj), values)
        sv = rsim.statevector(bound)
        words = ["".join(prng.choice(list("IXYZ"), n)) for _ in range(6)] + ["I" * n, "Z" * n]
        static.append({
            "kernel": kj, "values": values, "state": cvec(sv.amps), "norm": sv.norm(),
            "expval": [[w, rsim.expval_pauli(sv, w)] for w in words],
        })
    write("static.json", static)

    sampling = []
    for i, n in enumerate([1, 2, 3, 5, 8, 10]):
        kern = workloads.random_static(n, 10 * n + 5, seed=700 + i)
        width = n
        kern.classical_layout = [("m", width)]
        order = list(range(n))
        np.random.default_rng(i).shuffle(order)
        kern.body += [ir.Measure(q, ("m", j)) for j, q in enumerate(order)]
        kj = ir.kernel_to_json(kern)
        bound = rkir.bind(to_ref(kj), [])
        assert not rsim._needs_trajectories(bound.kernel)
        counts = rsim.sample(bound, 4096, 31 + i).counts
        sampling.append({"kernel": kj, "seed": 31 + i, "shots": 4096, "counts": counts})
    write("static_sampling.json", sampling)

    # ---- dynamic random circuits (trajectory path) -----------------------
    dyn = []
    for i, (n, nops) in enumerate([(1, 12), (2, 16), (2, 24), (3, 30), (3, 30), (4, 40), (4, 40), (5, 50),
                                   (6, 50), (7, 60), (8, 60), (8, 80)]):
        kern = workloads.random_dynamic(n, nops, seed=900 + i)
        kj = ir.kernel_to_json(kern)
        bound = rkir.bind(to_ref(kj), [])
        seed = 17 + i
        rec = {"kernel": kj, "seed": seed, "needs_trajectories": rsim._needs_trajectories(bound.kernel)}
        try:
            rec["counts_512"] = rsim.sample(bound, 512, seed).counts
        except DegenerateNorm as e:
            rec["counts_512"] = None
            rec["sample_error"] = str(e)
        rec["shots"] = [traj_record(bound, seed, s, with_state=(s < 8)) for s in range(48)]
        dyn.append(rec)
    write("dynamic.json", dyn)

    # ---- pre-drawn uniform streams (north_star contract) + degenerate branch
    predrawn = []
    src, kern = workloads.dyn_circuit(n=6, layers=6, every=3, nmeas=2, seed=66)
    kj = ir.kernel_to_json(kern)
    bound = rkir.bind(to_ref(kj), [])
    urng = np.random.default_rng(5)
    for j in range(6):
        vals = [float(v) for v in urng.uniform(0, 1, 64)]
        predrawn.append({"kernel": kj, "values": vals, "record": traj_record(bound, 0, j, values=vals)})
    # p1 = sin^2(1e-9) ~ 1e-18 > 0 and u = 0.0 selects the 1 branch -> DegenerateNorm
    deg = ir.Kernel(1, [("q", 1)], [], [("c", 1)], [ir.Gate("rx", (2e-9,), (0,), ()), ir.Measure(0, ("c", 0))])
    kj = ir.kernel_to_json(deg)
    predrawn.append({"kernel": kj, "values": [0.0], "record": traj_record(rkir.bind(to_ref(kj), []), 0, 0, values=[0.0])})
    write("predrawn.json", predrawn)

    # ---- workload twins: DYN8, RDC10, VQE6, and the first DYN20 shots ------
    twins = {}
    src, kern = sources["dyn8"]
    kj = ir.kernel_to_json(kern)
    bound = rkir.bind(to_ref(kj), [])
    twins["dyn8"] = {"kernel": kj, "seed": 1234, "counts_1024": rsim.sample(bound, 1024, 1234).counts,
                     "shots": [traj_record(bound, 1234, s, with_state=(s < 4)) for s in range(64)]}
    src, kern = sources["rdc10"]
    kj = ir.kernel_to_json(kern)
    bound = rkir.bind(to_ref(kj), [])
    twins["rdc10"] = {"kernel": kj, "seed": 1234, "shots": [traj_record(bound, 1234, s, with_state=(s < 2)) for s in range(8)]}
    src, kern = sources["vqe6"]
    ham = workloads.vqe_hamiltonian(6, 20, seed=11599)
    pts = workloads.vqe_points(4, kern.total_params, seed=4096)
    kj = ir.kernel_to_json(kern)
    rk = to_ref(kj)
    energies, per_term = [], []
    for p in pts:
        sv = rsim.statevector(rkir.bind(rk, list(p)))
        vals = [rsim.expval_pauli(sv, w) for _, w in ham]
        per_term.append(vals)
        energies.append(float(sum(c * v for (c, _), v in zip(ham, vals))))
    twins["vqe6"] = {"kernel": kj, "hamiltonian": ham, "points": [list(map(float, p)) for p in pts],
                     "energies": energies, "per_term": per_term}
    src, kern = sources["dyn20"]
    bound = rkir.bind(rsuites.compile_source(src), [])
    recs = []
    for s in range(2):
        r = traj_record(bound, 1234, s, with_state=False)
        recs.append(r)
    twins["dyn20"] = {"seed": 1234, "shots": recs}
    write("twins.json", twins)
    print(f"done in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
