"""The benchmark circuits are exactly what the reference frontend lowers from
their OpenQASM text (hashes recorded by tests/golden/make_goldens.py)."""

import hashlib
import json

from paper_2604_11599_b200 import ir, workloads


def _hash(k):
    return hashlib.sha256(json.dumps(ir.kernel_to_json(k), sort_keys=True).encode()).hexdigest()


def test_workload_ir_matches_reference_lowering(golden):
    g = golden("workload_ir.json")
    made = dict(workloads.ff_suite())
    made["dyn20"] = workloads.dyn_circuit()
    made["dyn8"] = workloads.dyn_circuit(n=8, layers=10, every=5, nmeas=2, seed=8)
    made["vqe24"] = workloads.vqe_ansatz()
    made["vqe6"] = workloads.vqe_ansatz(6, 2)
    made["rdc30"] = workloads.rdc_circuit()
    made["rdc10"] = workloads.rdc_circuit(n=10, depth=40, every=20, seed=10)
    assert set(made) == set(g)
    for name, (_, k) in made.items():
        assert _hash(k) == g[name]["reference"], name


def test_dyn20_counts():
    _, k = workloads.dyn_circuit()
    gates = sum(1 for o in k.body if type(o).__name__ == "Gate")
    assert gates == 1180
    assert sum(1 for o in k.body if type(o).__name__ == "Measure") == 32
    assert sum(1 for o in k.body if type(o).__name__ == "Reset") == 32
    _, v = workloads.vqe_ansatz()
    assert len(v.body) == 568 and v.total_params == 384


def test_json_roundtrip():
    _, k = workloads.ff_teleport()
    assert ir.kernel_to_json(ir.kernel_from_json(ir.kernel_to_json(k))) == ir.kernel_to_json(k)
