"""CPU-side checks of the drop-in boundary (no GPU needed).

* the sm_100a library exists, loads, and exports every symbol include/qsb.h declares;
* the ctypes record layout matches the C struct;
* the Python host mirror reproduces the reference's host-side logic (RNG streams,
  _needs_trajectories, predicates, gate matrices) exactly -- pinned to goldens.
"""

import os
import re

import numpy as np
import pytest

from paper_2604_11599_b200 import _lib, ir, sim, workloads

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(REPO, "include", "qsb.h")).read()
    return sorted(set(re.findall(r"^\S[^(;]*?\b(qsb_\w+)\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = _declared()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.EXPORTED)
    assert lib.qsb_abi_version() == 1


def test_library_is_sm100a():
    path = _lib.LIB_PATH
    data = open(path, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_op_record_layout_matches_header():
    assert _lib.OP_DTYPE.itemsize == 176
    src = open(os.path.join(REPO, "include", "qsb.h")).read()
    assert "uint64_t pred_rhs;" in src


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2604_11599_b200.errors import BackendError

    _, k = workloads.ff_teleport()
    with pytest.raises(BackendError):
        sim.sample(ir.bind(k, []), 16, 1)


def test_rng_known_answers(golden):
    g = golden("rng.json")
    r = sim.RngStream(42)
    assert [str(x) for x in (r.s0, r.s1, r.s2, r.s3)] == g["seed42_state"]
    assert [str(r.next_u64()) for _ in range(8)] == g["seed42_words"]
    for case in g["for_shot"]:
        r = sim.RngStream.for_shot(case["seed"], case["shot"])
        assert [str(x) for x in (r.s0, r.s1, r.s2, r.s3)] == case["state"]
        assert [r.uniform() for _ in range(6)] == case["uniforms"]


def test_needs_trajectories_rule(golden):
    for case in golden("dynamic.json"):
        k = ir.kernel_from_json(case["kernel"])
        assert sim._needs_trajectories(k) == case["needs_trajectories"]
    for case in golden("static_sampling.json"):
        assert not sim._needs_trajectories(ir.kernel_from_json(case["kernel"]))


def test_gate_matrix_matches_oracle():
    from oracle import sim_port as P

    k = workloads.random_static(4, 300, seed=9, nparams=3)
    vals = (0.3, -1.2, 2.5)
    for op in k.body:
        np.testing.assert_array_equal(sim.gate_matrix(op, vals), P.matrix_of(op, vals))


def test_predicate_eval():
    st = sim.ClassicalStore([("c", 3), ("d", 1)])
    st.write_bit("c", 0, 1)
    st.write_bit("c", 2, 1)
    assert st.register_uint("c") == 5
    assert sim._eval_predicate(ir.Predicate("c", None, ">=", 5), st)
    assert not sim._eval_predicate(ir.Predicate("c", None, ">", 5), st)
    assert sim._eval_predicate(ir.Predicate("c", 0, "truthy"), st)
    assert st.key() == "1010"


def test_tape_records_encode_predicates():
    rec = np.zeros(1, dtype=_lib.OP_DTYPE)
    sim._pred_record(rec[0], ir.Predicate("c", None, "==", 1 << 70), {"c": (0, 4)})
    assert rec["pred_cmp"][0] == _lib.CMP["<"] and rec["pred_rhs"][0] == 0  # never true
    sim._pred_record(rec[0], ir.Predicate("c", 2, "!=", 1), {"c": (3, 4)})
    assert rec["pred_bit"][0] == 5 and rec["pred_width"][0] == 1
