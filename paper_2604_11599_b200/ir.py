"""Kernel-IR contract consumed by the B200 backend.

The backend's input is the reference's canonical op sequence
(`/root/reference/pkg/src/qasm2cudaq/kir.py:41-106`): `Gate`, `Measure`, `Reset`,
`Nop`, `CondBlock(Predicate, then, else)`, wrapped in a `Kernel` and bound to a flat
parameter vector by `bind` (`kir.py:272-278`).  Angles are floats or
`ParamRef(slot)` (`sema.py:83-87`).

Two kinds of object are accepted everywhere in this package:

* the reference's own dataclasses (a user running the `qasm2cudaq` frontend hands
  us `qasm2cudaq.kir.Kernel` objects directly -- this is the drop-in case), and
* the mirror dataclasses below, for hosts without the frontend (the GPU box,
  benchmarks, golden fixtures).

Dispatch is therefore by class *name* (`op_kind`), never by `isinstance` against
one particular module.  The JSON codec is the on-disk format of the golden
fixtures in `tests/golden/`.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any

from .errors import ArityMismatch

CANONICAL_BASES = frozenset("x y z h s t sx rx ry rz p u swap".split())  # kir.py:18
POS = 1  # kir.py:21 -- positive control fires on |1>
NEG = 0  # kir.py:22 -- negative control fires on |0>


@dataclass(frozen=True)
class ParamRef:
    """One slot of the flat runtime-parameter vector (sema.py:83-87)."""

    slot: int


@dataclass
class ParamSpec:
    """Parameter declaration (sema.py:92-98)."""

    name: str
    count: int
    array: bool
    offset: int


@dataclass
class Gate:
    base: str
    angles: tuple = ()
    targets: tuple = ()
    controls: tuple = ()  # ((qubit, POS|NEG), ...)
    adjoint: bool = False


@dataclass
class Measure:
    qubit: int
    bit: tuple  # (register, index)


@dataclass
class Reset:
    qubit: int


@dataclass
class Nop:
    qubits: tuple = ()


@dataclass
class Predicate:
    register: str
    index: int | None  # None: whole register, unsigned, bit 0 most significant
    comparator: str  # == != < <= > >= truthy
    rhs: int = 0


@dataclass
class CondBlock:
    predicate: Predicate
    then_body: list
    else_body: list


@dataclass
class Kernel:
    qubit_count: int
    qubit_layout: list = field(default_factory=list)
    param_layout: list = field(default_factory=list)
    classical_layout: list = field(default_factory=list)
    body: list = field(default_factory=list)

    @property
    def total_params(self) -> int:
        return sum(p.count for p in self.param_layout)


@dataclass
class BoundKernel:
    kernel: Any
    values: tuple


def bind(kernel, values) -> BoundKernel:
    """Attach parameter values without re-lowering (kir.py:272-278)."""
    total = sum(p.count for p in kernel.param_layout)
    if len(values) != total:
        raise ArityMismatch(f"kernel takes {total} parameter value(s), got {len(values)}")
    return BoundKernel(kernel, tuple(float(v) for v in values))


# ---------------------------------------------------------------------------
# duck typing over reference / mirror objects
# ---------------------------------------------------------------------------

_KINDS = {
    "Gate": "gate",
    "Measure": "measure",
    "Reset": "reset",
    "Nop": "nop",
    "CondBlock": "cond",
}


def op_kind(op) -> str:
    kind = _KINDS.get(type(op).__name__)
    if kind is None:
        raise TypeError(f"unknown op {op!r}")
    return kind


def is_param_ref(a) -> bool:
    return not isinstance(a, (int, float)) and hasattr(a, "slot")


# ---------------------------------------------------------------------------
# JSON codec (golden fixtures)
# ---------------------------------------------------------------------------


def _angle_to_json(a):
    return {"slot": int(a.slot)} if is_param_ref(a) else float(a)


def _angle_from_json(a):
    return ParamRef(int(a["slot"])) if isinstance(a, dict) else float(a)


def op_to_json(op) -> dict:
    kind = op_kind(op)
    if kind == "gate":
        return {
            "op": "gate",
            "base": op.base,
            "angles": [_angle_to_json(a) for a in op.angles],
            "targets": [int(t) for t in op.targets],
            "controls": [[int(q), int(p)] for q, p in op.controls],
            "adjoint": bool(op.adjoint),
        }
    if kind == "measure":
        return {"op": "measure", "qubit": int(op.qubit), "bit": [op.bit[0], int(op.bit[1])]}
    if kind == "reset":
        return {"op": "reset", "qubit": int(op.qubit)}
    if kind == "nop":
        return {"op": "nop", "qubits": [int(q) for q in op.qubits]}
    p = op.predicate
    return {
        "op": "cond",
        "pred": {"register": p.register, "index": p.index, "comparator": p.comparator, "rhs": int(p.rhs)},
        "then": [op_to_json(o) for o in op.then_body],
        "else": [op_to_json(o) for o in op.else_body],
    }


def op_from_json(d: dict):
    kind = d["op"]
    if kind == "gate":
        return Gate(
            d["base"],
            tuple(_angle_from_json(a) for a in d["angles"]),
            tuple(d["targets"]),
            tuple((int(q), int(p)) for q, p in d["controls"]),
            bool(d["adjoint"]),
        )
    if kind == "measure":
        return Measure(int(d["qubit"]), (d["bit"][0], int(d["bit"][1])))
    if kind == "reset":
        return Reset(int(d["qubit"]))
    if kind == "nop":
        return Nop(tuple(d["qubits"]))
    if kind == "cond":
        p = d["pred"]
        return CondBlock(
            Predicate(p["register"], p["index"], p["comparator"], int(p["rhs"])),
            [op_from_json(o) for o in d["then"]],
            [op_from_json(o) for o in d["else"]],
        )
    raise ValueError(f"unknown op kind {kind!r}")


def kernel_to_json(kernel) -> dict:
    return {
        "qubit_count": int(kernel.qubit_count),
        "qubit_layout": [[n, int(w)] for n, w in kernel.qubit_layout],
        "param_layout": [[p.name, int(p.count), bool(p.array), int(p.offset)] for p in kernel.param_layout],
        "classical_layout": [[n, int(w)] for n, w in kernel.classical_layout],
        "body": [op_to_json(o) for o in kernel.body],
    }


def kernel_from_json(d: dict) -> Kernel:
    return Kernel(
        qubit_count=int(d["qubit_count"]),
        qubit_layout=[(n, int(w)) for n, w in d["qubit_layout"]],
        param_layout=[ParamSpec(n, int(c), bool(a), int(o)) for n, c, a, o in d["param_layout"]],
        classical_layout=[(n, int(w)) for n, w in d["classical_layout"]],
        body=[op_from_json(o) for o in d["body"]],
    )
