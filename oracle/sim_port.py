"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference simulator
`/root/reference/pkg/src/qasm2cudaq/sim.py` (the path the B200 backend replaces).
Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline / reference
arm may import this module, and only as the checker or the timed CPU baseline.
The product package (`paper_2604_11599_b200`) never imports it: its entry points
fail loudly when the CUDA library is missing.

Parity pin: `tests/golden/make_goldens.py` runs the real reference (importable in
the build container) on the golden workloads; `tests/test_oracle_goldens.py`
checks this port against those fixtures bit-for-bit (RNG words, histograms,
per-shot keys) and to 0 ulp on amplitudes for the recorded circuits.  The
arithmetic below deliberately follows the reference's numpy call sequence
(moveaxis + matmul, masked pairwise sum, sequential cumsum, vdot) so that the
rounding matches, which is what makes those comparisons exact.

The op objects are duck-typed by class name, so the reference's own kir
dataclasses and the mirror in `paper_2604_11599_b200.ir` both work.
"""

from __future__ import annotations

import math
from collections import Counter

import numpy as np

M64 = (1 << 64) - 1
PHI64 = 0x9E3779B97F4A7C15


# ---------------------------------------------------------------------------
# RNG  (sim.py:26-72)
# ---------------------------------------------------------------------------


def splitmix_step(x: int) -> tuple[int, int]:
    """One splitmix64 step: returns (advanced state, output)  (sim.py:30-35)."""
    x = (x + PHI64) & M64
    z = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return x, z ^ (z >> 31)


def rotl64(v: int, r: int) -> int:
    return ((v << r) | (v >> (64 - r))) & M64


class PortRng:
    """xoshiro256++ seeded by chained splitmix64 (sim.py:42-72)."""

    def __init__(self, seed: int):
        x = seed & M64  # negative seeds wrap two's-complement (sim.py:48)
        words = []
        for _ in range(4):
            x, out = splitmix_step(x)
            words.append(out)
        self.s = words

    @classmethod
    def for_shot(cls, seed: int, shot: int) -> "PortRng":
        # sim.py:54-57: derived = splitmix64(seed + (shot+1)*golden).output
        return cls(splitmix_step((seed + (shot + 1) * PHI64) & M64)[1])

    def next_u64(self) -> int:  # sim.py:59-68
        s0, s1, s2, s3 = self.s
        out = (rotl64((s0 + s3) & M64, 23) + s0) & M64
        t = (s1 << 17) & M64
        s2 ^= s0
        s3 ^= s1
        s1 ^= s2
        s0 ^= s3
        s2 ^= t
        s3 = rotl64(s3, 45)
        self.s = [s0, s1, s2, s3]
        return out

    def uniform(self) -> float:  # sim.py:70-72
        return (self.next_u64() >> 11) * 2.0**-53


class PredrawnStream:
    """A fixed list of uniforms consumed in order -- the 'same pre-drawn uniform
    stream' the north_star parity contract is stated on."""

    def __init__(self, values):
        self.values = list(values)
        self.pos = 0

    def uniform(self) -> float:
        u = self.values[self.pos]
        self.pos += 1
        return u


# ---------------------------------------------------------------------------
# Gate matrices  (sim.py:139-200)
# ---------------------------------------------------------------------------

_R2 = 1.0 / math.sqrt(2.0)
_C = np.complex128
FIXED = {
    "x": np.array([[0, 1], [1, 0]], dtype=_C),
    "y": np.array([[0, -1j], [1j, 0]], dtype=_C),
    "z": np.array([[1, 0], [0, -1]], dtype=_C),
    "h": np.array([[_R2, _R2], [_R2, -_R2]], dtype=_C),
    "s": np.array([[1, 0], [0, 1j]], dtype=_C),
    "t": np.array([[1, 0], [0, np.exp(1j * math.pi / 4)]], dtype=_C),
    "sx": 0.5 * np.array([[1 + 1j, 1 - 1j], [1 - 1j, 1 + 1j]], dtype=_C),
}
SWAP4 = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=_C)


def _is_ref(a) -> bool:
    return not isinstance(a, (int, float)) and hasattr(a, "slot")


def angles_of(op, params) -> tuple:
    """ParamRef slots read from the bound values (sim.py:186-187)."""
    return tuple(params[a.slot] if _is_ref(a) else a for a in op.angles)


def rotation(base: str, ang: tuple) -> np.ndarray:
    """Parametric bases (sim.py:156-183)."""
    if base in ("rx", "ry"):
        half = ang[0] / 2
        c, s = math.cos(half), math.sin(half)
        if base == "rx":
            return np.array([[c, -1j * s], [-1j * s, c]], dtype=_C)
        return np.array([[c, -s], [s, c]], dtype=_C)
    if base == "rz":
        th = ang[0]
        return np.array([[np.exp(-0.5j * th), 0], [0, np.exp(0.5j * th)]], dtype=_C)
    if base == "p":
        return np.array([[1, 0], [0, np.exp(1j * ang[0])]], dtype=_C)
    if base == "u":
        th, ph, la = ang
        c, s = math.cos(th / 2), math.sin(th / 2)
        return np.array(
            [[c, -np.exp(1j * la) * s], [np.exp(1j * ph) * s, np.exp(1j * (ph + la)) * c]],
            dtype=_C,
        )
    raise ValueError(f"no matrix for gate {base!r}")


def matrix_of(op, params=()) -> np.ndarray:
    """Target-space unitary, adjoint = conjugate transpose (sim.py:190-200)."""
    if op.base in FIXED:
        m = FIXED[op.base]
    elif op.base == "swap":
        m = SWAP4
    else:
        m = rotation(op.base, angles_of(op, params))
    return m.conj().T if op.adjoint else m


# ---------------------------------------------------------------------------
# State-vector passes  (sim.py:80-95, 203-259)
# ---------------------------------------------------------------------------


class PortState:
    """Dense complex128, qubit k = index bit k (sim.py:3, 80-95)."""

    def __init__(self, n: int, amps: np.ndarray | None = None):
        self.n = n
        if amps is None:
            amps = np.zeros(1 << n, dtype=_C)
            amps[0] = 1.0
        self.amps = amps

    def norm(self) -> float:
        a = self.amps
        return float(np.sqrt(np.sum(a.real**2 + a.imag**2)))

    def copy(self) -> "PortState":
        return PortState(self.n, self.amps.copy())


def unitary_pass(st: PortState, mat, targets, controls) -> None:
    """sim.py:203-221: tensor view, control axes then target axes to the front,
    polarity selection, (2^k, rest) matmul, write back."""
    n = st.n
    view = st.amps.reshape((2,) * n)
    axes = [n - 1 - q for q, _ in controls] + [n - 1 - q for q in targets]
    front = np.moveaxis(view, axes, range(len(axes)))
    pick = tuple(pol for _, pol in controls)
    sub = front[pick]
    k = len(targets)
    tail = sub.shape[k:]
    front[pick] = (mat @ sub.reshape(1 << k, -1)).reshape((2,) * k + tail)


def gate_pass(st: PortState, op, params=()) -> PortState:
    unitary_pass(st, matrix_of(op, params), op.targets, op.controls)
    return st


class DegenerateBranch(Exception):
    """Raised where the reference raises DegenerateNorm (sim.py:243-246)."""


def measure_pass(st: PortState, q: int, rng) -> tuple[int, float]:
    """sim.py:237-248: masked pairwise sum for p1, u < p1 decides, p0 = 1 - p1,
    zero the other branch, multiply by the reciprocal sqrt."""
    ones = (np.arange(st.amps.size) >> q) & 1 == 1
    p1 = float(np.sum(st.amps.real[ones] ** 2 + st.amps.imag[ones] ** 2))
    outcome = 1 if rng.uniform() < p1 else 0
    p_sel = p1 if outcome == 1 else 1.0 - p1
    if p_sel < 1e-15:
        raise DegenerateBranch(f"branch {outcome} on qubit {q} has probability {p_sel}")
    st.amps[ones != outcome] = 0.0
    st.amps *= 1.0 / math.sqrt(p_sel)
    return outcome, p1


def reset_pass(st: PortState, q: int, rng) -> int:
    """sim.py:254-259: measure without a store write, then x if the outcome was 1."""
    outcome, _ = measure_pass(st, q, rng)
    if outcome == 1:
        unitary_pass(st, FIXED["x"], (q,), ())
    return outcome


# ---------------------------------------------------------------------------
# Classical store and predicates  (sim.py:98-131, 262-276)
# ---------------------------------------------------------------------------


class PortStore:
    def __init__(self, layout):
        self.layout = [(n, int(w)) for n, w in layout]
        self.bits = {n: [0] * w for n, w in self.layout}

    def register_value(self, reg: str) -> int:  # bit 0 is the MSB (sim.py:111-116)
        v = 0
        for b in self.bits[reg]:
            v = (v << 1) | b
        return v

    def key(self) -> str:  # sim.py:118-119
        return "".join("1" if b else "0" for n, _ in self.layout for b in self.bits[n])


_CMP = {
    "==": lambda a, b: a == b,
    "!=": lambda a, b: a != b,
    "<": lambda a, b: a < b,
    "<=": lambda a, b: a <= b,
    ">": lambda a, b: a > b,
    ">=": lambda a, b: a >= b,
}


def predicate_value(pred, store: PortStore) -> bool:  # sim.py:262-276
    if pred.index is not None:
        v = store.bits[pred.register][pred.index]
    else:
        v = store.register_value(pred.register)
    if pred.comparator == "truthy":
        return v != 0
    return _CMP[pred.comparator](v, pred.rhs)


# ---------------------------------------------------------------------------
# Interpreter, sampling, statevector, Pauli expectation  (sim.py:279-430)
# ---------------------------------------------------------------------------


def _kind(op) -> str:
    return type(op).__name__


def exec_body(ops, st: PortState, store: PortStore, params, rng, trace=None, log=None) -> None:
    """Program-order interpreter (sim.py:279-303).  `log` (oracle-only) records
    (kind, qubit, outcome, p1) for every executed measure/reset."""
    for op in ops:
        k = _kind(op)
        if k == "Gate":
            gate_pass(st, op, params)
        elif k == "Measure":
            out, p1 = measure_pass(st, op.qubit, rng)
            store.bits[op.bit[0]][op.bit[1]] = out
            if log is not None:
                log.append(("measure", op.qubit, out, p1))
        elif k == "Reset":
            ones = (np.arange(st.amps.size) >> op.qubit) & 1 == 1
            p1 = float(np.sum(st.amps.real[ones] ** 2 + st.amps.imag[ones] ** 2))
            out = reset_pass(st, op.qubit, rng)
            if log is not None:
                log.append(("reset", op.qubit, out, p1))
        elif k == "Nop":
            continue
        elif k == "CondBlock":
            taken = predicate_value(op.predicate, store)
            if trace is not None:
                trace.append((op.predicate, {n: list(b) for n, b in store.bits.items()}, taken))
            exec_body(op.then_body if taken else op.else_body, st, store, params, rng, trace, log)
        else:
            raise TypeError(f"unknown op {op!r}")


def trajectory(bound, rng, trace=None, log=None) -> tuple[PortStore, PortState]:
    """sim.py:306-314."""
    k = bound.kernel
    st = PortState(k.qubit_count)
    store = PortStore(k.classical_layout)
    exec_body(k.body, st, store, bound.values, rng, trace, log)
    return store, st


def is_dynamic(kernel) -> bool:
    """sim.py:322-335 -- top-level scan only."""
    seen: set[int] = set()
    for op in kernel.body:
        k = _kind(op)
        if k in ("CondBlock", "Reset"):
            return True
        if k == "Measure":
            if op.qubit in seen:
                return True
            seen.add(op.qubit)
        elif k == "Gate" and seen:
            return True
    return False


def gates_only(bound) -> PortState:
    st = PortState(bound.kernel.qubit_count)
    for op in bound.kernel.body:
        if _kind(op) == "Gate":
            gate_pass(st, op, bound.values)
    return st


def static_keys(bound, shots: int, seed: int, shot_begin: int = 0) -> list[str]:
    """sim.py:354-369 per-shot keys: sequential cumsum, searchsorted(side=right),
    clamp to the last index, top-level measures written in order."""
    k = bound.kernel
    st = gates_only(bound)
    cdf = np.cumsum(st.amps.real**2 + st.amps.imag**2)
    ms = [op for op in k.body if _kind(op) == "Measure"]
    keys = []
    for shot in range(shot_begin, shot_begin + shots):
        u = PortRng.for_shot(seed, shot).uniform()
        idx = min(int(np.searchsorted(cdf, u, side="right")), cdf.size - 1)
        store = PortStore(k.classical_layout)
        for m in ms:
            store.bits[m.bit[0]][m.bit[1]] = (idx >> m.qubit) & 1
        keys.append(store.key())
    return keys


def trajectory_keys(bound, seed: int, shot_begin: int, shots: int) -> list[str]:
    return [
        trajectory(bound, PortRng.for_shot(seed, s))[0].key()
        for s in range(shot_begin, shot_begin + shots)
    ]


def sample_counts(bound, shots: int, seed: int) -> dict[str, int]:
    """sim.py:372-391 (single worker; the reference's result is worker-invariant)."""
    if shots < 1:
        raise ValueError("shots must be >= 1")
    if not is_dynamic(bound.kernel):
        return dict(Counter(static_keys(bound, shots, seed)))
    return dict(Counter(trajectory_keys(bound, seed, 0, shots)))


def final_state(bound) -> PortState:
    """sim.py:394-409; raises ValueError where the reference raises DynamicCircuit."""
    for op in bound.kernel.body:
        if _kind(op) in ("Measure", "CondBlock", "Reset"):
            raise ValueError("dynamic circuit")
    return gates_only(bound)


PAULI = {"I": np.eye(2, dtype=_C), "X": FIXED["x"], "Y": FIXED["y"], "Z": FIXED["z"]}


def pauli_expectation(st: PortState, word: str) -> float:
    """sim.py:420-430: copy, one full pass per non-identity letter (letter k acts
    on qubit k), then Re vdot."""
    if len(word) != st.n or any(ch not in PAULI for ch in word):
        raise ValueError(f"bad pauli string {word!r}")
    work = st.copy()
    for q, ch in enumerate(word):
        if ch != "I":
            unitary_pass(work, PAULI[ch], (q,), ())
    return float(np.vdot(st.amps, work.amps).real)


def observe(bound, terms) -> float:
    """E = sum_k c_k <P_k> on the static final state (the caller-side composition
    at suites.py:319-323 / cli.py:101-107; coefficients are not a reference type)."""
    st = final_state(bound)
    return float(sum(c * pauli_expectation(st, w) for c, w in terms))
