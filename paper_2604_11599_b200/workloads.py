"""Synthetic workloads of BASELINE.json's configs.

Every generator returns both the OpenQASM 3.0 source text (what a user would feed
the reference frontend, `suites.compile_source`, `suites.py:67-69`) and the
kernel IR that lowering produces for it, built directly so that hosts without the
frontend (the GPU box) can run the same circuits.  `tests/golden/make_goldens.py`
compiles the text with the real frontend and `tests/test_workloads.py` checks the
two IRs are identical, so the benchmark circuits are exactly the reference's.

Configs:
  FF1..FF6  IBM feedforward guide suite, <=5 qubits (cfg 1)
  dyn       DYN20: layered u/cx circuit with measure + conditional-x + reset rounds (cfg 2)
  vqe       VQE24 hardware-efficient ansatz + 200-term Pauli Hamiltonian (cfg 3)
  rdc       RDC30 random dynamic circuit (cfg 4/5)
"""

from __future__ import annotations

import math
import random

from .ir import POS, CondBlock, Gate, Kernel, Measure, ParamRef, ParamSpec, Predicate, Reset

HEADER = 'OPENQASM 3.0;\ninclude "stdgates.inc";\n'


def _x(q):
    return Gate("x", (), (q,), ())


def _h(q):
    return Gate("h", (), (q,), ())


def _z(q):
    return Gate("z", (), (q,), ())


def _cx(c, t):
    return Gate("x", (), (t,), ((c, POS),))


def _eq(reg, idx, rhs):
    return Predicate(reg, idx, "==", rhs)


# ---------------------------------------------------------------------------
# cfg 1: feedforward suite
# ---------------------------------------------------------------------------


def ff_reset(prep_minus: bool):
    """FF1/FF2: suites._reset_source (suites.py:90-101) with the |+> / |-> prep."""
    prep = "x q; h q;" if prep_minus else "h q;"
    src = f"{HEADER}qubit q;\nbit c;\n{prep}\nc = measure q;\nif (c == 1) {{ x q; }}\nc = measure q;\n"
    body = ([_x(0)] if prep_minus else []) + [
        _h(0),
        Measure(0, ("c", 0)),
        CondBlock(_eq("c", 0, 1), [_x(0)], []),
        Measure(0, ("c", 0)),
    ]
    return src, Kernel(1, [("q", 1)], [], [("c", 1)], body)


def ff_ifelse():
    """FF3: golden `ifelse` (golden_cases.py:38-46) + a second bit reading q[1]."""
    src = (
        f"{HEADER}qubit[2] q;\nbit c;\nbit d;\nh q[0];\nc = measure q[0];\n"
        "if (c == 1) { x q[1]; z q[1]; } else { h q[1]; }\nd = measure q[1];\n"
    )
    body = [
        _h(0),
        Measure(0, ("c", 0)),
        CondBlock(_eq("c", 0, 1), [_x(1), _z(1)], [_h(1)]),
        Measure(1, ("d", 0)),
    ]
    return src, Kernel(2, [("q", 2)], [], [("c", 1), ("d", 1)], body)


def ff_multibit():
    """FF4: golden `registerpred` (golden_cases.py:47-56) + `r = measure q[0]`."""
    src = (
        f"{HEADER}qubit[3] q;\nbit[3] c;\nbit r;\nh q;\nc = measure q;\n"
        "if (c >= 5) { x q[0]; }\nif (c) { z q[1]; }\nr = measure q[0];\n"
    )
    body = [_h(0), _h(1), _h(2)]
    body += [Measure(i, ("c", i)) for i in range(3)]
    body += [
        CondBlock(Predicate("c", None, ">=", 5), [_x(0)], []),
        CondBlock(Predicate("c", None, "truthy", 0), [_z(1)], []),
        Measure(0, ("r", 0)),
    ]
    return src, Kernel(3, [("q", 3)], [], [("c", 3), ("r", 1)], body)


def ff_sequential():
    """FF5: sequential feedforward chain over 5 qubits."""
    src = (
        f"{HEADER}qubit[5] q;\nbit[5] c;\nh q[0];\n"
        "c[0] = measure q[0];\nif (c[0] == 1) { x q[1]; }\n"
        "c[1] = measure q[1];\nif (c[1] == 1) { h q[2]; }\n"
        "c[2] = measure q[2];\nif (c[2] == 1) { x q[3]; } else { h q[3]; }\n"
        "c[3] = measure q[3];\nif (c[3]) { x q[4]; }\n"
        "c[4] = measure q[4];\n"
    )
    body = [
        _h(0),
        Measure(0, ("c", 0)),
        CondBlock(_eq("c", 0, 1), [_x(1)], []),
        Measure(1, ("c", 1)),
        CondBlock(_eq("c", 1, 1), [_h(2)], []),
        Measure(2, ("c", 2)),
        CondBlock(_eq("c", 2, 1), [_x(3)], [_h(3)]),
        Measure(3, ("c", 3)),
        CondBlock(Predicate("c", 3, "truthy", 0), [_x(4)], []),
        Measure(4, ("c", 4)),
    ]
    return src, Kernel(5, [("q", 5)], [], [("c", 5)], body)


def ff_teleport(seed: int = 1234, corrections: bool = True):
    """FF6: suites._teleport_source (suites.py:133-154) with the suite's seeded
    angles (suites.py:162-165)."""
    rng = random.Random(seed)
    th = rng.uniform(0, math.pi)
    ph = rng.uniform(0, 2 * math.pi)
    la = rng.uniform(0, 2 * math.pi)
    fix = "if (c1 == 1) { x q[2]; }\nif (c0 == 1) { z q[2]; }\n" if corrections else ""
    src = (
        f"{HEADER}qubit[3] q;\nbit c0;\nbit c1;\nbit res;\n"
        f"u({th!r}, {ph!r}, {la!r}) q[0];\nh q[1];\ncx q[1], q[2];\ncx q[0], q[1];\nh q[0];\n"
        f"c0 = measure q[0];\nc1 = measure q[1];\n{fix}"
        f"u({-th!r}, {-la!r}, {-ph!r}) q[2];\nres = measure q[2];\n"
    )
    body = [
        Gate("u", (th, ph, la), (0,), ()),
        _h(1),
        _cx(1, 2),
        _cx(0, 1),
        _h(0),
        Measure(0, ("c0", 0)),
        Measure(1, ("c1", 0)),
    ]
    if corrections:
        body += [CondBlock(_eq("c1", 0, 1), [_x(2)], []), CondBlock(_eq("c0", 0, 1), [_z(2)], [])]
    body += [Gate("u", (-th, -la, -ph), (2,), ()), Measure(2, ("res", 0))]
    return src, Kernel(3, [("q", 3)], [], [("c0", 1), ("c1", 1), ("res", 1)], body)


def ff_suite() -> dict:
    return {
        "FF1_reset_plus": ff_reset(False),
        "FF2_reset_minus": ff_reset(True),
        "FF3_ifelse": ff_ifelse(),
        "FF4_multibit": ff_multibit(),
        "FF5_sequential": ff_sequential(),
        "FF6_teleport": ff_teleport(),
    }


# ---------------------------------------------------------------------------
# cfg 2: DYN20
# ---------------------------------------------------------------------------


def dyn_circuit(n: int = 20, layers: int = 40, every: int = 5, nmeas: int = 4, seed: int = 2604):
    """Layers of u(a,b,c) on every qubit + a brick of cx; after every `every`-th
    layer a round of, for k < nmeas: measure q[k] -> c, if (c==1) x q[k], reset
    q[nmeas+k].  Defaults are DYN20 (SURVEY.md §8(d) cfg 2): 1180 gates, 32
    measures, 32 resets, 64 draws per trajectory."""
    assert n >= 2 * nmeas
    rng = random.Random(seed)
    rounds = layers // every
    width = nmeas * rounds
    lines = [f"qubit[{n}] q;", f"bit[{width}] c;"]
    body = []
    r = 0
    for layer in range(layers):
        for q in range(n):
            a, b, c = (rng.uniform(-math.pi, math.pi) for _ in range(3))
            lines.append(f"u({a!r}, {b!r}, {c!r}) q[{q}];")
            body.append(Gate("u", (a, b, c), (q,), ()))
        start = 0 if layer % 2 == 0 else 1
        for ctl in range(start, n - 1, 2):
            lines.append(f"cx q[{ctl}], q[{ctl + 1}];")
            body.append(_cx(ctl, ctl + 1))
        if (layer + 1) % every == 0:
            for k in range(nmeas):
                bit = nmeas * r + k
                lines.append(f"c[{bit}] = measure q[{k}];")
                lines.append(f"if (c[{bit}] == 1) {{ x q[{k}]; }}")
                lines.append(f"reset q[{nmeas + k}];")
                body.append(Measure(k, ("c", bit)))
                body.append(CondBlock(_eq("c", bit, 1), [_x(k)], []))
                body.append(Reset(nmeas + k))
            r += 1
    src = HEADER + "\n".join(lines) + "\n"
    return src, Kernel(n, [("q", n)], [], [("c", width)], body)


# ---------------------------------------------------------------------------
# cfg 3: VQE24
# ---------------------------------------------------------------------------


def vqe_ansatz(n: int = 24, layers: int = 8):
    """Hardware-efficient ansatz: per layer ry(theta) x n, rz(theta) x n, cx chain."""
    total = 2 * n * layers
    lines = [f"input array[float[64], {total}] theta;", f"qubit[{n}] q;"]
    body = []
    for layer in range(layers):
        base = 2 * n * layer
        for q in range(n):
            lines.append(f"ry(theta[{base + q}]) q[{q}];")
            body.append(Gate("ry", (ParamRef(base + q),), (q,), ()))
        for q in range(n):
            lines.append(f"rz(theta[{base + n + q}]) q[{q}];")
            body.append(Gate("rz", (ParamRef(base + n + q),), (q,), ()))
        for q in range(n - 1):
            lines.append(f"cx q[{q}], q[{q + 1}];")
            body.append(_cx(q, q + 1))
    src = HEADER + "\n".join(lines) + "\n"
    return src, Kernel(n, [("q", n)], [ParamSpec("theta", total, True, 0)], [], body)


def vqe_hamiltonian(n: int = 24, terms: int = 200, seed: int = 11599) -> list:
    """[(coef, pauli_word)], locality U{1..4}, letter q acts on qubit q."""
    rng = random.Random(seed)
    out = []
    for _ in range(terms):
        k = rng.randint(1, min(4, n))
        qs = rng.sample(range(n), k)
        word = ["I"] * n
        for q in qs:
            word[q] = rng.choice("XYZ")
        out.append((rng.uniform(-1.0, 1.0), "".join(word)))
    return out


def vqe_points(npoints: int = 4096, nparams: int = 384, seed: int = 4096):
    import numpy as np

    return np.random.default_rng(seed).uniform(-math.pi, math.pi, (npoints, nparams))


# ---------------------------------------------------------------------------
# cfg 4/5: random dynamic circuit
# ---------------------------------------------------------------------------

_RDC_1Q = ("h", "sx", "t", "rx", "ry", "rz")


def rdc_circuit(n: int = 30, depth: int = 200, every: int = 20, seed: int = 30200):
    """Per layer a random 1q gate on every qubit and cx on a random perfect
    matching; every `every` layers measure 3 random qubits a, b, d, conditionally
    flip a, reset b (SURVEY.md §8(d) cfg 4)."""
    assert n >= 3
    rng = random.Random(seed)
    rounds = depth // every
    width = 3 * rounds
    lines = [f"qubit[{n}] q;", f"bit[{width}] c;"]
    body = []
    r = 0
    for layer in range(depth):
        for q in range(n):
            g = rng.choice(_RDC_1Q)
            if g in ("rx", "ry", "rz"):
                th = rng.uniform(-math.pi, math.pi)
                lines.append(f"{g}({th!r}) q[{q}];")
                body.append(Gate(g, (th,), (q,), ()))
            else:
                lines.append(f"{g} q[{q}];")
                body.append(Gate(g, (), (q,), ()))
        perm = list(range(n))
        rng.shuffle(perm)
        for i in range(n // 2):
            a, b = perm[2 * i], perm[2 * i + 1]
            lines.append(f"cx q[{a}], q[{b}];")
            body.append(_cx(a, b))
        if (layer + 1) % every == 0:
            a, b, d = rng.sample(range(n), 3)
            for j, q in enumerate((a, b, d)):
                lines.append(f"c[{3 * r + j}] = measure q[{q}];")
                body.append(Measure(q, ("c", 3 * r + j)))
            lines.append(f"if (c[{3 * r}] == 1) {{ x q[{a}]; }}")
            body.append(CondBlock(_eq("c", 3 * r, 1), [_x(a)], []))
            lines.append(f"reset q[{b}];")
            body.append(Reset(b))
            r += 1
    src = HEADER + "\n".join(lines) + "\n"
    return src, Kernel(n, [("q", n)], [], [("c", width)], body)


# ---------------------------------------------------------------------------
# random static circuits over every canonical base (parity fuzz)
# ---------------------------------------------------------------------------


def random_static(n: int, gates: int, seed: int, nparams: int = 0, max_controls: int = 2):
    """IR-only generator covering x y z h s t sx rx ry rz p u swap, adjoint,
    positive and negative controls and ParamRef angles."""
    rng = random.Random(seed)
    body = []
    for _ in range(gates):
        base = rng.choice(sorted(("x", "y", "z", "h", "s", "t", "sx", "rx", "ry", "rz", "p", "u", "swap")))
        nt = 2 if base == "swap" else 1
        if n < nt:
            base, nt = "h", 1
        nc = rng.randint(0, min(max_controls, n - nt))
        qs = rng.sample(range(n), nt + nc)
        targets = tuple(qs[:nt])
        controls = tuple((q, rng.choice((0, 1))) for q in qs[nt:])
        arity = {"rx": 1, "ry": 1, "rz": 1, "p": 1, "u": 3}.get(base, 0)
        angles = []
        for _ in range(arity):
            if nparams and rng.random() < 0.5:
                angles.append(ParamRef(rng.randrange(nparams)))
            else:
                angles.append(rng.uniform(-math.pi, math.pi))
        body.append(Gate(base, tuple(angles), targets, controls, rng.random() < 0.3))
    layout = [ParamSpec("theta", nparams, True, 0)] if nparams else []
    return Kernel(n, [("q", n)], layout, [], body)


def random_dynamic(n: int, ops: int, seed: int, nbits: int = 6, depth: int = 2):
    """IR-only generator of dynamic circuits: gates, measures into a register,
    resets, barriers, and (nested) if/else on single bits or the whole register
    with every comparator.  Predicates only read bits already written on every
    path (the lowering rule of kir.py:228-255)."""
    rng = random.Random(seed)
    from .ir import Nop

    def gate():
        g = random_static(n, 1, rng.randrange(1 << 30), max_controls=1).body[0]
        return g

    def block(count, written, level):
        out = []
        for _ in range(count):
            r = rng.random()
            if r < 0.55:
                out.append(gate())
            elif r < 0.72:
                b = rng.randrange(nbits)
                out.append(Measure(rng.randrange(n), ("c", b)))
                written.add(b)
            elif r < 0.8:
                out.append(Reset(rng.randrange(n)))
            elif r < 0.83:
                out.append(Nop(()))
            elif written and level < depth:
                if len(written) == nbits and rng.random() < 0.4:
                    cmp = rng.choice(("==", "!=", "<", "<=", ">", ">=", "truthy"))
                    pred = Predicate("c", None, cmp, rng.randrange(1 << nbits))
                    reads = set(range(nbits))
                else:
                    b = rng.choice(sorted(written))
                    cmp = rng.choice(("==", "!=", "truthy"))
                    pred = Predicate("c", b, cmp, rng.randrange(2))
                    reads = {b}
                tw, ew = set(written), set(written)
                then = block(rng.randint(1, 3), tw, level + 1)
                other = block(rng.randint(0, 2), ew, level + 1) if rng.random() < 0.5 else []
                # a body may not measure into a bit its own predicate reads (kir.py:248-253)
                then = [o for o in then if not (type(o).__name__ == "Measure" and o.bit[1] in reads)]
                other = [o for o in other if not (type(o).__name__ == "Measure" and o.bit[1] in reads)]
                out.append(CondBlock(pred, then, other))
                written |= tw & ew
            else:
                out.append(gate())
        return out

    body = block(ops, set(), 0)
    return Kernel(n, [("q", n)], [], [("c", nbits)], body)
