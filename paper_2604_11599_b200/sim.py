"""Drop-in replacement for `qasm2cudaq.sim` (reference: /root/reference/pkg/src/
qasm2cudaq/sim.py) executing on B200 through the sm_100a C ABI (include/qsb.h).

Same names, signatures, return types, error classes and RNG streams as the
reference simulator target:

    sample(bound, shots, seed, workers=1) -> ShotHistogram          sim.py:372-391
    statevector(bound) -> StateVector                               sim.py:402-409
    expval_pauli(state, pauli) -> float                             sim.py:420-430
    run_trajectory(bound, rng, trace=None) -> (store, state)        sim.py:306-314
    apply_gate / measure / reset on StateVector objects             sim.py:224-259
    RngStream, StateVector, ClassicalStore, ShotHistogram           sim.py:42-131
    gate_matrix, resolve_angles, _needs_trajectories, _eval_predicate, _exec_ops

plus `observe(bound_or_kernel, hamiltonian, points=None)` (batched energies, the
caller-side composition of suites.py:319-323) and keyword extensions
(`precision="c64"`, `device=`).

The computation never runs on the host: every state pass, reduction and sample
is a CUDA kernel.  Host work is limited to compiling the Kernel IR into a tape
once per Kernel, RNG bookkeeping for the per-op API, and rendering histogram
keys.  Without the library / a B200 every call raises NativeLibraryMissing or
BackendError.
"""

from __future__ import annotations

import ctypes
import math
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import BackendError, BadPauliString, DegenerateNorm, DynamicCircuit, SimError
from .ir import op_kind

__all__ = [
    "RngStream",
    "StateVector",
    "ClassicalStore",
    "ShotHistogram",
    "gate_matrix",
    "resolve_angles",
    "apply_gate",
    "measure",
    "reset",
    "run_trajectory",
    "sample",
    "statevector",
    "expval_pauli",
    "observe",
    "compile_tape",
    "last_stats",
    "set_default_precision",
]

_DEFAULT = {"precision": "c128", "device": None}


def set_default_precision(precision: str) -> None:
    """'c128' (default; the reference's arithmetic) or 'c64'."""
    if precision not in ("c128", "c64"):
        raise ValueError(precision)
    _DEFAULT["precision"] = precision


def _prec(precision) -> int:
    p = precision or _DEFAULT["precision"]
    if p not in ("c128", "c64"):
        raise ValueError(f"precision must be 'c128' or 'c64', not {p!r}")
    return _lib.C64 if p == "c64" else _lib.C128


def _ctx(device=None) -> _lib.Context:
    return _lib.context(device if device is not None else _DEFAULT["device"])


def last_stats(device=None) -> dict:
    """Device counters of the last run on `device` (launches, passes, CUDA-event
    times, algorithmic pass bytes, logical gate updates, tie-band decisions)."""
    return _ctx(device).stats()


# ---------------------------------------------------------------------------
# RNG (sim.py:26-72): host copy of the stream, used by the per-op API; the batched
# paths run the identical generator on the device.
# ---------------------------------------------------------------------------

_M64 = (1 << 64) - 1
_PHI = 0x9E3779B97F4A7C15


def _mix(x: int) -> tuple[int, int]:
    x = (x + _PHI) & _M64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return x, z ^ (z >> 31)


class RngStream:
    """xoshiro256++ seeded by chained splitmix64; RngStream.for_shot(seed, shot)
    derives the per-shot stream exactly as the reference does."""

    __slots__ = ("s0", "s1", "s2", "s3")

    def __init__(self, seed: int):
        x = seed & _M64
        x, self.s0 = _mix(x)
        x, self.s1 = _mix(x)
        x, self.s2 = _mix(x)
        x, self.s3 = _mix(x)

    @classmethod
    def for_shot(cls, seed: int, shot: int) -> "RngStream":
        return cls(_mix((seed + (shot + 1) * _PHI) & _M64)[1])

    def next_u64(self) -> int:
        s0, s1, s2, s3 = self.s0, self.s1, self.s2, self.s3
        out = ((((s0 + s3) & _M64) << 23 | ((s0 + s3) & _M64) >> 41) & _M64)
        out = (out + s0) & _M64
        t = (s1 << 17) & _M64
        s2 ^= s0
        s3 ^= s1
        s1 ^= s2
        s0 ^= s3
        s2 ^= t
        s3 = ((s3 << 45) | (s3 >> 19)) & _M64
        self.s0, self.s1, self.s2, self.s3 = s0, s1, s2, s3
        return out

    def uniform(self) -> float:
        return (self.next_u64() >> 11) * 2.0**-53


def _rng_words(rng):
    """4 state words if `rng` is an xoshiro stream (ours or the reference's)."""
    if all(hasattr(rng, a) for a in ("s0", "s1", "s2", "s3")):
        return np.array([rng.s0, rng.s1, rng.s2, rng.s3], dtype=np.uint64)
    return None


# ---------------------------------------------------------------------------
# Classical store / histogram (sim.py:98-131)
# ---------------------------------------------------------------------------


class ClassicalStore:
    """Bit registers; never-written bits read as 0."""

    def __init__(self, layout):
        self.layout = [(n, int(w)) for n, w in layout]
        self.bits = {name: [0] * width for name, width in self.layout}

    def write_bit(self, register: str, index: int, value: int) -> None:
        self.bits[register][index] = value

    def read_bit(self, register: str, index: int) -> int:
        return self.bits[register][index]

    def register_uint(self, register: str) -> int:
        """Register as unsigned integer, bit 0 most significant."""
        v = 0
        for b in self.bits[register]:
            v = (v << 1) | b
        return v

    def key(self) -> str:
        return "".join(str(b) for name, _ in self.layout for b in self.bits[name])

    @classmethod
    def _from_words(cls, layout, words: np.ndarray) -> "ClassicalStore":
        st = cls(layout)
        f = 0
        for name, width in st.layout:
            for i in range(width):
                st.bits[name][i] = int((int(words[f >> 6]) >> (f & 63)) & 1)
                f += 1
        return st


@dataclass
class ShotHistogram:
    counts: dict
    total_shots: int

    def sorted_items(self) -> list:
        return sorted(self.counts.items())

    def probability(self, key: str) -> float:
        return self.counts.get(key, 0) / self.total_shots


# ---------------------------------------------------------------------------
# Gate matrices (sim.py:139-200) -- built on the host with the reference's numpy
# expressions so literal-angle matrices are bit-identical to the reference's.
# ---------------------------------------------------------------------------

_H = 1.0 / math.sqrt(2.0)
_CT = np.complex128
_FIXED = {
    "x": np.array([[0, 1], [1, 0]], dtype=_CT),
    "y": np.array([[0, -1j], [1j, 0]], dtype=_CT),
    "z": np.array([[1, 0], [0, -1]], dtype=_CT),
    "h": np.array([[_H, _H], [_H, -_H]], dtype=_CT),
    "s": np.array([[1, 0], [0, 1j]], dtype=_CT),
    "t": np.array([[1, 0], [0, np.exp(1j * math.pi / 4)]], dtype=_CT),
    "sx": 0.5 * np.array([[1 + 1j, 1 - 1j], [1 - 1j, 1 + 1j]], dtype=_CT),
}
_SWAP = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=_CT)


def _param_matrix(base: str, a: tuple) -> np.ndarray:
    if base == "rx":
        c, s = math.cos(a[0] / 2), math.sin(a[0] / 2)
        return np.array([[c, -1j * s], [-1j * s, c]], dtype=_CT)
    if base == "ry":
        c, s = math.cos(a[0] / 2), math.sin(a[0] / 2)
        return np.array([[c, -s], [s, c]], dtype=_CT)
    if base == "rz":
        return np.array([[np.exp(-0.5j * a[0]), 0], [0, np.exp(0.5j * a[0])]], dtype=_CT)
    if base == "p":
        return np.array([[1, 0], [0, np.exp(1j * a[0])]], dtype=_CT)
    if base == "u":
        th, ph, la = a
        c, s = math.cos(th / 2), math.sin(th / 2)
        return np.array(
            [[c, -np.exp(1j * la) * s], [np.exp(1j * ph) * s, np.exp(1j * (ph + la)) * c]], dtype=_CT
        )
    raise SimError(f"no matrix for gate '{base}'")


def _is_ref(a) -> bool:
    return not isinstance(a, (int, float)) and hasattr(a, "slot")


def resolve_angles(op, params=()) -> tuple:
    return tuple(params[a.slot] if _is_ref(a) else a for a in op.angles)


def gate_matrix(op, params=()) -> np.ndarray:
    """Unitary of the canonical gate on its targets (controls excluded)."""
    if op.base in _FIXED:
        m = _FIXED[op.base]
    elif op.base == "swap":
        m = _SWAP
    else:
        m = _param_matrix(op.base, resolve_angles(op, params))
    return m.conj().T if op.adjoint else m


# ---------------------------------------------------------------------------
# Kernel IR -> tape (compile once per Kernel; bind supplies only values)
# ---------------------------------------------------------------------------


def _classical_offsets(layout) -> dict:
    off, out = 0, {}
    for name, width in layout:
        out[name] = (off, int(width))
        off += int(width)
    return out


def _gate_record(rec, op, params_known: bool) -> None:
    rec["kind"] = _lib.OP_GATE
    if op.base not in _lib.BASES:
        raise SimError(f"no matrix for gate '{op.base}'")
    rec["base"] = _lib.BASES[op.base]
    rec["adjoint"] = 1 if op.adjoint else 0
    nt = len(op.targets)
    rec["ntargets"] = nt
    rec["target"][:nt] = op.targets
    cm = cv = 0
    for q, pol in op.controls:
        cm |= 1 << q
        if pol:
            cv |= 1 << q
    rec["ctrl_mask"] = cm
    rec["ctrl_val"] = cv
    rec["angle_slot"][:] = -1
    symbolic = False
    for j, a in enumerate(op.angles):
        if _is_ref(a):
            rec["angle_slot"][j] = a.slot
            symbolic = True
        else:
            rec["angle"][j] = float(a)
    if not symbolic:
        m = gate_matrix(op)
        if op.base != "swap":
            rec["mat"][:] = [m[0, 0].real, m[0, 0].imag, m[0, 1].real, m[0, 1].imag,
                             m[1, 0].real, m[1, 0].imag, m[1, 1].real, m[1, 1].imag]
        rec["has_matrix"] = 1


_ALWAYS = (_lib.CMP[">="], 0)  # v >= 0
_NEVER = (_lib.CMP["<"], 0)   # v < 0


def _pred_record(rec, pred, offsets) -> None:
    rec["kind"] = _lib.OP_IF
    base, width = offsets[pred.register]
    if pred.index is not None:
        rec["pred_bit"], rec["pred_width"] = base + pred.index, 1
        width = 1
    else:
        if width > 64:
            raise BackendError(f"register predicates are limited to 64 bits (register {pred.register!r} has {width})")
        # an empty register (width 0) reads 0: no bits are gathered
        rec["pred_bit"], rec["pred_width"] = (0, 0) if width == 0 else (base, width)
    cmp, rhs = pred.comparator, int(pred.rhs)
    if cmp == "truthy":
        rec["pred_cmp"], rec["pred_rhs"] = _lib.CMP["truthy"], 0
        return
    if rhs < 0 or rhs > _M64:  # constant outcome for out-of-range right-hand sides
        big = rhs > 0
        truth = {"==": False, "!=": True, "<": big, "<=": big, ">": not big, ">=": not big}[cmp]
        rec["pred_cmp"], rec["pred_rhs"] = _ALWAYS if truth else _NEVER
        return
    rec["pred_cmp"], rec["pred_rhs"] = _lib.CMP[cmp], rhs


def _flatten(ops, out: list, offsets: dict) -> None:
    for op in ops:
        k = op_kind(op)
        if k == "gate":
            out.append(("gate", op))
        elif k == "measure":
            base, width = offsets[op.bit[0]]
            if not 0 <= op.bit[1] < width:
                raise SimError(f"bit {op.bit} outside register")
            out.append(("measure", op.qubit, base + op.bit[1]))
        elif k == "reset":
            out.append(("reset", op.qubit))
        elif k == "nop":
            continue
        else:
            out.append(("if", op.predicate))
            _flatten(op.then_body, out, offsets)
            if op.else_body:
                out.append(("else",))
                _flatten(op.else_body, out, offsets)
            out.append(("endif",))


def tape_records(kernel) -> np.ndarray:
    """The flat qsb_op record array of `kernel` (host only, no device needed)."""
    offsets = _classical_offsets([(n, int(w)) for n, w in kernel.classical_layout])
    flat: list = []
    _flatten(kernel.body, flat, offsets)
    recs = np.zeros(len(flat), dtype=_lib.OP_DTYPE)
    for i, item in enumerate(flat):
        r = recs[i]
        if item[0] == "gate":
            _gate_record(r, item[1], True)
        elif item[0] == "measure":
            r["kind"], r["qubit"], r["bit"] = _lib.OP_MEASURE, item[1], item[2]
        elif item[0] == "reset":
            r["kind"], r["qubit"] = _lib.OP_RESET, item[1]
        elif item[0] == "if":
            _pred_record(r, item[1], offsets)
        elif item[0] == "else":
            r["kind"] = _lib.OP_ELSE
        else:
            r["kind"] = _lib.OP_ENDIF
    return recs


class Tape:
    """A compiled Kernel on one device context (qsb_tape)."""

    def __init__(self, kernel, ctx: _lib.Context):
        # no reference to `kernel`: the cache entry dies with the kernel (compile_tape)
        self.ctx = ctx
        self.n = int(kernel.qubit_count)
        self.layout = [(n, int(w)) for n, w in kernel.classical_layout]
        self.offsets = _classical_offsets(self.layout)
        self.nbits = sum(w for _, w in self.layout)
        self.nwords = max(1, (self.nbits + 63) // 64)
        self.nparams = sum(p.count for p in kernel.param_layout)
        recs = tape_records(kernel)
        self.records = recs
        self.ngates_static = int(np.count_nonzero(recs["kind"] == _lib.OP_GATE))
        h = ctypes.c_void_p()
        _lib.check(ctx.lib.qsb_tape_create(ctx.handle, _lib.ptr(recs), len(recs), self.n, self.nbits,
                                           self.nparams, ctypes.byref(h)))
        self.handle = h
        dyn = ctypes.c_int32()
        _lib.check(ctx.lib.qsb_tape_is_dynamic(h, ctypes.byref(dyn)))
        self.dynamic = bool(dyn.value)
        self._finalizer = weakref.finalize(self, ctx.lib.qsb_tape_destroy, h)

    def params(self, values) -> np.ndarray | None:
        if self.nparams == 0:
            return None
        v = np.ascontiguousarray(values, dtype=np.float64)
        return v

    def keys(self, words: np.ndarray) -> list:
        """Packed classical words [shots][nwords] -> ClassicalStore.key() strings."""
        if self.nbits == 0:
            return [""] * len(words)
        bits = np.zeros((len(words), self.nbits), dtype=np.uint8)
        for f in range(self.nbits):
            bits[:, f] = (words[:, f >> 6] >> np.uint64(f & 63)) & np.uint64(1)
        rows = (bits + ord("0")).view(f"S{self.nbits}") if bits.flags.c_contiguous else None
        return [r.decode() for r in rows.reshape(-1)]


_tape_cache: dict = {}


def compile_tape(kernel, device=None) -> Tape:
    """The tape of `kernel` on `device`, compiled on first use and cached for the
    kernel's lifetime (compile-once; `bind` never recompiles)."""
    ctx = _ctx(device)
    key = (id(kernel), ctx.device)
    hit = _tape_cache.get(key)
    if hit is not None:
        tape, body_id, body_len = hit
        if body_id == id(kernel.body) and body_len == len(kernel.body):
            return tape
    tape = Tape(kernel, ctx)
    _tape_cache[key] = (tape, id(kernel.body), len(kernel.body))
    try:
        weakref.finalize(kernel, _tape_cache.pop, key, None)
    except TypeError:  # un-weakref-able kernel objects just stay cached
        pass
    return tape


# ---------------------------------------------------------------------------
# StateVector (sim.py:80-95): device-resident amplitudes, host view on demand
# ---------------------------------------------------------------------------


class StateVector:
    """Dense state, qubit k = index bit k, resident on the device.

    `amps` downloads a host snapshot on first access and hands it out READ-ONLY, so a
    caller that only reads it (every caller in the reference: suites.py, cli.py:104,
    its tests) costs one download and no re-upload -- the device copy stays
    authoritative.  Writing works as with the reference's numpy buffer (sim.py:80-95)
    in two explicit ways: assign `state.amps = array`, or flip the snapshot's
    `flags.writeable` back on and edit it in place; either way the host array is
    uploaded before the next device operation.  An in-place write to the read-only
    snapshot raises numpy's ValueError instead of being silently lost."""

    def __init__(self, n: int, amps: np.ndarray | None = None, *, precision=None, device=None):
        self.n = int(n)
        self._ctx = _ctx(device)
        self._prec = _prec(precision)
        h = ctypes.c_void_p()
        _lib.check(self._ctx.lib.qsb_state_create(self._ctx.handle, self.n, self._prec, ctypes.byref(h)))
        self._h = h
        self._fin = weakref.finalize(self, self._ctx.lib.qsb_state_destroy, h)
        self._host = None
        self._host_snapshot = False  # True: _host is an unmodified read-only download
        if amps is not None:
            a = np.ascontiguousarray(amps, dtype=np.complex128)
            if a.shape != (1 << self.n,):
                raise SimError(f"amplitude vector of shape {a.shape} for {self.n} qubits")
            self._host = a

    @classmethod
    def zero(cls, n: int, *, precision=None, device=None) -> "StateVector":
        return cls(n, precision=precision, device=device)

    # device sync ---------------------------------------------------------
    def _device(self):
        """Handle with the device copy current (uploads a handed-out host view that
        the caller modified, or one that was assigned)."""
        if self._host is not None:
            if not self._host_snapshot or self._host.flags.writeable:
                _lib.check(self._ctx.lib.qsb_state_set(self._h, _lib.ptr(np.ascontiguousarray(self._host))))
                self.uploads += 1
            self._host = None
            self._host_snapshot = False
        return self._h

    uploads = 0  # host -> device state uploads (instrumentation for the tests)

    @property
    def amps(self) -> np.ndarray:
        if self._host is None:
            out = np.empty(1 << self.n, dtype=np.complex128)
            _lib.check(self._ctx.lib.qsb_state_get(self._h, _lib.ptr(out)))
            out.flags.writeable = False
            self._host = out
            self._host_snapshot = True
        return self._host

    @amps.setter
    def amps(self, value) -> None:
        a = np.ascontiguousarray(value, dtype=np.complex128)
        if a.shape != (1 << self.n,):
            raise SimError(f"amplitude vector of shape {a.shape} for {self.n} qubits")
        self._host = a
        self._host_snapshot = False

    @property
    def precision(self) -> str:
        return "c64" if self._prec == _lib.C64 else "c128"

    def __array__(self, dtype=None, copy=None):
        """numpy interop (`np.asarray(state)`): the amplitudes, as for callers that
        treat a StateVector and an amplitude array alike (oracle.py:121-127)."""
        a = self.amps
        return a if dtype is None else a.astype(dtype)

    def norm(self) -> float:
        out = ctypes.c_double()
        _lib.check(self._ctx.lib.qsb_state_norm(self._device(), ctypes.byref(out)))
        return float(out.value)

    def copy(self) -> "StateVector":
        dup = StateVector(self.n, precision=self.precision, device=self._ctx.device)
        _lib.check(self._ctx.lib.qsb_state_copy(dup._h, self._device()))
        return dup

    def __repr__(self) -> str:
        return f"StateVector(n={self.n}, precision={self.precision}, device={self._ctx.device})"


# ---------------------------------------------------------------------------
# per-op API (sim.py:203-259)
# ---------------------------------------------------------------------------


def apply_gate(state: StateVector, op, params=()) -> StateVector:
    """Apply one canonical gate op in place; returns the same StateVector."""
    rec = np.zeros(1, dtype=_lib.OP_DTYPE)
    _gate_record(rec[0], op, True)
    if any(_is_ref(a) for a in op.angles):  # resolve ParamRef on the host (gate_matrix)
        m = gate_matrix(op, params)
        if op.base != "swap":
            rec["mat"][0][:] = [m[0, 0].real, m[0, 0].imag, m[0, 1].real, m[0, 1].imag,
                                m[1, 0].real, m[1, 0].imag, m[1, 1].real, m[1, 1].imag]
        rec["has_matrix"] = 1
        rec["angle_slot"][0][:] = -1
    _lib.check(state._ctx.lib.qsb_apply_gate(state._device(), _lib.ptr(rec), None, 0))
    return state


def measure(state: StateVector, qubit: int, rng, store=None, target_bit=None) -> int:
    """Projective Z measurement: collapse, renormalise, record the outcome."""
    u = rng.uniform()
    out = ctypes.c_int32()
    p1 = ctypes.c_double()
    rc = state._ctx.lib.qsb_measure(state._device(), int(qubit), float(u), ctypes.byref(out), ctypes.byref(p1))
    if rc == _lib.ERR_DEGENERATE:
        pout = p1.value if out.value == 1 else 1.0 - p1.value
        raise DegenerateNorm(
            f"selected measurement branch {out.value} on qubit {qubit} has probability {pout}"
        )
    _lib.check(rc)
    if store is not None and target_bit is not None:
        store.write_bit(target_bit[0], target_bit[1], out.value)
    return out.value


def reset(state: StateVector, qubit: int, rng) -> StateVector:
    """Force a qubit to |0>: measure, then flip if the outcome was 1."""
    u = rng.uniform()
    out = ctypes.c_int32()
    rc = state._ctx.lib.qsb_reset(state._device(), int(qubit), float(u), ctypes.byref(out))
    if rc == _lib.ERR_DEGENERATE:
        raise DegenerateNorm(f"selected measurement branch {out.value} on qubit {qubit} is degenerate")
    _lib.check(rc)
    return state


_CMPF = {
    "==": lambda a, b: a == b,
    "!=": lambda a, b: a != b,
    "<": lambda a, b: a < b,
    "<=": lambda a, b: a <= b,
    ">": lambda a, b: a > b,
    ">=": lambda a, b: a >= b,
}


def _eval_predicate(pred, store) -> bool:
    """sim.py:262-276 (host-side classical logic)."""
    value = store.read_bit(pred.register, pred.index) if pred.index is not None else store.register_uint(pred.register)
    if pred.comparator == "truthy":
        return value != 0
    return _CMPF[pred.comparator](value, pred.rhs)


def _exec_ops(ops, state, store, params, rng, trace) -> None:
    """Op-by-op interpreter (sim.py:279-303): every op is one device call; the
    predicate is evaluated once per CondBlock on the host classical store."""
    for op in ops:
        k = op_kind(op)
        if k == "gate":
            apply_gate(state, op, params)
        elif k == "measure":
            measure(state, op.qubit, rng, store, op.bit)
        elif k == "reset":
            reset(state, op.qubit, rng)
        elif k == "nop":
            continue
        else:
            taken = _eval_predicate(op.predicate, store)
            if trace is not None:
                trace.append((op.predicate, {n: list(b) for n, b in store.bits.items()}, taken))
            _exec_ops(op.then_body if taken else op.else_body, state, store, params, rng, trace)


def _needs_trajectories(kernel) -> bool:
    """sim.py:322-335: any top-level CondBlock / Reset, a re-measured qubit, or a
    gate after a measurement selects the trajectory path."""
    measured: set = set()
    for op in kernel.body:
        k = op_kind(op)
        if k in ("cond", "reset"):
            return True
        if k == "measure":
            if op.qubit in measured:
                return True
            measured.add(op.qubit)
        elif k == "gate" and measured:
            return True
    return False


# ---------------------------------------------------------------------------
# whole-kernel entry points
# ---------------------------------------------------------------------------


def _predicates_of(ops, out: list) -> None:
    for op in ops:
        if op_kind(op) == "cond":
            out.append(op.predicate)
            _predicates_of(op.then_body, out)
            _predicates_of(op.else_body, out)


def run_trajectory(bound, rng, trace=None, *, precision=None, device=None):
    """Execute one stochastic shot (sim.py:306-314) on the device.  `rng` is
    advanced by exactly the uniforms consumed.  For xoshiro streams the whole
    shot is one device call; any other object with `.uniform()` (e.g. a
    pre-drawn stream) is driven op by op through the per-op device kernels."""
    kernel = bound.kernel
    words = _rng_words(rng)
    if words is None:
        state = StateVector.zero(kernel.qubit_count, precision=precision, device=device)
        store = ClassicalStore(kernel.classical_layout)
        _exec_ops(kernel.body, state, store, bound.values, rng, trace)
        return store, state
    tape = compile_tape(kernel, device)
    ctx = tape.ctx
    prec = _prec(precision)
    state = StateVector(tape.n, precision="c64" if prec == _lib.C64 else "c128", device=ctx.device)
    params = tape.params(bound.values)
    bits = np.zeros(tape.nwords, dtype=np.uint64)
    preds: list = []
    _predicates_of(kernel.body, preds)
    max_trace = 4096 if trace is not None else 0
    tbuf = np.zeros(max(1, max_trace) * (2 + tape.nwords), dtype=np.int64) if trace is not None else None
    nt, nd = ctypes.c_int32(), ctypes.c_int32()
    rc = ctx.lib.qsb_run_trajectory(tape.handle, prec, _lib.ptr(params), _lib.ptr(words), 0, 0, None, 0,
                                    _lib.ptr(bits), state._h, _lib.ptr(tbuf), max_trace, ctypes.byref(nt),
                                    ctypes.byref(nd))
    rng.s0, rng.s1, rng.s2, rng.s3 = (int(w) for w in words)
    _lib.check(rc)
    store = ClassicalStore._from_words(tape.layout, bits)
    if trace is not None:
        if nt.value > max_trace:
            raise BackendError("trace longer than the 4096-entry device buffer")
        ifs = [i for i, r in enumerate(tape.records) if r["kind"] == _lib.OP_IF]
        pred_of = dict(zip(ifs, preds))
        for e in range(nt.value):
            row = tbuf[e * (2 + tape.nwords):(e + 1) * (2 + tape.nwords)]
            snap = ClassicalStore._from_words(tape.layout, row[2:].astype(np.uint64))
            trace.append((pred_of[int(row[0])], {n: list(b) for n, b in snap.bits.items()}, bool(row[1])))
    return store, state


def sample_words(bound, shots: int, seed: int, *, shot_begin: int = 0, precision=None, device=None,
                 predrawn=None) -> tuple[np.ndarray, Tape]:
    """Per-shot packed classical words [shots][nwords] for global shots
    [shot_begin, shot_begin + shots) -- the sharding primitive under `sample`."""
    if shots < 1:
        raise SimError("shots must be >= 1")
    tape = compile_tape(bound.kernel, device)
    ctx = tape.ctx
    out = np.zeros((shots, tape.nwords), dtype=np.uint64)
    params = tape.params(bound.values)
    seed64 = int(seed) & _M64
    if tape.dynamic or predrawn is not None:
        pre = None
        stride = 0
        if predrawn is not None:
            pre = np.ascontiguousarray(predrawn, dtype=np.float64)
            stride = pre.shape[1]
        status = np.zeros(shots, dtype=np.int32)
        rc = ctx.lib.qsb_sample_trajectories(tape.handle, _prec(precision), _lib.ptr(params), seed64,
                                             int(shot_begin), int(shots), _lib.ptr(pre), stride, _lib.ptr(out),
                                             _lib.ptr(status))
        _lib.check(rc)
    else:
        _lib.check(ctx.lib.qsb_sample_static(tape.handle, _prec(precision), _lib.ptr(params), seed64,
                                             int(shot_begin), int(shots), _lib.ptr(out)))
    return out, tape


def sample_final_states(bound, shots: int, seed: int, nstates: int, *, shot_begin: int = 0, precision=None,
                        device=None) -> tuple[np.ndarray, list]:
    """`sample_words` of global shots [shot_begin, shot_begin + shots) through the batched
    streaming engine, plus the final StateVector of the first `nstates` of those shots
    as that engine left them (history dedup, fused passes, collapse applied) -- what
    run_trajectory (sim.py:306-314) returns for each, for parity checks of the
    production path at config size."""
    if shots < 1:
        raise SimError("shots must be >= 1")
    tape = compile_tape(bound.kernel, device)
    ctx = tape.ctx
    pname = "c64" if _prec(precision) == _lib.C64 else "c128"
    states = [StateVector(tape.n, precision=pname, device=ctx.device) for _ in range(nstates)]
    handles = (ctypes.c_void_p * max(1, nstates))(*[st._h.value for st in states])
    out = np.zeros((shots, tape.nwords), dtype=np.uint64)
    status = np.zeros(shots, dtype=np.int32)
    _lib.check(ctx.lib.qsb_sample_trajectories_states(tape.handle, _prec(precision), _lib.ptr(tape.params(bound.values)),
                                                      int(seed) & _M64, int(shot_begin), int(shots), _lib.ptr(out),
                                                      _lib.ptr(status), int(nstates), ctypes.cast(handles, ctypes.c_void_p)))
    return out, states


def histogram_from_words(tape: Tape, words: np.ndarray, shots: int) -> ShotHistogram:
    if tape.nbits == 0:
        return ShotHistogram({"": int(shots)}, int(shots))
    uniq, counts = np.unique(words, axis=0, return_counts=True)
    keys = tape.keys(uniq)
    return ShotHistogram({k: int(c) for k, c in zip(keys, counts)}, int(shots))


def sample(bound, shots: int, seed: int, workers: int = 1, *, precision=None, device=None) -> ShotHistogram:
    """Sample the kernel; identical (seed, shots) gives identical histograms
    regardless of `workers` (accepted for signature compatibility: every shot
    derives its own RNG stream from (seed, global shot index), so the device
    batch layout cannot change the result)."""
    if shots < 1:
        raise SimError("shots must be >= 1")
    tape = compile_tape(bound.kernel, device)
    if tape.nwords == 1:
        uniq, counts = sample_counts(bound, shots, seed, precision=precision, device=device)
        keys = tape.keys(uniq) if tape.nbits else [""] * len(uniq)
        return ShotHistogram({k: int(c) for k, c in zip(keys, counts)}, int(shots))
    words, tape = sample_words(bound, shots, seed, precision=precision, device=device)
    return histogram_from_words(tape, words, shots)


def sample_counts(bound, shots: int, seed: int, *, shot_begin: int = 0, precision=None,
                  device=None) -> tuple[np.ndarray, np.ndarray]:
    """Distinct per-shot words (ascending) and their counts, histogrammed on the
    device (qsb_sample_counts): only the distinct outcomes leave the GPU."""
    if shots < 1:
        raise SimError("shots must be >= 1")
    tape = compile_tape(bound.kernel, device)
    ctx = tape.ctx
    params = tape.params(bound.values)
    cap = min(int(shots), 1 << min(tape.nbits, 40))
    while True:
        uniq = np.zeros((cap, 1), dtype=np.uint64)
        counts = np.zeros(cap, dtype=np.int64)
        nu = ctypes.c_int64()
        rc = ctx.lib.qsb_sample_counts(tape.handle, _prec(precision), _lib.ptr(params), int(seed) & _M64,
                                       int(shot_begin), int(shots), _lib.ptr(uniq), _lib.ptr(counts), cap,
                                       ctypes.byref(nu))
        if rc == _lib.ERR_ARG and nu.value > cap:  # pragma: no cover - cap >= shots >= distinct outcomes
            cap = nu.value
            continue
        _lib.check(rc)
        return uniq[:nu.value], counts[:nu.value]


def statevector(bound, *, precision=None, device=None) -> StateVector:
    """Final state of a static (measurement- and reset-free) kernel."""
    for op in bound.kernel.body:
        if op_kind(op) in ("measure", "cond", "reset"):
            raise DynamicCircuit(f"{type(op).__name__} requires trajectory sampling; use sample()")
    tape = compile_tape(bound.kernel, device)
    st = StateVector(tape.n, precision=precision, device=tape.ctx.device)
    _lib.check(tape.ctx.lib.qsb_statevector(tape.handle, _lib.ptr(tape.params(bound.values)), st._h))
    return st


def _pauli_masks(word: str, n: int):
    if len(word) != n:
        raise BadPauliString(f"pauli string length {len(word)} != {n} qubits")
    if any(ch not in "IXYZ" for ch in word):
        raise BadPauliString(f"pauli string may only contain I, X, Y, Z: {word!r}")
    x = z = ny = 0
    for q, ch in enumerate(word):
        if ch in "XY":
            x |= 1 << q
        if ch in "ZY":
            z |= 1 << q
        if ch == "Y":
            ny += 1
    return x, z, ny


def expval_pauli(state: StateVector, pauli: str) -> float:
    """<psi|P|psi> for a Pauli string; character k acts on qubit k."""
    x, z, ny = _pauli_masks(pauli, state.n)
    out = ctypes.c_double()
    _lib.check(state._ctx.lib.qsb_expval_pauli(state._device(), x, z, ny, ctypes.byref(out)))
    return float(out.value)


def observe(bound_or_kernel, hamiltonian, points=None, *, precision=None, device=None, return_terms=False):
    """Energies E[p] = sum_k c_k <psi(theta_p)|P_k|psi(theta_p)> for a static kernel,
    batched over parameter points on the device (the VQE observe() of BASELINE
    cfg 3).  `hamiltonian` is [(coef, pauli_word)], letter q acting on qubit q.
    `points` is [npoints][nparams] (defaults to the bound values)."""
    if hasattr(bound_or_kernel, "kernel"):
        kernel = bound_or_kernel.kernel
        if points is None:
            points = [bound_or_kernel.values]
    else:
        kernel = bound_or_kernel
        if points is None:
            points = [()]
    for op in kernel.body:
        if op_kind(op) in ("measure", "cond", "reset"):
            raise DynamicCircuit(f"{type(op).__name__} requires trajectory sampling; use sample()")
    tape = compile_tape(kernel, device)
    n = tape.n
    terms = list(hamiltonian)
    xm = np.zeros(len(terms), dtype=np.uint64)
    zm = np.zeros(len(terms), dtype=np.uint64)
    ny = np.zeros(len(terms), dtype=np.int32)
    coef = np.zeros(len(terms), dtype=np.float64)
    for i, (c, w) in enumerate(terms):
        x, z, y = _pauli_masks(w, n)
        xm[i], zm[i], ny[i], coef[i] = x, z, y, float(c)
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(len(points), -1))
    if pts.shape[1] != tape.nparams:
        from .errors import ArityMismatch

        raise ArityMismatch(f"kernel takes {tape.nparams} parameter value(s), got {pts.shape[1]}")
    energies = np.zeros(len(pts), dtype=np.float64)
    tv = np.zeros((len(pts), max(1, len(terms))), dtype=np.float64) if return_terms else None
    _lib.check(tape.ctx.lib.qsb_observe(tape.handle, _prec(precision), _lib.ptr(pts) if tape.nparams else None,
                                        len(pts), _lib.ptr(xm), _lib.ptr(zm), _lib.ptr(ny), _lib.ptr(coef),
                                        len(terms), _lib.ptr(energies), _lib.ptr(tv)))
    if return_terms:
        return energies, tv[:, : len(terms)]
    return energies
