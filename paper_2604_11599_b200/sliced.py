"""Global-qubit slicing of one state vector over 2^G slices (BASELINE cfg 5:
34 qubits complex128 over 8 B200s).

Layout.  The top G *physical* qubit positions are global: slice s holds the 2^L
amplitudes (L = n - G) whose physical global bits equal `s ^ gframe`.  Logical qubit q
lives at physical position perm[q].  One slice per rank (one GPU per process) in
production; all slices in one process for the single-device emulation used by the
tests.

Operations (reference semantics: sim.py:203-259, 279-314):
* gate with local targets: applied to every slice by the device kernels; controls on
  global qubits select slices, controls on local qubits go to the kernel;
* diagonal gate on a global target: a per-slice phase (folded into a diagonal gate on
  a local control qubit when there is one);
* non-diagonal gate on a global target: the global qubit is first swapped with the
  top local position -- partner slices (s, s ^ bit) exchange one contiguous half of
  their buffers (the only data movement: NCCL send/recv between GPUs, a device copy in
  emulation) -- then applied locally;
* swap gates are relabelings of `perm` (no data movement); X on a global qubit after
  a reset flips `gframe`;
* measure / reset: per-slice partial probabilities (deterministic device reductions)
  summed in slice order -- identical on every rank -- then every rank draws the same
  uniform from the same stream, so decisions agree without further communication.

The slice backend (device kernels) and the transport (exchange / all-gather) are
injected; `GpuSliceBackend` + `LocalTransport` / `DistTransport` are the product
paths.  Local gates between two exchanges / measurements run as one fused tape per
slice (`GpuSliceBackend.flush`, C ABI `qsb_apply_tape`).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from .errors import DegenerateNorm
from .ir import op_kind

_DIAG = frozenset(("z", "s", "t", "rz", "p"))


class _G:  # minimal Gate stand-in for local application
    __slots__ = ("base", "angles", "targets", "controls", "adjoint")

    def __init__(self, base, targets, controls, adjoint=False, angles=()):
        self.base, self.targets, self.controls, self.adjoint, self.angles = base, targets, controls, adjoint, angles


# ---------------------------------------------------------------------------
# backends
# ---------------------------------------------------------------------------


class GpuSliceBackend:
    """Slices are device StateVectors on one GPU; kernels through the C ABI.

    Local gates are queued per slice and run as ONE fused tape (`qsb_apply_tape`: the
    streaming engine's register-blocked passes, in place) when the slice is next
    needed for anything else -- an exchange, a probability, a collapse, a scale or a
    read -- so the gates between two exchanges cost a few state passes instead of one
    pass each.  The fused tapes use the generic kernel (no per-tape NVRTC compile).
    Small slices (the 1-GPU emulations) stay per-op: building a tape costs more than
    a pass over them."""

    # below this many local qubits a slice pass is cheaper than building a fused tape
    # (tape + plan construction costs ~ms on the host)
    FUSE_MIN_LOCAL = 24

    def __init__(self, precision=None, device=None, fuse: bool | None = None):
        self.precision = precision
        self.device = device
        self.fuse = fuse  # None: fuse slices of >= FUSE_MIN_LOCAL qubits
        self._queue: dict = {}  # id(slice) -> (slice, [qsb_op records])

    def new_slice(self, L: int, initial_one: bool):
        from . import sim

        st = sim.StateVector.zero(L, precision=self.precision, device=self.device)
        if not initial_one:
            self.scale(st, 0.0)
        return st

    def flush(self, st=None) -> None:
        """Run the queued gates of `st` (or of every slice) as one fused tape."""
        from . import _lib

        keys = [id(st)] if st is not None else list(self._queue)
        for key in keys:
            item = self._queue.pop(key, None)
            if item is None:
                continue
            sl, recs = item
            ops = np.concatenate(recs)
            ctx = sl._ctx
            tape = ctypes.c_void_p()
            ctx.set_option("jit", 0)
            try:
                _lib.check(ctx.lib.qsb_tape_create(ctx.handle, _lib.ptr(ops), len(ops), sl.n, 0, 0, ctypes.byref(tape)))
                try:
                    _lib.check(ctx.lib.qsb_apply_tape(tape, None, sl._device()))
                finally:
                    ctx.lib.qsb_tape_destroy(tape)
            finally:
                ctx.set_option("jit", 1)

    def apply(self, st, base, matrix, target, ctrl_local):
        from . import _lib

        rec = np.zeros(1, dtype=_lib.OP_DTYPE)
        r = rec[0]
        r["kind"] = _lib.OP_GATE
        r["base"] = _lib.BASES[base]  # selects the update class (perm / anti / diag / dense)
        r["ntargets"] = 1
        r["target"][0] = target
        cm = cv = 0
        for q, pol in ctrl_local:
            cm |= 1 << q
            cv |= (1 << q) if pol else 0
        r["ctrl_mask"], r["ctrl_val"] = cm, cv
        r["angle_slot"][:] = -1
        rec["mat"][0][:] = [matrix[0, 0].real, matrix[0, 0].imag, matrix[0, 1].real, matrix[0, 1].imag,
                            matrix[1, 0].real, matrix[1, 0].imag, matrix[1, 1].real, matrix[1, 1].imag]
        rec["has_matrix"] = 1
        if self.fuse or (self.fuse is None and st.n >= self.FUSE_MIN_LOCAL):
            self._queue.setdefault(id(st), (st, []))[1].append(rec)
            return
        _lib.check(st._ctx.lib.qsb_apply_gate(st._device(), _lib.ptr(rec), None, 0))

    def scale(self, st, c: complex):
        from . import _lib

        self.flush(st)
        c = complex(c)
        _lib.check(st._ctx.lib.qsb_state_scale(st._device(), c.real, c.imag))

    def prob1(self, st, q: int) -> float:
        from . import _lib

        self.flush(st)
        out = ctypes.c_double()
        _lib.check(st._ctx.lib.qsb_state_prob1(st._device(), int(q), ctypes.byref(out)))
        return float(out.value)

    def collapse(self, st, q, outcome, scale, flip):
        from . import _lib

        self.flush(st)
        _lib.check(st._ctx.lib.qsb_state_collapse(st._device(), int(q), int(outcome), float(scale), int(flip)))

    def view(self, st):
        """Zero-copy torch view (float64 / float32 pairs) of the slice's device buffer."""
        import torch

        from . import _lib

        self.flush(st)
        ptr = ctypes.c_void_p()
        _lib.check(st._ctx.lib.qsb_state_device_ptr(st._device(), ctypes.byref(ptr)))
        st._ctx.synchronize()
        c64 = st.precision == "c64"

        class _Buf:
            __cuda_array_interface__ = {"shape": (2 << st.n,), "typestr": "<f4" if c64 else "<f8",
                                        "data": (ptr.value, False), "version": 3, "strides": None}

        return torch.as_tensor(_Buf(), device=f"cuda:{st._ctx.device}")

    def sync_after_transport(self, st):
        import torch

        torch.cuda.synchronize(st._ctx.device)

    def to_numpy(self, st) -> np.ndarray:
        self.flush(st)
        return st.amps.copy()


# ---------------------------------------------------------------------------
# transports
# ---------------------------------------------------------------------------


class LocalTransport:
    """All slices in this process (single-device emulation of 2^G ranks)."""

    def __init__(self, nslices: int):
        self.nslices = nslices
        self.owned = list(range(nslices))

    def exchange(self, backend, slices, pairs):
        """pairs: [(a, b)] where slice a sends/receives its upper half, b its lower."""
        for a, b in pairs:
            va, vb = backend.view(slices[a]), backend.view(slices[b])
            h = va.numel() // 2
            tmp = va[h:].clone()
            va[h:].copy_(vb[:h])
            vb[:h].copy_(tmp)
            backend.sync_after_transport(slices[a])

    def allgather_sum(self, values: dict) -> float:
        return float(sum(values[s] for s in range(self.nslices)))


class DistTransport:
    """One slice per rank of the default torch.distributed group (NCCL on GPUs,
    gloo for the CPU protocol tests)."""

    def __init__(self):
        import torch.distributed as dist

        self.dist = dist
        self.rank = dist.get_rank()
        self.nslices = dist.get_world_size()
        self.owned = [self.rank]

    def exchange(self, backend, slices, pairs):
        dist = self.dist
        for a, b in pairs:
            if self.rank not in (a, b):
                continue
            me = self.rank
            peer = b if me == a else a
            v = backend.view(slices[me])
            h = v.numel() // 2
            half = v[h:] if me == a else v[:h]
            tmp = half.clone()
            ops = [dist.P2POp(dist.isend, tmp, peer), dist.P2POp(dist.irecv, half, peer)]
            for r in dist.batch_isend_irecv(ops):
                r.wait()
            backend.sync_after_transport(slices[me])

    def allgather_sum(self, values: dict) -> float:
        import torch

        parts = [None] * self.nslices
        self.dist.all_gather_object(parts, float(values[self.rank]))
        return float(sum(parts))  # rank order


# ---------------------------------------------------------------------------
# the sliced executor
# ---------------------------------------------------------------------------


class SlicedState:
    def __init__(self, n: int, G: int, backend, transport):
        if not 0 <= G < n:
            raise ValueError("need 0 <= G < n")
        self.n, self.G, self.L = n, G, n - G
        self.backend, self.transport = backend, transport
        self.perm = list(range(n))  # logical -> physical
        self.gframe = 0
        self.slices = {s: backend.new_slice(self.L, s == 0) for s in transport.owned}
        self.exchanges = 0

    # -- helpers --------------------------------------------------------------
    def content(self, s: int) -> int:
        return s ^ self.gframe

    def gbit(self, s: int, pos: int) -> int:
        return (self.content(s) >> (pos - self.L)) & 1

    def _swap_to_local(self, gpos: int) -> None:
        """Exchange global position gpos with the top local position L-1."""
        top = self.L - 1
        bit = 1 << (gpos - self.L)
        pairs = []
        for s in range(2**self.G):
            if self.content(s) & bit == 0:
                partner = s ^ bit
                pairs.append((s, partner))  # s keeps content bit 0: sends/receives its upper half
        self.transport.exchange(self.backend, self.slices, pairs)
        self.exchanges += 1
        qa, qb = self.perm.index(gpos), self.perm.index(top)
        self.perm[qa], self.perm[qb] = top, gpos

    # -- operations ----------------------------------------------------------
    def apply_gate(self, op, params=()) -> None:
        from .sim import gate_matrix

        base = op.base
        if base == "swap":
            a, b = op.targets
            if not op.controls:
                self.perm[a], self.perm[b] = self.perm[b], self.perm[a]
                return
            # Fredkin = CX(b->a) . CCX(ctrls, a -> b) . CX(b->a)
            seq = [_G("x", (a,), ((b, 1),)), _G("x", (b,), tuple(op.controls) + ((a, 1),)), _G("x", (a,), ((b, 1),))]
            for g in seq:
                self.apply_gate(g)
            return
        m = gate_matrix(op, params)
        t = self.perm[op.targets[0]]
        if t >= self.L and base not in _DIAG:
            self._swap_to_local(t)
            t = self.perm[op.targets[0]]
        ctrl = [(self.perm[q], pol) for q, pol in op.controls]
        local = [(p, pol) for p, pol in ctrl if p < self.L]
        glob = [(p, pol) for p, pol in ctrl if p >= self.L]
        for s, st in self.slices.items():
            if any(self.gbit(s, p) != pol for p, pol in glob):
                continue
            if t < self.L:
                self.backend.apply(st, base, m, t, local)
                continue
            d = m[1, 1] if self.gbit(s, t) else m[0, 0]
            if d == 1:
                continue
            if not local:
                self.backend.scale(st, d)
            else:  # phase on the first local control, the rest stay controls
                (c, pol), rest = local[0], local[1:]
                dm = np.array([[1, 0], [0, d]] if pol else [[d, 0], [0, 1]], dtype=np.complex128)
                # a general diagonal ("rz" class): with pol = 0 the |0> entry is not 1
                self.backend.apply(st, "rz", dm, c, rest)

    def _p1(self, q: int) -> float:
        p = self.perm[q]
        vals = {}
        for s, st in self.slices.items():
            if p < self.L:
                vals[s] = self.backend.prob1(st, p)
            else:
                vals[s] = self.backend.prob1(st, -1) if self.gbit(s, p) else 0.0
        return self.transport.allgather_sum(vals)

    def measure(self, q: int, rng, flip_if_one: bool = False) -> int:
        """sim.py:230-259 on the sliced state (reset = flip_if_one)."""
        p = self.perm[q]
        p1 = self._p1(q)
        u = rng.uniform()
        outcome = 1 if u < p1 else 0
        p_out = p1 if outcome == 1 else 1.0 - p1
        if p_out < 1e-15:
            raise DegenerateNorm(f"selected measurement branch {outcome} on qubit {q} has probability {p_out}")
        scale = 1.0 / math.sqrt(p_out)
        flip = flip_if_one and outcome == 1
        for s, st in self.slices.items():
            if p < self.L:
                self.backend.collapse(st, p, outcome, scale, 1 if flip else 0)
            else:
                self.backend.scale(st, scale if self.gbit(s, p) == outcome else 0.0)
        if flip and p >= self.L:
            self.gframe ^= 1 << (p - self.L)
        return outcome

    def gather(self) -> np.ndarray:
        """Logical amplitude vector (all slices must be local to this process)."""
        out = np.zeros(1 << self.n, dtype=np.complex128)
        local_idx = np.arange(1 << self.L)
        for s, st in self.slices.items():
            a = self.backend.to_numpy(st)
            phys = (self.content(s) << self.L) | local_idx
            logical = np.zeros_like(phys)
            for q in range(self.n):
                logical |= ((phys >> self.perm[q]) & 1) << q
            out[logical] = a
        return out


def run_trajectory_sliced(bound, rng, global_qubits: int, *, backend=None, transport=None, trace=None):
    """run_trajectory (sim.py:306-314) on a state sliced over 2^global_qubits slices."""
    from .sim import ClassicalStore, _eval_predicate

    k = bound.kernel
    n = int(k.qubit_count)
    backend = backend or GpuSliceBackend()
    transport = transport or LocalTransport(2**global_qubits)
    st = SlicedState(n, global_qubits, backend, transport)
    store = ClassicalStore(k.classical_layout)

    def run(ops):
        for op in ops:
            kind = op_kind(op)
            if kind == "gate":
                st.apply_gate(op, bound.values)
            elif kind == "measure":
                store.write_bit(op.bit[0], op.bit[1], st.measure(op.qubit, rng))
            elif kind == "reset":
                st.measure(op.qubit, rng, flip_if_one=True)
            elif kind == "nop":
                continue
            else:
                taken = _eval_predicate(op.predicate, store)
                if trace is not None:
                    trace.append((op.predicate, {nm: list(b) for nm, b in store.bits.items()}, taken))
                run(op.then_body if taken else op.else_body)

    run(k.body)
    if hasattr(backend, "flush"):
        backend.flush()
    return store, st
